// Symbolic expressions for the host front-end (see include/twoscale/expr.hpp).
// Semantics follow the reference grammar and evaluation rules
// (/root/reference/proj/src/expr.cpp: parser 459-607, folding 76-143,
// derivatives 192-251, tape 617-701); the implementation is independent.
#include "twoscale/expr.hpp"

#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>

namespace twoscale {

const char* var_name(Var v) {
    static const char* names[4] = {"x0", "x1", "y0", "y1"};
    return names[static_cast<int>(v)];
}

namespace detail {

enum class K : unsigned char { Num, Sym, Par, Neg, Sin, Cos, Exp, Sqrt, Add, Sub, Mul, Div, Pow };

struct Node {
    K k;
    double num = 0.0;  // Num
    int idx = 0;       // Sym: variable index; Pow: exponent
    std::string name;  // Par
    NodePtr l, r;      // operands (unary uses l)
};

namespace {

bool is_unary(K k) { return k == K::Neg || k == K::Sin || k == K::Cos || k == K::Exp || k == K::Sqrt; }
bool is_binary(K k) { return k == K::Add || k == K::Sub || k == K::Mul || k == K::Div; }

NodePtr leaf_num(double v) {
    auto n = std::make_shared<Node>();
    n->k = K::Num;
    n->num = v;
    return n;
}

bool num_of(const NodePtr& n, double& v) {
    if (n->k != K::Num) return false;
    v = n->num;
    return true;
}

bool is_num(const NodePtr& n, double v) { return n->k == K::Num && n->num == v; }

NodePtr mk_unary(K k, NodePtr a);

// Constant folding and identity stripping, applied at every construction.
NodePtr mk_binary(K k, NodePtr a, NodePtr b) {
    double va = 0.0, vb = 0.0;
    const bool ca = num_of(a, va), cb = num_of(b, vb);
    if (k == K::Add) {
        if (ca && cb) return leaf_num(va + vb);
        if (is_num(a, 0.0)) return b;
        if (is_num(b, 0.0)) return a;
    } else if (k == K::Sub) {
        if (ca && cb) return leaf_num(va - vb);
        if (is_num(b, 0.0)) return a;
        if (is_num(a, 0.0)) return mk_unary(K::Neg, b);
    } else if (k == K::Mul) {
        if (ca && cb) return leaf_num(va * vb);
        if (is_num(a, 0.0) || is_num(b, 0.0)) return leaf_num(0.0);
        if (is_num(a, 1.0)) return b;
        if (is_num(b, 1.0)) return a;
    } else {  // Div
        if (is_num(a, 0.0) && !is_num(b, 0.0)) return leaf_num(0.0);
        if (ca && cb && vb != 0.0) return leaf_num(va / vb);
        if (is_num(b, 1.0)) return a;
    }
    auto n = std::make_shared<Node>();
    n->k = k;
    n->l = std::move(a);
    n->r = std::move(b);
    return n;
}

NodePtr mk_unary(K k, NodePtr a) {
    double v = 0.0;
    if (num_of(a, v)) {
        switch (k) {
            case K::Neg: return leaf_num(-v);
            case K::Sin: return leaf_num(std::sin(v));
            case K::Cos: return leaf_num(std::cos(v));
            case K::Exp: return leaf_num(std::exp(v));
            case K::Sqrt:
                if (v >= 0.0) return leaf_num(std::sqrt(v));
                break;
            default: break;
        }
    }
    if (k == K::Neg && a->k == K::Neg) return a->l;
    auto n = std::make_shared<Node>();
    n->k = k;
    n->l = std::move(a);
    return n;
}

NodePtr mk_pow(NodePtr a, int e) {
    if (e < 0) throw std::invalid_argument("negative exponent not supported");
    if (e == 0) return leaf_num(1.0);
    if (e == 1) return a;
    double v = 0.0;
    if (num_of(a, v)) return leaf_num(std::pow(v, e));
    auto n = std::make_shared<Node>();
    n->k = K::Pow;
    n->idx = e;
    n->l = std::move(a);
    return n;
}

double ipow(double a, int e) {  // repeated multiplication, as the reference tape does
    double r = 1.0;
    for (int i = 0; i < e; ++i) r *= a;
    return r;
}

double eval(const Node& n, const EvalEnv& env) {
    switch (n.k) {
        case K::Num: return n.num;
        case K::Sym: return env.vars[n.idx];
        case K::Par: {
            if (env.params) {
                auto it = env.params->find(n.name);
                if (it != env.params->end()) return it->second;
            }
            throw EvalError("unbound parameter '" + n.name + "'");
        }
        case K::Neg: return -eval(*n.l, env);
        case K::Sin: return std::sin(eval(*n.l, env));
        case K::Cos: return std::cos(eval(*n.l, env));
        case K::Exp: return std::exp(eval(*n.l, env));
        case K::Sqrt: {
            const double a = eval(*n.l, env);
            if (a < 0.0) throw EvalError("sqrt of negative value");
            return std::sqrt(a);
        }
        case K::Pow: return ipow(eval(*n.l, env), n.idx);
        case K::Add: return eval(*n.l, env) + eval(*n.r, env);
        case K::Sub: return eval(*n.l, env) - eval(*n.r, env);
        case K::Mul: return eval(*n.l, env) * eval(*n.r, env);
        case K::Div: {
            const double a = eval(*n.l, env), b = eval(*n.r, env);
            if (b == 0.0) throw EvalError("division by zero");
            return a / b;
        }
    }
    throw EvalError("corrupt expression");
}

NodePtr derive(const NodePtr& n, int v) {
    switch (n->k) {
        case K::Num:
        case K::Par: return leaf_num(0.0);
        case K::Sym: return leaf_num(n->idx == v ? 1.0 : 0.0);
        case K::Neg: return mk_unary(K::Neg, derive(n->l, v));
        case K::Sin: return mk_binary(K::Mul, mk_unary(K::Cos, n->l), derive(n->l, v));
        case K::Cos:
            return mk_unary(K::Neg, mk_binary(K::Mul, mk_unary(K::Sin, n->l), derive(n->l, v)));
        case K::Exp: return mk_binary(K::Mul, mk_unary(K::Exp, n->l), derive(n->l, v));
        case K::Sqrt:
            return mk_binary(K::Div, derive(n->l, v),
                             mk_binary(K::Mul, leaf_num(2.0), mk_unary(K::Sqrt, n->l)));
        case K::Add: return mk_binary(K::Add, derive(n->l, v), derive(n->r, v));
        case K::Sub: return mk_binary(K::Sub, derive(n->l, v), derive(n->r, v));
        case K::Mul:
            return mk_binary(K::Add, mk_binary(K::Mul, derive(n->l, v), n->r),
                             mk_binary(K::Mul, n->l, derive(n->r, v)));
        case K::Div:
            return mk_binary(K::Div,
                             mk_binary(K::Sub, mk_binary(K::Mul, derive(n->l, v), n->r),
                                       mk_binary(K::Mul, n->l, derive(n->r, v))),
                             mk_pow(n->r, 2));
        case K::Pow:
            return mk_binary(K::Mul,
                             mk_binary(K::Mul, leaf_num(static_cast<double>(n->idx)),
                                       mk_pow(n->l, n->idx - 1)),
                             derive(n->l, v));
    }
    throw EvalError("corrupt expression");
}

// Rebuilds a tree bottom-up through the smart constructors; `leaf` may replace leaves.
NodePtr rebuild(const NodePtr& n, const std::function<NodePtr(const NodePtr&)>& leaf) {
    if (n->k == K::Num || n->k == K::Sym || n->k == K::Par) return leaf(n);
    if (n->k == K::Pow) return mk_pow(rebuild(n->l, leaf), n->idx);
    if (is_unary(n->k)) return mk_unary(n->k, rebuild(n->l, leaf));
    return mk_binary(n->k, rebuild(n->l, leaf), rebuild(n->r, leaf));
}

bool uses(const Node& n, int v) {
    if (n.k == K::Sym) return n.idx == v;
    if (n.l && uses(*n.l, v)) return true;
    return n.r && uses(*n.r, v);
}

void params_of(const Node& n, std::set<std::string>& out) {
    if (n.k == K::Par) out.insert(n.name);
    if (n.l) params_of(*n.l, out);
    if (n.r) params_of(*n.r, out);
}

// Printing: precedence 1 (+ -), 2 (* /), 3 (unary -), 4 (^), 5 (atoms, calls).
int prec(const Node& n) {
    if (n.k == K::Add || n.k == K::Sub) return 1;
    if (n.k == K::Mul || n.k == K::Div) return 2;
    if (n.k == K::Neg) return 3;
    if (n.k == K::Pow) return 4;
    return 5;
}

void print(const Node& n, std::string& s, int outer) {
    const int p = prec(n);
    if (p < outer) s += '(';
    switch (n.k) {
        case K::Num: {
            char buf[40];
            std::snprintf(buf, sizeof buf, "%.17g", n.num);
            if (n.num < 0.0)
                s += std::string("(") + buf + ")";
            else
                s += buf;
            break;
        }
        case K::Sym: s += var_name(static_cast<Var>(n.idx)); break;
        case K::Par: s += n.name; break;
        case K::Neg:
            s += '-';
            print(*n.l, s, 4);
            break;
        case K::Sin:
        case K::Cos:
        case K::Exp:
        case K::Sqrt: {
            static const char* fn[] = {"sin", "cos", "exp", "sqrt"};
            s += fn[static_cast<int>(n.k) - static_cast<int>(K::Sin)];
            s += '(';
            print(*n.l, s, 0);
            s += ')';
            break;
        }
        case K::Pow:
            print(*n.l, s, 5);
            s += '^' + std::to_string(n.idx);
            break;
        default: {
            static const char ops[] = {'+', '-', '*', '/'};
            print(*n.l, s, p);
            s += ops[static_cast<int>(n.k) - static_cast<int>(K::Add)];
            const bool tight = n.k == K::Sub || n.k == K::Div;
            print(*n.r, s, tight ? p + 1 : p);
        }
    }
    if (p < outer) s += ')';
}

}  // namespace
}  // namespace detail

using detail::K;
using detail::Node;
using detail::NodePtr;

Expr::Expr() : node_(detail::leaf_num(0.0)) {}
Expr::Expr(double c) : node_(detail::leaf_num(c)) {}

Expr Expr::variable(Var v) {
    auto n = std::make_shared<Node>();
    n->k = K::Sym;
    n->idx = static_cast<int>(v);
    return Expr(NodePtr(n));
}

Expr Expr::parameter(const std::string& name) {
    auto n = std::make_shared<Node>();
    n->k = K::Par;
    n->name = name;
    return Expr(NodePtr(n));
}

double Expr::eval(const EvalEnv& env) const { return detail::eval(*node_, env); }
Expr Expr::diff(Var v) const { return Expr(detail::derive(node_, static_cast<int>(v))); }

Expr Expr::subst(const std::array<std::optional<Expr>, 4>& map) const {
    return Expr(detail::rebuild(node_, [&](const NodePtr& leaf) -> NodePtr {
        if (leaf->k == K::Sym && map[leaf->idx]) return map[leaf->idx]->node();
        return leaf;
    }));
}

Expr Expr::simplified() const {
    return Expr(detail::rebuild(node_, [](const NodePtr& leaf) { return leaf; }));
}

std::string Expr::str() const {
    std::string s;
    detail::print(*node_, s, 0);
    return s;
}

bool Expr::is_constant(double* value) const {
    if (node_->k != K::Num) return false;
    if (value) *value = node_->num;
    return true;
}

bool Expr::depends_on(Var v) const { return detail::uses(*node_, static_cast<int>(v)); }

std::set<std::string> Expr::parameters() const {
    std::set<std::string> out;
    detail::params_of(*node_, out);
    return out;
}

Expr operator+(const Expr& a, const Expr& b) { return Expr(detail::mk_binary(K::Add, a.node(), b.node())); }
Expr operator-(const Expr& a, const Expr& b) { return Expr(detail::mk_binary(K::Sub, a.node(), b.node())); }
Expr operator*(const Expr& a, const Expr& b) { return Expr(detail::mk_binary(K::Mul, a.node(), b.node())); }
Expr operator/(const Expr& a, const Expr& b) { return Expr(detail::mk_binary(K::Div, a.node(), b.node())); }
Expr operator-(const Expr& a) { return Expr(detail::mk_unary(K::Neg, a.node())); }
Expr pow(const Expr& a, int n) { return Expr(detail::mk_pow(a.node(), n)); }
Expr sin(const Expr& a) { return Expr(detail::mk_unary(K::Sin, a.node())); }
Expr cos(const Expr& a) { return Expr(detail::mk_unary(K::Cos, a.node())); }
Expr exp(const Expr& a) { return Expr(detail::mk_unary(K::Exp, a.node())); }
Expr sqrt(const Expr& a) { return Expr(detail::mk_unary(K::Sqrt, a.node())); }

// ------------------------------------------------------------------ parser --
// Recursive descent over:  sum := prod (('+'|'-') prod)* ; prod := signed (('*'|'/') signed)* ;
// signed := ('-'|'+') signed | power ; power := atom ('^' uint)? ;
// atom := '(' sum ')' | number | x0|x1|y0|y1 | sin|cos|exp|sqrt '(' sum ')' | parameter
namespace {

class Reader {
public:
    Reader(const std::string& t, const std::set<std::string>& p) : s_(t), params_(p) {}

    Expr run() {
        Expr e = sum();
        if (!at_end()) error("unexpected trailing input");
        return e;
    }

private:
    const std::string& s_;
    const std::set<std::string>& params_;
    std::size_t i_ = 0;

    [[noreturn]] void error(const std::string& m) { throw ParseError(m, i_); }
    void ws() {
        while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
    }
    bool at_end() {
        ws();
        return i_ >= s_.size();
    }
    bool take(char c) {
        ws();
        if (i_ < s_.size() && s_[i_] == c) {
            ++i_;
            return true;
        }
        return false;
    }

    Expr sum() {
        Expr acc = prod();
        for (;;) {
            if (take('+'))
                acc = acc + prod();
            else if (take('-'))
                acc = acc - prod();
            else
                return acc;
        }
    }
    Expr prod() {
        Expr acc = sign();
        for (;;) {
            if (take('*'))
                acc = acc * sign();
            else if (take('/'))
                acc = acc / sign();
            else
                return acc;
        }
    }
    Expr sign() {
        if (take('-')) return -sign();
        if (take('+')) return sign();
        Expr base = atom();
        if (!take('^')) return base;
        ws();
        const std::size_t start = i_;
        int e = 0;
        while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) e = e * 10 + (s_[i_++] - '0');
        if (i_ == start) error("expected non-negative integer exponent after '^'");
        return pow(base, e);
    }
    Expr atom() {
        ws();
        if (i_ >= s_.size()) error("unexpected end of expression");
        const char c = s_[i_];
        if (c == '(') {
            ++i_;
            Expr e = sum();
            if (!take(')')) error("expected ')'");
            return e;
        }
        if (std::isdigit(static_cast<unsigned char>(c)) || c == '.') return number();
        if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') return word();
        error(std::string("unexpected character '") + c + "'");
    }
    Expr number() {
        const std::size_t start = i_;
        while (i_ < s_.size() && (std::isdigit(static_cast<unsigned char>(s_[i_])) || s_[i_] == '.')) ++i_;
        if (i_ < s_.size() && (s_[i_] == 'e' || s_[i_] == 'E')) {
            std::size_t j = i_ + 1;
            if (j < s_.size() && (s_[j] == '+' || s_[j] == '-')) ++j;
            if (j < s_.size() && std::isdigit(static_cast<unsigned char>(s_[j]))) {
                i_ = j;
                while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) ++i_;
            }
        }
        const std::string tok = s_.substr(start, i_ - start);
        char* end = nullptr;
        const double v = std::strtod(tok.c_str(), &end);
        if (end != tok.c_str() + tok.size()) {
            i_ = start;
            error("malformed number '" + tok + "'");
        }
        return Expr(v);
    }
    Expr word() {
        const std::size_t start = i_;
        while (i_ < s_.size() && (std::isalnum(static_cast<unsigned char>(s_[i_])) || s_[i_] == '_')) ++i_;
        const std::string w = s_.substr(start, i_ - start);
        static const char* vars[4] = {"x0", "x1", "y0", "y1"};
        for (int k = 0; k < 4; ++k)
            if (w == vars[k]) return Expr::variable(static_cast<Var>(k));
        if (w == "sin" || w == "cos" || w == "exp" || w == "sqrt") {
            if (!take('(')) error("expected '(' after function '" + w + "'");
            Expr arg = sum();
            if (!take(')')) error("expected ')'");
            if (w == "sin") return sin(arg);
            if (w == "cos") return cos(arg);
            if (w == "exp") return exp(arg);
            return sqrt(arg);
        }
        if (params_.count(w)) return Expr::parameter(w);
        i_ = start;
        error("unknown identifier '" + w + "'");
    }
};

}  // namespace

Expr parse(const std::string& text, const std::set<std::string>& params) {
    return Reader(text, params).run();
}

// ------------------------------------------------------------------- tape ---
CompiledExpr::CompiledExpr() = default;

CompiledExpr::CompiledExpr(const Expr& e, const ParamMap& params) {
    double c = 0.0;
    zero_ = e.is_constant(&c) && c == 0.0;
    if (!zero_) emit(*e.node(), params, 1);
}

void CompiledExpr::emit(const Node& n, const ParamMap& params, int depth) {
    if (depth > max_stack_) max_stack_ = depth;
    auto push = [&](int op, int arg, double v) {
        op_.push_back(op);
        arg_.push_back(arg);
        val_.push_back(v);
    };
    switch (n.k) {
        case K::Num: push(TS_OP_PUSH_CONST, 0, n.num); return;
        case K::Sym: push(TS_OP_PUSH_VAR, n.idx, 0.0); return;
        case K::Par: {
            auto it = params.find(n.name);
            if (it == params.end()) throw EvalError("unbound parameter '" + n.name + "'");
            push(TS_OP_PUSH_CONST, 0, it->second);
            return;
        }
        case K::Pow:
            emit(*n.l, params, depth);
            push(TS_OP_POW, n.idx, 0.0);
            return;
        case K::Neg:
        case K::Sin:
        case K::Cos:
        case K::Exp:
        case K::Sqrt: {
            emit(*n.l, params, depth);
            const int op = n.k == K::Neg   ? TS_OP_NEG
                           : n.k == K::Sin ? TS_OP_SIN
                           : n.k == K::Cos ? TS_OP_COS
                           : n.k == K::Exp ? TS_OP_EXP
                                           : TS_OP_SQRT;
            push(op, 0, 0.0);
            return;
        }
        default: {
            emit(*n.l, params, depth);
            emit(*n.r, params, depth + 1);
            const int op = n.k == K::Add   ? TS_OP_ADD
                           : n.k == K::Sub ? TS_OP_SUB
                           : n.k == K::Mul ? TS_OP_MUL
                                           : TS_OP_DIV;
            push(op, 0, 0.0);
        }
    }
}

double CompiledExpr::operator()(const std::array<double, 4>& x) const {
    if (zero_) return 0.0;
    std::vector<double> st(max_stack_ + 1);
    int t = -1;
    for (std::size_t k = 0; k < op_.size(); ++k) {
        switch (op_[k]) {
            case TS_OP_PUSH_CONST: st[++t] = val_[k]; break;
            case TS_OP_PUSH_VAR: st[++t] = x[arg_[k]]; break;
            case TS_OP_NEG: st[t] = -st[t]; break;
            case TS_OP_SIN: st[t] = std::sin(st[t]); break;
            case TS_OP_COS: st[t] = std::cos(st[t]); break;
            case TS_OP_EXP: st[t] = std::exp(st[t]); break;
            case TS_OP_SQRT:
                if (st[t] < 0.0) throw EvalError("sqrt of negative value");
                st[t] = std::sqrt(st[t]);
                break;
            case TS_OP_POW: st[t] = detail::ipow(st[t], arg_[k]); break;
            case TS_OP_ADD: --t; st[t] += st[t + 1]; break;
            case TS_OP_SUB: --t; st[t] -= st[t + 1]; break;
            case TS_OP_MUL: --t; st[t] *= st[t + 1]; break;
            case TS_OP_DIV:
                --t;
                if (st[t + 1] == 0.0) throw EvalError("division by zero");
                st[t] /= st[t + 1];
                break;
        }
    }
    return st[0];
}

double CompiledExpr::operator()(double x0, double x1, double y0, double y1) const {
    return (*this)(std::array<double, 4>{x0, x1, y0, y1});
}

ts_tape CompiledExpr::tape() const {
    ts_tape t{};
    if (zero_) return t;
    t.n = static_cast<int32_t>(op_.size());
    t.max_stack = max_stack_;
    t.op = op_.data();
    t.arg = arg_.data();
    t.val = val_.data();
    return t;
}

}  // namespace twoscale
