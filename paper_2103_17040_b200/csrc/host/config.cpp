// INI front-end (see include/twoscale/config.hpp) and the ts_ctx_create_ini entry
// point.  Grammar, defaults, required keys and messages follow the reference's
// config.cpp:126-266 and problem.cpp:30-66.
#include "twoscale/config.hpp"

#include <algorithm>
#include <cctype>
#include <cstdlib>
#include <fstream>
#include <map>
#include <set>
#include <sstream>

#include "twoscale/assembly.hpp"
#include "../internal.h"

namespace twoscale {

namespace {

using Section = std::map<std::string, std::string>;
using Ini = std::map<std::string, Section>;

std::string strip(const std::string& s) {
    std::size_t b = 0, e = s.size();
    while (b < e && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
    while (e > b && std::isspace(static_cast<unsigned char>(s[e - 1]))) --e;
    return s.substr(b, e - b);
}

bool as_number(const std::string& s, double* out) {
    if (s.empty()) return false;
    char* end = nullptr;
    const double v = std::strtod(s.c_str(), &end);
    if (end != s.c_str() + s.size()) return false;
    if (out) *out = v;
    return true;
}

Ini read_ini(const std::string& text) {
    Ini ini;
    std::istringstream in(text);
    std::string line, current;
    for (int no = 1; std::getline(in, line); ++no) {
        const std::size_t hash = line.find_first_of("#;");
        if (hash != std::string::npos) line.erase(hash);
        line = strip(line);
        if (line.empty()) continue;
        if (line[0] == '[') {
            if (line.back() != ']') throw ConfigError("line " + std::to_string(no) + ": malformed section header");
            current = strip(line.substr(1, line.size() - 2));
            ini[current];
            continue;
        }
        const std::size_t eq = line.find('=');
        if (eq == std::string::npos) throw ConfigError("line " + std::to_string(no) + ": expected key = value");
        if (current.empty()) throw ConfigError("line " + std::to_string(no) + ": key outside any section");
        ini[current][strip(line.substr(0, eq))] = strip(line.substr(eq + 1));
    }
    return ini;
}

class Reader {
public:
    Reader(const Ini& ini, const std::string& name) : name_(name) {
        auto it = ini.find(name);
        kv_ = it == ini.end() ? nullptr : &it->second;
    }
    bool has(const std::string& k) const { return kv_ && kv_->count(k); }
    const std::string* raw(const std::string& k) {
        used_.insert(k);
        if (!kv_) return nullptr;
        auto it = kv_->find(k);
        return it == kv_->end() ? nullptr : &it->second;
    }
    double num(const std::string& k, double dflt) {
        const std::string* v = raw(k);
        if (!v) return dflt;
        double out;
        if (!as_number(*v, &out)) throw ConfigError("[" + name_ + "] " + k + ": expected a number, got '" + *v + "'");
        return out;
    }
    int integer(const std::string& k, int dflt) {
        const double v = num(k, dflt);
        if (v != static_cast<int>(v)) throw ConfigError("[" + name_ + "] " + k + ": expected an integer");
        return static_cast<int>(v);
    }
    std::string text(const std::string& k, const std::string& dflt) {
        const std::string* v = raw(k);
        return v ? *v : dflt;
    }
    void no_leftovers() const {
        if (!kv_) return;
        for (const auto& kv : *kv_)
            if (!used_.count(kv.first)) throw ConfigError("[" + name_ + "] unknown key '" + kv.first + "'");
    }
    const Section* section() const { return kv_; }
    bool used(const std::string& k) const { return used_.count(k) != 0; }

private:
    std::string name_;
    const Section* kv_;
    std::set<std::string> used_;
};

Side side_of(const std::string& s, const std::string& where) {
    static const char* names[4] = {"left", "right", "bottom", "top"};
    for (int k = 0; k < 4; ++k)
        if (s == names[k]) return static_cast<Side>(k);
    throw ConfigError(where + ": unknown side '" + s + "'");
}

std::vector<Side> sides_of(const std::string& list, const std::string& where) {
    std::vector<Side> out;
    std::istringstream in(list);
    std::string tok;
    while (std::getline(in, tok, ',')) {
        tok = strip(tok);
        if (!tok.empty()) out.push_back(side_of(tok, where));
    }
    return out;
}

}  // namespace

Config parse_config(const std::string& text) {
    const Ini ini = read_ini(text);
    static const std::set<std::string> known = {"macro", "micro", "parameters", "solver", "mms", "output"};
    for (const auto& s : ini)
        if (!known.count(s.first)) throw ConfigError("unknown section [" + s.first + "]");
    static const std::pair<const char*, const char*> required[] = {
        {"macro", "n0"},          {"macro", "n1"},          {"micro", "n0"},          {"micro", "n1"},
        {"micro", "zeta0"},       {"micro", "zeta1"},       {"parameters", "kappa1"}, {"parameters", "kappa2"},
        {"parameters", "kappa3"}, {"parameters", "kappa4"}, {"parameters", "Dv"},     {"parameters", "Dw"}};
    std::string missing;
    for (const auto& [sec, key] : required) {
        auto it = ini.find(sec);
        if (it == ini.end() || !it->second.count(key)) missing += std::string(" ") + sec + "." + key;
    }
    if (!missing.empty()) throw ConfigError("missing required keys:" + missing);

    Config cfg;
    Reader mac(ini, "macro");
    cfg.macro_domain.lo = {mac.num("lo0", -1.0), mac.num("lo1", -1.0)};
    cfg.macro_domain.hi = {mac.num("hi0", 1.0), mac.num("hi1", 1.0)};
    cfg.macro_n0 = mac.integer("n0", 8);
    cfg.macro_n1 = mac.integer("n1", 8);
    cfg.roles.macro.fill(MacroBC::Neumann);
    for (Side s : sides_of(mac.text("dirichlet", "left"), "[macro] dirichlet"))
        cfg.roles.macro[static_cast<int>(s)] = MacroBC::Dirichlet;
    mac.no_leftovers();

    Reader mic(ini, "micro");
    cfg.micro_domain.lo = {mic.num("lo0", -1.0), mic.num("lo1", -1.0)};
    cfg.micro_domain.hi = {mic.num("hi0", 1.0), mic.num("hi1", 1.0)};
    cfg.micro_n0 = mic.integer("n0", 8);
    cfg.micro_n1 = mic.integer("n1", 8);
    cfg.zeta0 = mic.text("zeta0", "y0");
    cfg.zeta1 = mic.text("zeta1", "y1");
    {
        const bool explicit_roles = mic.has("gamma_i") || mic.has("gamma_o") || mic.has("gamma_n");
        int count[4] = {0, 0, 0, 0};
        const std::pair<const char*, MicroRole> groups[3] = {
            {"gamma_i", MicroRole::GammaI}, {"gamma_o", MicroRole::GammaO}, {"gamma_n", MicroRole::GammaN}};
        const char* dflt[3] = {"left", "right", "bottom,top"};
        for (int g = 0; g < 3; ++g)
            for (Side s : sides_of(mic.text(groups[g].first, dflt[g]), std::string("[micro] ") + groups[g].first)) {
                cfg.roles.micro[static_cast<int>(s)] = groups[g].second;
                ++count[static_cast<int>(s)];
            }
        if (explicit_roles)
            for (int s = 0; s < 4; ++s)
                if (count[s] != 1)
                    throw ConfigError(std::string("[micro] side '") + side_name(static_cast<Side>(s)) +
                                      "' must be assigned exactly one role");
    }
    mic.no_leftovers();

    Reader par(ini, "parameters");
    cfg.kappa1 = par.num("kappa1", 1.0);
    cfg.kappa2 = par.num("kappa2", 1.0);
    cfg.kappa3 = par.num("kappa3", 1.0);
    cfg.kappa4 = par.num("kappa4", 1.0);
    cfg.Dv = par.num("Dv", 1.0);
    cfg.dw = par.text("Dw", "1");
    cfg.fu = par.text("fu", "0");
    cfg.fv = par.text("fv", "0");
    cfg.fw = par.text("fw", "0");
    cfg.u0 = par.text("u0", "0");
    if (const Section* kv = par.section())
        for (const auto& [key, value] : *kv) {
            if (par.used(key)) continue;
            double v;
            if (!as_number(value, &v))
                throw ConfigError("[parameters] " + key + ": extra keys must be numeric parameter bindings");
            cfg.params[key] = v;
        }
    cfg.params["kappa1"] = cfg.kappa1;
    cfg.params["kappa2"] = cfg.kappa2;
    cfg.params["kappa3"] = cfg.kappa3;
    cfg.params["kappa4"] = cfg.kappa4;
    cfg.params["Dv"] = cfg.Dv;
    {
        double v;
        if (as_number(cfg.dw, &v)) cfg.params["Dw"] = v;
    }

    Reader sol(ini, "solver");
    cfg.inner_tol = sol.num("inner_tol", 1e-10);
    cfg.inner_maxit = sol.integer("inner_maxit", 20000);
    cfg.outer_tol = sol.num("outer_tol", 1e-8);
    cfg.max_outer = sol.integer("max_outer", 100);
    cfg.bounds.lo = sol.num("det_lo", 1e-6);
    cfg.bounds.hi = sol.num("det_hi", 1e6);
    sol.no_leftovers();

    if (ini.count("mms")) {
        Reader mms(ini, "mms");
        const std::string *u = mms.raw("u"), *v = mms.raw("v"), *w = mms.raw("w");
        if (!u || !v || !w) throw ConfigError("[mms] requires keys u, v and w");
        cfg.has_mms = true;
        cfg.mms_u = *u;
        cfg.mms_v = *v;
        cfg.mms_w = *w;
        mms.no_leftovers();
    }
    Reader out(ini, "output");
    cfg.micro_viz_scale = out.num("micro_viz_scale", 0.1);
    out.no_leftovers();
    if (cfg.macro_n0 < 1 || cfg.macro_n1 < 1 || cfg.micro_n0 < 1 || cfg.micro_n1 < 1)
        throw ConfigError("grid sizes must be >= 1");
    return cfg;
}

Config load_config(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw ConfigError("cannot open config file '" + path + "'");
    std::stringstream ss;
    ss << in.rdbuf();
    return parse_config(ss.str());
}

namespace {
Expr field(const std::string& text, const std::set<std::string>& names, const std::string& where, bool micro_vars) {
    Expr e;
    try {
        e = parse(text, names);
    } catch (const ParseError& err) {
        throw ConfigError(where + ": " + err.what());
    }
    if (!micro_vars && (e.depends_on(Var::y0) || e.depends_on(Var::y1)))
        throw ConfigError(where + ": expression must not depend on y0/y1");
    return e;
}
}  // namespace

ProblemSetup make_problem(const Config& cfg) {
    std::set<std::string> names;
    for (const auto& kv : cfg.params) names.insert(kv.first);
    ProblemData d;
    d.kappa1 = cfg.kappa1;
    d.kappa2 = cfg.kappa2;
    d.kappa3 = cfg.kappa3;
    d.kappa4 = cfg.kappa4;
    d.Dv = cfg.Dv;
    d.Dw = field(cfg.dw, names, "[parameters] Dw", false);
    d.fu = field(cfg.fu, names, "[parameters] fu", false);
    d.fv = field(cfg.fv, names, "[parameters] fv", true);
    d.fw = field(cfg.fw, names, "[parameters] fw", false);
    d.u0 = field(cfg.u0, names, "[parameters] u0", false);
    d.diffeo = Diffeo::from_map(
        {field(cfg.zeta0, names, "[micro] zeta0", true), field(cfg.zeta1, names, "[micro] zeta1", true)});
    d.roles = cfg.roles;
    d.bounds = cfg.bounds;
    d.params = cfg.params;
    ProblemSetup setup{d, Grid(cfg.macro_domain, cfg.macro_n0, cfg.macro_n1),
                       Grid(cfg.micro_domain, cfg.micro_n0, cfg.micro_n1), ManufacturedCase{}};
    if (cfg.has_mms) {
        setup.mms.u = field(cfg.mms_u, names, "[mms] u", false);
        setup.mms.v = field(cfg.mms_v, names, "[mms] v", true);
        setup.mms.w = field(cfg.mms_w, names, "[mms] w", false);
        setup.mms.base = setup.data;
        setup.mms.macro_domain = cfg.macro_domain;
        setup.mms.micro_domain = cfg.micro_domain;
    }
    return setup;
}

}  // namespace twoscale

extern "C" int32_t ts_ctx_create_ini(const char* ini_text, const ts_ext_desc* ext, ts_ctx** out) {
    using namespace twoscale;
    if (!out || !ini_text) return TS_ERR_INVALID;
    *out = nullptr;
    try {
        const Config cfg = parse_config(ini_text);
        ProblemSetup setup = make_problem(cfg);
        if (ext) {
            setup.data.D = {ext->D[0], ext->D[1], ext->D[2], ext->D[3]};
            setup.data.reaction_kind = ext->reaction_kind;
            for (int k = 0; k < 5; ++k) setup.data.reaction[k] = ext->reaction[k];
            auto& X = setup.data;
            X.micro_dim = ext->micro_dim == 3 ? 3 : 2;
            X.micro_order = ext->micro_order == 2 ? 2 : 1;
            X.micro_n2 = ext->micro_n2;
            X.micro_lo2 = ext->micro_lo2;
            X.micro_hi2 = ext->micro_hi2;
            for (int k = 0; k < 9; ++k) X.D3[k] = ext->D3[k];
            for (int k = 0; k < 2; ++k)
                X.micro_role3[k] = ext->micro_role3[k] == TS_GAMMA_I   ? MicroRole::GammaI
                                   : ext->micro_role3[k] == TS_GAMMA_O ? MicroRole::GammaO
                                                                       : MicroRole::GammaN;
            X.reaction_cz = ext->reaction_cz;
            X.force_generic = ext->force_generic != 0;
            if (ext->map_kind == TS_MAP_AFFINE_BUBBLE_TABLE || ext->map_kind == TS_MAP_FOURIER_TABLE) {
                if (!ext->A_table) throw std::invalid_argument("tabulated map without A_table");
                const std::size_t stride = ext->map_kind == TS_MAP_FOURIER_TABLE ? 16 : X.micro_dim == 3 ? 9 : 4;
                X.table.kind = ext->map_kind;
                X.table.A.assign(ext->A_table, ext->A_table + stride * static_cast<std::size_t>(setup.macro.node_count()));
                X.table.s_kind = ext->s_kind;
                X.table.amp = ext->amp;
            }
        }
        LoweredProblem L = lower_problem(setup.data, setup.macro, setup.micro);
        const int rc = ts_ctx_create(&L.desc, out);
        if (rc != TS_OK) return rc;
        const ts_solve_opts o{cfg.inner_tol, cfg.inner_maxit, cfg.outer_tol, cfg.max_outer};
        tsb_set_default_opts(*out, &o);
        return TS_OK;
    } catch (const ConfigError& e) {
        return ts_set_error_for_front_end(TS_ERR_CONFIG, e.what());
    } catch (const ParseError& e) {
        return ts_set_error_for_front_end(TS_ERR_EXPR, e.what());
    } catch (const EvalError& e) {
        return ts_set_error_for_front_end(TS_ERR_EXPR, e.what());
    } catch (const std::exception& e) {
        return ts_set_error_for_front_end(TS_ERR_INVALID, e.what());
    }
}
