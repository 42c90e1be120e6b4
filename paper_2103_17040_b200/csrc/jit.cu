// Compiled tapes: the expression tapes the host front-end emits
// (CompiledExpr, src/expr.cpp:617-701) become straight-line device functions, compiled at
// run time with NVRTC for sm_100a into the kernels that evaluate them per quadrature point.
// The interpreter (device_common.cuh tape_eval) keeps its stack in local memory and
// dispatches on every instruction; a compiled tape is a chain of register operations.
//
// Bitwise contract: each tape instruction becomes the same IEEE operation the interpreter
// performs (__dadd_rn / __dsub_rn / __dmul_rn / __ddiv_rn are never contracted or
// reassociated; sin / cos / exp / sqrt are the same libdevice routines; Pow is the same
// repeated multiplication), and the kernel around the tapes is the same source
// (errnorm_kernel.cuh) compiled with the same default flags — so a compiled kernel returns
// the interpreter's bits (tests/test_gpu_mms.py checks this).
//
// NVRTC is loaded with dlopen on first use (no link-time dependency); if it is missing or
// a compile fails, the interpreted kernel runs instead and ts_jit_status() says why.
// Compiled kernels are cached per process by source text.
#include <dlfcn.h>

#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "jit.h"
#include "mms.h"

namespace tsb {

namespace {

// Headers the run-time compiled sources include, embedded at build time (Makefile).
struct EmbeddedHeader {
    const char* name;
    const char* text;
};
const EmbeddedHeader kHeaders[] = {
#include "jit_headers.inc"
};

// ---- NVRTC, resolved at run time ----
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;
struct Nvrtc {
    nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int, const char* const*, const char* const*);
    nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*);
    nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*);
    nvrtcResult_t (*log)(nvrtcProgram_t, char*);
    nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*);
    nvrtcResult_t (*cubin)(nvrtcProgram_t, char*);
    nvrtcResult_t (*destroy)(nvrtcProgram_t*);
    bool ok = false;
    std::string why;
};

const Nvrtc& nvrtc() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12",
                               "/usr/local/cuda/lib64/libnvrtc.so"};
        void* h = nullptr;
        for (const char* nm : names)
            if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
        if (!h) {
            n.why = "libnvrtc not found";
            return;
        }
        auto sym = [&](const char* s) { return dlsym(h, s); };
        n.create = reinterpret_cast<decltype(n.create)>(sym("nvrtcCreateProgram"));
        n.compile = reinterpret_cast<decltype(n.compile)>(sym("nvrtcCompileProgram"));
        n.log_size = reinterpret_cast<decltype(n.log_size)>(sym("nvrtcGetProgramLogSize"));
        n.log = reinterpret_cast<decltype(n.log)>(sym("nvrtcGetProgramLog"));
        n.cubin_size = reinterpret_cast<decltype(n.cubin_size)>(sym("nvrtcGetCUBINSize"));
        n.cubin = reinterpret_cast<decltype(n.cubin)>(sym("nvrtcGetCUBIN"));
        n.destroy = reinterpret_cast<decltype(n.destroy)>(sym("nvrtcDestroyProgram"));
        n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.destroy;
        if (!n.ok) n.why = "libnvrtc lacks an entry point";
    });
    return n;
}

std::mutex g_mu;
std::map<std::string, cudaKernel_t> g_cache;  // source -> kernel (per process; the library owns the modules)
std::string g_status = "not used";
int g_compiles = 0, g_jit_launches = 0;

std::string hex_double(double v) {
    unsigned long long b;
    std::memcpy(&b, &v, sizeof b);
    char buf[48];
    std::snprintf(buf, sizeof buf, "__longlong_as_double(0x%016llxULL)", b);
    return buf;
}

}  // namespace

// One tape as a device function double name(x0, x1, y0, y1): the postfix program run on a
// compile-time stack, each push a new SSA value (src/expr.cpp:663-701 semantics).
std::string tape_function(const ts_tape& t, const std::string& name) {
    std::string s = "__device__ __forceinline__ double " + name +
                    "(double x0, double x1, double y0, double y1) {\n";
    if (t.n == 0) return s + "    return 0.0;\n}\n";
    std::vector<std::string> st;
    int next = 0;
    auto fresh = [&](const std::string& expr) {
        const std::string v = "v" + std::to_string(next++);
        s += "    const double " + v + " = " + expr + ";\n";
        return v;
    };
    static const char* vars[4] = {"x0", "x1", "y0", "y1"};
    for (int k = 0; k < t.n; ++k) {
        switch (t.op[k]) {
            case TS_OP_PUSH_CONST: st.push_back(fresh(hex_double(t.val[k]))); break;
            case TS_OP_PUSH_VAR: st.push_back(vars[t.arg[k] >= 0 && t.arg[k] < 4 ? t.arg[k] : 3]); break;
            case TS_OP_NEG: st.back() = fresh("-" + st.back()); break;
            case TS_OP_SIN: st.back() = fresh("sin(" + st.back() + ")"); break;
            case TS_OP_COS: st.back() = fresh("cos(" + st.back() + ")"); break;
            case TS_OP_EXP: st.back() = fresh("exp(" + st.back() + ")"); break;
            case TS_OP_SQRT: st.back() = fresh("sqrt(" + st.back() + ")"); break;
            case TS_OP_POW: {
                std::string r = fresh("1.0");
                for (int i = 0; i < t.arg[k]; ++i) r = fresh("__dmul_rn(" + r + ", " + st.back() + ")");
                st.back() = r;
                break;
            }
            case TS_OP_ADD: case TS_OP_SUB: case TS_OP_MUL: case TS_OP_DIV: {
                const std::string b = st.back();
                st.pop_back();
                const char* fn = t.op[k] == TS_OP_ADD ? "__dadd_rn" : t.op[k] == TS_OP_SUB ? "__dsub_rn"
                                 : t.op[k] == TS_OP_MUL ? "__dmul_rn" : "__ddiv_rn";
                st.back() = fresh(std::string(fn) + "(" + st.back() + ", " + b + ")");
                break;
            }
            default: break;
        }
    }
    return s + "    return " + (st.empty() ? std::string("0.0") : st.front()) + ";\n}\n";
}

namespace {

// Compile (or fetch) `source`'s kernel `entry`.  Returns nullptr and sets g_status on failure.
cudaKernel_t compiled(const std::string& source, const char* entry) {
    std::lock_guard<std::mutex> lock(g_mu);
    auto it = g_cache.find(source);
    if (it != g_cache.end()) return it->second;
    const Nvrtc& n = nvrtc();
    if (!n.ok) {
        g_status = "interpreter (" + n.why + ")";
        return nullptr;
    }
    std::vector<const char*> hn, ht;
    for (const auto& h : kHeaders) {
        hn.push_back(h.name);
        ht.push_back(h.text);
    }
    nvrtcProgram_t prog = nullptr;
    if (n.create(&prog, source.c_str(), "ts_jit.cu", (int)hn.size(), ht.data(), hn.data()) != 0) {
        g_status = "interpreter (nvrtcCreateProgram failed)";
        return nullptr;
    }
    const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo"};
    const int rc = n.compile(prog, 3, opts);
    std::vector<char> cubin;
    if (rc == 0) {
        size_t sz = 0;
        n.cubin_size(prog, &sz);
        cubin.resize(sz);
        n.cubin(prog, cubin.data());
    } else {
        size_t ls = 0;
        n.log_size(prog, &ls);
        std::string log(ls, '\0');
        n.log(prog, &log[0]);
        g_status = "interpreter (NVRTC compile failed: " + log.substr(0, 400) + ")";
    }
    n.destroy(&prog);
    if (rc != 0) return nullptr;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t k = nullptr;
    if (cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
        cudaLibraryGetKernel(&k, lib, entry) != cudaSuccess) {
        cudaGetLastError();
        g_status = "interpreter (loading the compiled module failed)";
        return nullptr;
    }
    ++g_compiles;
    g_cache.emplace(source, k);
    return k;
}

bool jit_enabled() {
    const char* e = std::getenv("TS_JIT");
    return !(e && e[0] == '0');
}

}  // namespace

bool launch_error_norms_jit(const ErrNormArgs& a, const ts_tape* tapes, double* partials, cudaStream_t s) {
    if (!jit_enabled()) {
        std::lock_guard<std::mutex> lock(g_mu);
        g_status = "interpreter (TS_JIT=0)";
        return false;
    }
    std::string src = "#include \"errnorm_kernel.cuh\"\nnamespace tsb {\nnamespace jit {\n";
    for (int k = 0; k < 12; ++k) src += tape_function(tapes[k], "tape" + std::to_string(k));
    src += "struct Tapes {\n    __device__ __forceinline__ double operator()(int k, double x0, double x1, double y0, "
           "double y1) const {\n        switch (k) {\n";
    for (int k = 0; k < 12; ++k)
        src += "            case " + std::to_string(k) + ": return tape" + std::to_string(k) + "(x0, x1, y0, y1);\n";
    src += "        }\n        return 0.0;\n    }\n};\n}  // namespace jit\n}  // namespace tsb\n"
           "extern \"C\" __global__ void __launch_bounds__(256) k_error_norms_jit(const tsb::ErrNormArgs a, "
           "double* partials) {\n    extern __shared__ double sm[];\n"
           "    tsb::error_norms_block(a, partials, sm, tsb::jit::Tapes{});\n}\n";
    cudaKernel_t k = compiled(src, "k_error_norms_jit");
    if (!k) return false;
    const size_t smem = error_norms_smem(a.micro);
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaKernelSetAttributeForDevice(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem, dev) !=
        cudaSuccess) {
        cudaGetLastError();
        std::lock_guard<std::mutex> lock(g_mu);
        g_status = "interpreter (shared-memory attribute refused)";
        return false;
    }
    ErrNormArgs args = a;
    void* params[] = {&args, &partials};
    if (cudaLaunchKernel(reinterpret_cast<const void*>(k), dim3(a.macro.cells()), dim3(256), params, smem, s) !=
        cudaSuccess) {
        cudaGetLastError();
        std::lock_guard<std::mutex> lock(g_mu);
        g_status = "interpreter (launch of the compiled kernel failed)";
        return false;
    }
    std::lock_guard<std::mutex> lock(g_mu);
    g_status = "compiled";
    ++g_jit_launches;
    return true;
}

std::string jit_status() {
    std::lock_guard<std::mutex> lock(g_mu);
    return g_status + " (compiles " + std::to_string(g_compiles) + ", launches " + std::to_string(g_jit_launches) + ")";
}

}  // namespace tsb
