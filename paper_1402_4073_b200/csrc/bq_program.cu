// JIT execution of the reference's straight-line BitPrograms on the GPU
// (reference circuits/programs.py).
//
// A BitProgram (programs.py:56-72) is a list of (opcode, dst, a, b) over slots;
// inputs occupy slots 0..arity-1.  The reference interprets it over whole
// bitmaps (`execute`, :163-193) or 256-word batches (`execute_horizontal`,
// :196-237).  Here it is turned into CUDA source -- one thread per 32-bit half word,
// every slot a 32-bit register variable -- compiled once with NVRTC for sm_100a
// and launched through the driver API.  Loads are coalesced across a warp
// (consecutive words of one input), so the program runs at HBM speed until its
// gate count makes it compute-bound.  Semantics match `execute`: missing
// trailing words read as zero, ONE is all-ones, NOT complements, and bits >= r
// of the result are cleared (the reference keeps every intermediate within r,
// which agrees with masking the result because every operation is bitwise).
//
// libnvrtc and libcuda are loaded lazily with dlopen, so libbq.so still loads
// (and its CPU-side functions work) on machines without a GPU driver.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "bq_internal.h"

namespace bq {

enum { OP_ZERO = 0, OP_ONE = 1, OP_AND = 2, OP_OR = 3, OP_XOR = 4, OP_ANDNOT = 5, OP_NOT = 6, OP_RECLAIM = 7 };  // programs.py:21-28

// ---- minimal dynamic bindings ---------------------------------------------
typedef int nvrtcResult_t;
typedef void *nvrtcProgram_t;
typedef int CUresult_t;
typedef void *CUmodule_t;
typedef void *CUfunction_t;

struct Jit {
    bool ok = false;
    std::string why;
    nvrtcResult_t (*nvrtcCreateProgram)(nvrtcProgram_t *, const char *, const char *, int, const char *const *,
                                        const char *const *);
    nvrtcResult_t (*nvrtcCompileProgram)(nvrtcProgram_t, int, const char *const *);
    nvrtcResult_t (*nvrtcGetProgramLogSize)(nvrtcProgram_t, size_t *);
    nvrtcResult_t (*nvrtcGetProgramLog)(nvrtcProgram_t, char *);
    nvrtcResult_t (*nvrtcGetCUBINSize)(nvrtcProgram_t, size_t *);
    nvrtcResult_t (*nvrtcGetCUBIN)(nvrtcProgram_t, char *);
    nvrtcResult_t (*nvrtcDestroyProgram)(nvrtcProgram_t *);
    CUresult_t (*cuModuleLoadData)(CUmodule_t *, const void *);
    CUresult_t (*cuModuleGetFunction)(CUfunction_t *, CUmodule_t, const char *);
    CUresult_t (*cuModuleUnload)(CUmodule_t);
    CUresult_t (*cuLaunchKernel)(CUfunction_t, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                                 void *, void **, void **);
};

static void *open_first(const char *const *names) {
    for (int i = 0; names[i]; ++i)
        if (void *h = dlopen(names[i], RTLD_NOW | RTLD_GLOBAL)) return h;
    return nullptr;
}

template <typename F>
static bool sym(void *h, const char *name, F &f) {
    f = reinterpret_cast<F>(dlsym(h, name));
    return f != nullptr;
}

static Jit &jit() {
    static Jit j;
    static std::once_flag once;
    std::call_once(once, [] {
        static const char *nv[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12", nullptr};
        static const char *cu[] = {"libcuda.so.1", "libcuda.so", nullptr};
        void *hn = open_first(nv);
        void *hc = open_first(cu);
        if (!hn) {
            j.why = "libnvrtc.so.12 not found";
            return;
        }
        if (!hc) {
            j.why = "libcuda.so.1 not found";
            return;
        }
        j.ok = sym(hn, "nvrtcCreateProgram", j.nvrtcCreateProgram) && sym(hn, "nvrtcCompileProgram", j.nvrtcCompileProgram) &&
               sym(hn, "nvrtcGetProgramLogSize", j.nvrtcGetProgramLogSize) &&
               sym(hn, "nvrtcGetProgramLog", j.nvrtcGetProgramLog) && sym(hn, "nvrtcGetCUBINSize", j.nvrtcGetCUBINSize) &&
               sym(hn, "nvrtcGetCUBIN", j.nvrtcGetCUBIN) && sym(hn, "nvrtcDestroyProgram", j.nvrtcDestroyProgram) &&
               sym(hc, "cuModuleLoadData", j.cuModuleLoadData) && sym(hc, "cuModuleGetFunction", j.cuModuleGetFunction) &&
               sym(hc, "cuModuleUnload", j.cuModuleUnload) && sym(hc, "cuLaunchKernel", j.cuLaunchKernel);
        if (!j.ok) j.why = "missing NVRTC / driver symbols";
    });
    return j;
}

// One thread per 32-bit half of an output word: every slot is a 32-bit register
// (the program is bitwise, so the halves are independent), which halves the
// registers per thread against 64-bit slots (SSum(64,32): 78 instead of 171) and
// triples the warps an SM can hold to overlap the loads with the gate network.
static std::string gen_source(const int32_t *ins, int n_ins, int arity, int n_slots, int result) {
    std::ostringstream o;
    o << "// generated from a bitquorum BitProgram: arity=" << arity << " slots=" << n_slots << " ops=" << n_ins << "\n"
      << "typedef unsigned long long u64;\n"
      << "typedef unsigned int u32;\n"
      << "extern \"C\" __global__ void __launch_bounds__(256) bq_prog(const u64 *const *ptrs, const u64 *lens,\n"
      << "    u64 nwords, u64 full_words, u64 last_mask, u64 *out, u64 *popcnt, u64 *last_nz) {\n"
      << "  u64 pc = 0, lnz = 0;\n"
      << "  for (u64 h = (u64)blockIdx.x * blockDim.x + threadIdx.x; h < 2 * nwords; h += (u64)gridDim.x * blockDim.x) {\n"
      << "    const u64 w = h >> 1;\n"
      << "    const bool full = w < full_words;\n";
    for (int i = 0; i < arity; ++i)
        o << "    u32 s" << i << " = (full || w < lens[" << i << "]) ? __ldg((const u32 *)ptrs[" << i << "] + h) : 0u;\n";
    if (n_slots > arity) {
        o << "    u32";
        for (int k = arity; k < n_slots; ++k) o << (k > arity ? ", " : " ") << "s" << k << " = 0u";
        o << ";\n";
    }
    for (int k = 0; k < n_ins; ++k) {
        const int op = ins[4 * k], d = ins[4 * k + 1], a = ins[4 * k + 2], b = ins[4 * k + 3];
        switch (op) {
            case OP_ZERO: o << "    s" << d << " = 0u;\n"; break;
            case OP_ONE: o << "    s" << d << " = ~0u;\n"; break;
            case OP_AND: o << "    s" << d << " = s" << a << " & s" << b << ";\n"; break;
            case OP_OR: o << "    s" << d << " = s" << a << " | s" << b << ";\n"; break;
            case OP_XOR: o << "    s" << d << " = s" << a << " ^ s" << b << ";\n"; break;
            case OP_ANDNOT: o << "    s" << d << " = s" << a << " & ~s" << b << ";\n"; break;
            case OP_NOT: o << "    s" << d << " = ~s" << a << ";\n"; break;
            default: break;  // reclaim: register allocation is the compiler's job
        }
    }
    o << "    u32 r = s" << result << ";\n"
      << "    if (w == nwords - 1) r &= (u32)(last_mask >> (32 * (h & 1)));\n"
      << "    ((u32 *)out)[h] = r;\n"
      << "    pc += __popc(r);\n"
      << "    if (r) lnz = w + 1;\n"
      << "  }\n"
      << "  for (int o = 16; o > 0; o >>= 1) {\n"
      << "    pc += __shfl_down_sync(0xffffffffu, pc, o);\n"
      << "    u64 t = __shfl_down_sync(0xffffffffu, lnz, o); lnz = t > lnz ? t : lnz;\n"
      << "  }\n"
      << "  if ((threadIdx.x & 31) == 0) {\n"
      << "    if (popcnt && pc) atomicAdd(popcnt, pc);\n"
      << "    if (last_nz && lnz) atomicMax(last_nz, lnz);\n"
      << "  }\n"
      << "}\n";
    return o.str();
}

}  // namespace bq

using namespace bq;

struct bq_program {
    int arity, n_slots, result_slot, n_ins;
    std::string source;
    std::vector<char> cubin;
    // the module is loaded into each device's primary context on first use there: a
    // function handle from one context cannot be launched in another
    std::map<int, std::pair<CUmodule_t, CUfunction_t>> per_device;
    std::mutex mu;
};

// The program's kernel in the current device's context (loaded on first use).
static int program_function(bq_program *p, CUfunction_t *fn) {
    int dev = 0;
    cudaError_t ce = cudaGetDevice(&dev);
    if (ce != cudaSuccess) return cuda_error(ce, "cudaGetDevice");
    std::lock_guard<std::mutex> g(p->mu);
    auto it = p->per_device.find(dev);
    if (it != p->per_device.end()) {
        *fn = it->second.second;
        return BQ_OK;
    }
    cudaFree(0);  // make sure the device's primary context is current for the driver API
    Jit &j = jit();
    CUmodule_t mod = nullptr;
    CUfunction_t f = nullptr;
    if (j.cuModuleLoadData(&mod, p->cubin.data()) != 0 || j.cuModuleGetFunction(&f, mod, "bq_prog") != 0) {
        if (mod) j.cuModuleUnload(mod);
        return set_error(BQ_ECUDA, "cuModuleLoadData/cuModuleGetFunction failed on device %d", dev);
    }
    p->per_device.emplace(dev, std::make_pair(mod, f));
    *fn = f;
    return BQ_OK;
}

// Layout of bq_query needed here (defined in bq_api.cu): the public accessor is enough.
extern "C" {

BQ_API int bq_program_compile(const int32_t *instr, int n_instr, int arity, int n_slots, int result_slot,
                              bq_program **out) {
    if (!out) return set_error(BQ_EINPUT, "out is NULL");
    *out = nullptr;
    if (arity < 1 || n_slots < arity || result_slot < 0 || result_slot >= n_slots || n_instr < 0 ||
        (n_instr && !instr))
        return set_error(BQ_EINPUT, "malformed program header");
    for (int k = 0; k < n_instr; ++k) {  // the checks loads_program implies (programs.py:276-321)
        const int op = instr[4 * k], d = instr[4 * k + 1], a = instr[4 * k + 2], b = instr[4 * k + 3];
        if (op < OP_ZERO || op > OP_RECLAIM) return set_error(BQ_EFORMAT, "unknown opcode %d", op);
        if (d < 0 || d >= n_slots) return set_error(BQ_EFORMAT, "instruction %d: slot %d out of range", k, d);
        const bool two = (op >= OP_AND && op <= OP_NOT), three = (op >= OP_AND && op <= OP_ANDNOT);
        if (two && (a < 0 || a >= n_slots)) return set_error(BQ_EFORMAT, "instruction %d: slot %d out of range", k, a);
        if (three && (b < 0 || b >= n_slots)) return set_error(BQ_EFORMAT, "instruction %d: slot %d out of range", k, b);
    }
    Jit &j = jit();
    if (!j.ok) return set_error(BQ_ECUDA, "program JIT unavailable: %s", j.why.c_str());
    cudaFree(0);  // make sure the primary context is current for the driver API
    bq_program *p = new bq_program();
    p->arity = arity;
    p->n_slots = n_slots;
    p->result_slot = result_slot;
    p->n_ins = n_instr;
    p->source = gen_source(instr, n_instr, arity, n_slots, result_slot);
    nvrtcProgram_t prog = nullptr;
    if (j.nvrtcCreateProgram(&prog, p->source.c_str(), "bq_prog.cu", 0, nullptr, nullptr) != 0) {
        delete p;
        return set_error(BQ_ECUDA, "nvrtcCreateProgram failed");
    }
    const char *opts[] = {"--gpu-architecture=sm_100a", "-default-device", "--std=c++17"};
    const int rc = j.nvrtcCompileProgram(prog, 3, opts);
    if (rc != 0) {
        size_t n = 0;
        j.nvrtcGetProgramLogSize(prog, &n);
        std::string log(n, '\0');
        if (n) j.nvrtcGetProgramLog(prog, &log[0]);
        j.nvrtcDestroyProgram(&prog);
        delete p;
        return set_error(BQ_ECUDA, "NVRTC compile failed: %.400s", log.c_str());
    }
    size_t n = 0;
    j.nvrtcGetCUBINSize(prog, &n);
    p->cubin.resize(n);
    j.nvrtcGetCUBIN(prog, p->cubin.data());
    j.nvrtcDestroyProgram(&prog);
    CUfunction_t fn = nullptr;  // load (and so validate) the module on the current device now
    if (int rc2 = program_function(p, &fn)) {
        delete p;
        return rc2;
    }
    *out = p;
    return BQ_OK;
}

BQ_API void bq_program_destroy(bq_program *p) {
    if (!p) return;
    if (jit().ok) {
        int prev = -1;
        cudaGetDevice(&prev);
        for (auto &kv : p->per_device) {  // unload in each module's own context
            cudaSetDevice(kv.first);
            cudaFree(0);
            jit().cuModuleUnload(kv.second.first);
        }
        if (prev >= 0) cudaSetDevice(prev);
    }
    delete p;
}

BQ_API int bq_program_source(const bq_program *p, char *buf, uint64_t cap, uint64_t *len) {
    if (!p) return set_error(BQ_EINPUT, "program is NULL");
    if (len) *len = p->source.size() + 1;
    if (buf && cap) {
        const size_t k = std::min<size_t>(cap - 1, p->source.size());
        memcpy(buf, p->source.data(), k);
        buf[k] = '\0';
    }
    return BQ_OK;
}

}  // extern "C"

namespace bq {
// implemented in bq_api.cu: the query's device tables and geometry
int query_view(const bq_query *q, const uint64_t *const **ptrs, const uint64_t **lens, int *n, uint64_t *nwords,
               uint64_t *full_words, uint64_t *last_mask, int *device);
}  // namespace bq

extern "C" BQ_API int bq_program_execute(bq_program *p, bq_query *q, uint64_t *d_out, unsigned long long *d_popcnt,
                                         unsigned long long *d_last_nz, void *stream) {
    if (!p) return set_error(BQ_EINPUT, "program is NULL");
    const uint64_t *const *ptrs;
    const uint64_t *lens;
    int n, device;
    uint64_t nwords, full, last_mask;
    int rc = query_view(q, &ptrs, &lens, &n, &nwords, &full, &last_mask, &device);
    if (rc) return rc;
    if (n != p->arity) return set_error(BQ_EINPUT, "program expects %d inputs, got %d", p->arity, n);  // programs.py:241-242
    if (nwords && !d_out) return set_error(BQ_EINPUT, "d_out is NULL");
    if (!nwords) return BQ_OK;
    DeviceGuard dg;
    if ((rc = dg.set(device))) return rc;
    CUfunction_t fn = nullptr;
    if ((rc = program_function(p, &fn))) return rc;
    const unsigned threads = 256;
    uint64_t grid = (2 * nwords + threads - 1) / threads;  // a thread per 32-bit half word
    const uint64_t cap = (uint64_t)sm_count() * 8;
    if (grid > cap) grid = cap;
    void *args[] = {(void *)&ptrs, (void *)&lens, (void *)&nwords, (void *)&full, (void *)&last_mask,
                    (void *)&d_out, (void *)&d_popcnt, (void *)&d_last_nz};
    const int r = jit().cuLaunchKernel(fn, (unsigned)grid, 1, 1, threads, 1, 1, 0, stream, args, nullptr);
    if (r != 0) return set_error(BQ_ECUDA, "cuLaunchKernel(bq_prog) failed (CUresult %d)", r);
    return BQ_OK;
}
