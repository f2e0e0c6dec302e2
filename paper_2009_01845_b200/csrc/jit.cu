// Runtime specialisation of fused passes: NVRTC compiles the straight-line consumer body that
// paper_2009_01845_b200/jit.py generates for one pass *structure* (bit positions, layouts, op
// kinds; matrix / phase values stay runtime coefficients), for sm_100a, and the driver API
// loads and launches it.  Same TMA producer, mbarrier ring and tile addressing as the
// interpreted kernel in pass.cu; no dispatch loop, every amplitude stays in a named register.
#include <atomic>
#include <mutex>
#include <dlfcn.h>
#include <stdio.h>
#include <string.h>

#include "pass_host.h"
#include "qsb_common.cuh"

namespace qsb {
namespace jit {

// --- NVRTC (dlopen'ed: the library does not hard-link it) ----------------------------------
typedef int nvrtcResult_t;
typedef void* nvrtcProgram_t;
struct Nvrtc {
  nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int, const char* const*, const char* const*);
  nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*);
  nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*cubin)(nvrtcProgram_t, char*);
  nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*log)(nvrtcProgram_t, char*);
  nvrtcResult_t (*destroy)(nvrtcProgram_t*);
  bool ok = false;
};

static Nvrtc* nvrtc(const char* path_hint) {
  static Nvrtc n;
  static bool tried = false;
  if (tried) return n.ok ? &n : nullptr;
  tried = true;
  const char* cands[] = {path_hint, "libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"};
  void* h = nullptr;
  for (const char* c : cands) {
    if (!c || !*c) continue;
    h = dlopen(c, RTLD_NOW | RTLD_LOCAL);
    if (h) break;
  }
  if (!h) return nullptr;
#define QSB_SYM(field, name)                                              \
  n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name));          \
  if (!n.field) return nullptr;
  QSB_SYM(create, "nvrtcCreateProgram")
  QSB_SYM(compile, "nvrtcCompileProgram")
  QSB_SYM(cubin_size, "nvrtcGetCUBINSize")
  QSB_SYM(cubin, "nvrtcGetCUBIN")
  QSB_SYM(log_size, "nvrtcGetProgramLogSize")
  QSB_SYM(log, "nvrtcGetProgramLog")
  QSB_SYM(destroy, "nvrtcDestroyProgram")
#undef QSB_SYM
  n.ok = true;
  return &n;
}

// --- driver API through the runtime's entry-point query (no -lcuda) -------------------------
struct Driver {
  CUresult (*load)(CUmodule*, const void*);
  CUresult (*get_fn)(CUfunction*, CUmodule, const char*);
  CUresult (*set_attr)(CUfunction, CUfunction_attribute, int);
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                     void**, void**);
  bool ok = false;
};

static Driver* driver() {
  static Driver d;
  static bool tried = false;
  if (tried) return d.ok ? &d : nullptr;
  tried = true;
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
#define QSB_DRV(field, name)                                                                    \
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) \
    return nullptr;                                                                             \
  d.field = reinterpret_cast<decltype(d.field)>(p);
  QSB_DRV(load, "cuModuleLoadData")
  QSB_DRV(get_fn, "cuModuleGetFunction")
  QSB_DRV(set_attr, "cuFuncSetAttribute")
  QSB_DRV(launch, "cuLaunchKernel")
#undef QSB_DRV
  d.ok = true;
  return &d;
}

}  // namespace jit
}  // namespace qsb

using namespace qsb;

extern "C" int qsb_jit_available(const char* nvrtc_path) {
  return (jit::nvrtc(nvrtc_path) && jit::driver()) ? 1 : 0;
}

// Compile `source` (CUDA C++) with NVRTC for sm_100a and return the CUfunction `name`.
extern "C" int qsb_jit_compile(const char* source, const char* name, const char* nvrtc_path, void** func_out,
                               char* log_out, size_t log_cap) {
  return qsb_jit_compile_cubin(source, name, nvrtc_path, func_out, log_out, log_cap, nullptr, 0, nullptr);
}

extern "C" int qsb_jit_compile_cubin(const char* source, const char* name, const char* nvrtc_path, void** func_out,
                                     char* log_out, size_t log_cap, void* cubin_out, size_t cubin_cap,
                                     size_t* cubin_size) {
  jit::Nvrtc* nv = jit::nvrtc(nvrtc_path);
  jit::Driver* dr = jit::driver();
  if (!nv || !dr) {
    set_error("qsb_jit_compile: NVRTC or the CUDA driver API is unavailable");
    return QSB_ERR_CUDA;
  }
  // NVRTC needs a current context for nothing, but module loading does: make sure the runtime
  // has initialised the primary context on this thread.
  cudaFree(nullptr);
  jit::nvrtcProgram_t prog = nullptr;
  if (nv->create(&prog, source, "qsb_pass.cu", 0, nullptr, nullptr) != 0) {
    set_error("nvrtcCreateProgram failed");
    return QSB_ERR_CUDA;
  }
  const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-default-device", "-lineinfo", "--use_fast_math=false"};
  const int rc = nv->compile(prog, 4, opts);
  size_t ls = 0;
  nv->log_size(prog, &ls);
  if (log_out && log_cap) {
    log_out[0] = 0;
    if (ls > 1) {
      char* buf = new char[ls];
      nv->log(prog, buf);
      snprintf(log_out, log_cap, "%s", buf);
      delete[] buf;
    }
  }
  if (rc != 0) {
    nv->destroy(&prog);
    set_error("NVRTC compilation failed (see log)");
    return QSB_ERR_ARG;
  }
  size_t cs = 0;
  nv->cubin_size(prog, &cs);
  char* cubin = new char[cs];
  nv->cubin(prog, cubin);
  nv->destroy(&prog);
  if (cubin_out) {  // hand the image to the caller's on-disk cache
    if (cubin_size) *cubin_size = cs;
    if (cs <= cubin_cap) memcpy(cubin_out, cubin, cs);
  }
  const int st = qsb_jit_load(cubin, name, func_out);
  delete[] cubin;
  return st;
}

// Tile counters of the dynamically scheduled pass kernels: 2 x u64 per slot (next tile
// chunk, retired producers), zero between launches (the last producer of a launch re-arms its
// slot).  Launches take slots round-robin, so concurrent launches on different streams do not
// share a counter unless kSchedSlots launches are in flight at once.
constexpr int kSchedSlots = 1024;
// launches recorded into a CUDA graph keep their counter for the graph's lifetime: they take
// slots from a separate, never-recycled range (a replay must not share a counter with a live
// launch on another stream)
constexpr int kSchedGraphSlots = 8192;
static unsigned long long* g_sched[64];
static std::atomic<unsigned> g_sched_next{0};
static std::atomic<unsigned> g_sched_graph_next{0};
static std::mutex g_sched_mu;

static int sched_slot(unsigned long long** out, cudaStream_t st = nullptr, bool check_capture = false) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) {
    set_error("qsb_jit_run_pass: device %d out of range", dev);
    return QSB_ERR_ARG;
  }
  if (!g_sched[dev]) {
    std::lock_guard<std::mutex> lk(g_sched_mu);
    if (!g_sched[dev]) {
      void* p = nullptr;
      const size_t bytes = (size_t)(kSchedSlots + kSchedGraphSlots) * 2 * sizeof(unsigned long long);
      cudaError_t e = cudaMalloc(&p, bytes);
      if (e != cudaSuccess) return cuda_status(e, "tile counters");
      e = cudaMemset(p, 0, bytes);
      if (e != cudaSuccess) return cuda_status(e, "tile counters");
      cudaDeviceSynchronize();
      g_sched[dev] = static_cast<unsigned long long*>(p);
    }
  }
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (check_capture && cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusActive) {
    const unsigned k = g_sched_graph_next.fetch_add(1);
    if (k >= (unsigned)kSchedGraphSlots) {
      set_error("qsb_jit_run_pass: more than %d pass launches captured in CUDA graphs", kSchedGraphSlots);
      return QSB_ERR_CAPACITY;
    }
    *out = g_sched[dev] + 2 * ((size_t)kSchedSlots + k);
    return QSB_OK;
  }
  *out = g_sched[dev] + 2 * (g_sched_next.fetch_add(1) % kSchedSlots);
  return QSB_OK;
}

extern "C" int qsb_jit_load(const void* cubin, const char* name, void** func_out) {
  jit::Driver* dr = jit::driver();
  if (!dr) {
    set_error("qsb_jit_load: the CUDA driver API is unavailable");
    return QSB_ERR_CUDA;
  }
  cudaFree(nullptr);  // the runtime's primary context current on this thread
  unsigned long long* slot = nullptr;  // allocate the tile counters now, never under capture
  if (int rc = sched_slot(&slot)) return rc;
  CUmodule mod = nullptr;
  CUresult r = dr->load(&mod, cubin);
  if (r != CUDA_SUCCESS) {
    set_error("cuModuleLoadData failed (%d)", (int)r);
    return QSB_ERR_CUDA;
  }
  CUfunction fn = nullptr;
  r = dr->get_fn(&fn, mod, name);
  if (r != CUDA_SUCCESS) {
    set_error("cuModuleGetFunction(%s) failed (%d)", name, (int)r);
    return QSB_ERR_CUDA;
  }
  *func_out = reinterpret_cast<void*>(fn);
  return QSB_OK;
}

// Launch a JIT pass kernel: params (src, dst, tensor map, coefficients, tile counter).  The tensor map is
// encoded here from `tdesc` (jit.py tma_plan: rank, dims[5], byte strides[4], box[5]) over the
// 8-byte elements of the state at `src`.
static int encode_desc(CUtensorMap* map, void* base, const int64_t* tdesc) {
  cuuint64_t gdim[5], gstride[4];
  cuuint32_t box[5], estride[5];
  for (int d = 0; d < 5; ++d) {
    gdim[d] = (cuuint64_t)tdesc[1 + d];
    box[d] = (cuuint32_t)tdesc[10 + d];
    estride[d] = 1;
    if (d < 4) gstride[d] = (cuuint64_t)tdesc[6 + d];
  }
  return pass::encode_tensor_map(map, base, gdim, gstride, box, estride);
}

static int run_pass_impl(void* func, const void* src, void* dst, const int64_t* tdesc, const int64_t* tdesc_out,
                         uint64_t n_tiles,
                         const double* coeffs, int64_t n_coeffs, bool coeffs_on_device, const void* params,
                         int64_t param_bytes, int threads, int smem_bytes, int grid, void* stream) {
  jit::Driver* dr = jit::driver();
  if (!dr || !func) {
    set_error("qsb_jit_run_pass: no driver / function");
    return QSB_ERR_CUDA;
  }
  if (!tdesc || tdesc[0] != 5 || n_tiles == 0 || !params || param_bytes <= 0 || param_bytes > 31616) {
    set_error("qsb_jit_run_pass: bad tile descriptor");
    return QSB_ERR_ARG;
  }
  cudaStream_t st = as_stream(stream);
  void* dcoef = nullptr;
  if (n_coeffs > 0) {
    if (coeffs_on_device)
      dcoef = const_cast<double*>(coeffs);
    else if (int rc = pass::stage_words(coeffs, sizeof(double) * n_coeffs, &dcoef, st))
      return rc;
  }
  alignas(64) CUtensorMap map;
  alignas(64) CUtensorMap map_o;
  memset(&map, 0, sizeof map);
  if (int rc = encode_desc(&map, const_cast<void*>(src), tdesc)) return rc;
  if (tdesc_out) {
    if (tdesc_out[0] != 5) {
      set_error("qsb_jit_run_pass: bad output tile descriptor");
      return QSB_ERR_ARG;
    }
    memset(&map_o, 0, sizeof map_o);
    if (int rc = encode_desc(&map_o, dst, tdesc_out)) return rc;
  } else {
    map_o = map;
  }
  CUfunction fn = reinterpret_cast<CUfunction>(func);
  static CUfunction attr_done[256];
  static int n_attr = 0;
  bool seen = false;
  for (int i = 0; i < n_attr; ++i) seen |= attr_done[i] == fn;
  if (!seen) {
    CUresult r = dr->set_attr(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem_bytes);
    if (r != CUDA_SUCCESS) {
      set_error("cuFuncSetAttribute failed (%d)", (int)r);
      return QSB_ERR_CUDA;
    }
    if (n_attr < 256) attr_done[n_attr++] = fn;
  }
  if (grid <= 0 || (uint64_t)grid > n_tiles) {
    set_error("qsb_jit_run_pass: grid %d outside [1, n_tiles]", grid);
    return QSB_ERR_ARG;
  }
  const void* a_src = src;
  void* a_dst = dst;
  const double* a_cf = static_cast<const double*>(dcoef);
  unsigned long long* a_sched = nullptr;
  if (int rc = sched_slot(&a_sched, st, true)) return rc;
  // the last kernel parameter is the coefficient struct, copied by value from `params`
  void* args[] = {(void*)&a_src, (void*)&a_dst, (void*)&map, (void*)&map_o, (void*)&a_cf, (void*)&a_sched,
                  const_cast<void*>(params)};
  CUresult r = dr->launch(fn, (unsigned)grid, 1, 1, (unsigned)threads, 1, 1, (unsigned)smem_bytes, (CUstream)st, args,
                          nullptr);
  if (r != CUDA_SUCCESS) {
    set_error("cuLaunchKernel failed (%d)", (int)r);
    return QSB_ERR_CUDA;
  }
  return QSB_OK;
}

extern "C" int qsb_jit_run_pass(void* func, const void* src, void* dst, const int64_t* tdesc,
                                const int64_t* tdesc_out, uint64_t n_tiles, const double* tables, int64_t n_tables,
                                const void* params, int64_t param_bytes, int threads, int smem_bytes, int grid,
                                void* stream) {
  return run_pass_impl(func, src, dst, tdesc, tdesc_out, n_tiles, tables, n_tables, false, params, param_bytes,
                       threads, smem_bytes, grid, stream);
}

extern "C" int qsb_jit_run_pass_dev(void* func, const void* src, void* dst, const int64_t* tdesc,
                                    const int64_t* tdesc_out, uint64_t n_tiles, const double* dev_tables,
                                    int64_t n_tables, const void* params, int64_t param_bytes, int threads,
                                    int smem_bytes, int grid, void* stream) {
  return run_pass_impl(func, src, dst, tdesc, tdesc_out, n_tiles, dev_tables, n_tables, true, params, param_bytes,
                       threads, smem_bytes, grid, stream);
}
