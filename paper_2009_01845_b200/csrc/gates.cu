// Single-gate kernels, initial states and small reductions for the qsb200 engine.
//
// Each entry point replaces one numeric body of the reference simulator:
//   qsb_init_basis / qsb_init_uniform  <- state.py:67-75 zero_state, hamiltonians.py:115-117
//   qsb_apply_matrix                   <- gates.py:380-469 apply_matrix (all three bodies)
//   qsb_scale                          <- sharding.py:281-283 whole-shard phase, state.py:105
//   qsb_norm2 / qsb_vdot               <- state.py:109-122 norm / overlap
//   qsb_pack_half / qsb_unpack_half    <- sharding.py:100-111 _exchange_halves (staging side)
//
// Kernel design (B200): one thread owns ITEMS amplitude groups; all loads of a thread are
// issued before any arithmetic so every thread keeps 2*ITEMS (1q) or 4*ITEMS (2q) independent
// 8/16-byte loads in flight.  Group -> index mapping is the reference's zero-bit insertion done
// in registers.  Consecutive threads own consecutive groups, so whenever the lowest bits are
// not occupied a warp touches one contiguous 256 B / 512 B segment per load instruction.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <mutex>

#include "qsb_common.cuh"

namespace qsb {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
  set_error("%s: CUDA error %d (%s)", where, (int)e, cudaGetErrorString(e));
  return QSB_ERR_CUDA;
}

constexpr int kThreads = 256;

// ------------------------------------------------------------------------------------------
// initial states
// ------------------------------------------------------------------------------------------
template <typename R>
__global__ void k_set_one(cplx<R>* a, uint64_t idx) {
  cplx<R> v;
  v.x = R(1);
  v.y = R(0);
  a[idx] = v;
}

template <typename R>
__global__ void k_fill(cplx<R>* __restrict__ a, uint64_t n, R re, R im) {
  cplx<R> v;
  v.x = re;
  v.y = im;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) a[i] = v;
}

template <typename R>
__global__ void k_scale(cplx<R>* __restrict__ a, uint64_t n, cplx<R> s) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    a[i] = cmul(a[i], s);
}

// projective collapse: amplitudes whose bits under `mask` equal `value` are scaled by `s`, the
// rest are zeroed without being read (only the kept fraction is loaded)
template <typename R>
__global__ void k_collapse(cplx<R>* __restrict__ a, uint64_t n, uint64_t mask, uint64_t value, R s) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    cplx<R> v;
    if ((i & mask) == value) {
      v = a[i];
      v.x *= s;
      v.y *= s;
    } else {
      v.x = (R)0;
      v.y = (R)0;
    }
    a[i] = v;
  }
}

static int stream_grid(uint64_t n) {
  // enough CTAs for 8 resident per SM on 148 SMs, capped by the work
  uint64_t want = (n + kThreads - 1) / kThreads;
  uint64_t cap = 148ull * 16ull;
  return (int)(want < cap ? (want < 1 ? 1 : want) : cap);
}

// ------------------------------------------------------------------------------------------
// gate kernels
// ------------------------------------------------------------------------------------------
// Parameters of one group-structured gate launch.  `off[j]` is the bit pattern of matrix row j
// on the target bits (target_bits[0] = MSB of j), `cmask` the OR of the control bits.
template <typename R>
struct GateArgs {
  uint64_t n_groups;
  uint64_t cmask;
  uint64_t off[4];
  OccBits occ;
  cplx<R> m[16];       // general: row-major 2^t x 2^t; diag: m[r] for r < nrows
  uint32_t rows[4];    // diag: rows to multiply; perm: destination rows
  uint32_t src[4];     // perm: source row of each destination row
  uint32_t use_phase;  // perm: bit r set -> multiply row r by m[r]
  int nrows;
};

template <typename R, int ITEMS>
__global__ void __launch_bounds__(kThreads) k_general1(cplx<R>* __restrict__ a, const GateArgs<R> p) {
  using C = cplx<R>;
  const uint64_t g0 = (uint64_t)blockIdx.x * (kThreads * ITEMS) + threadIdx.x;
  uint64_t base[ITEMS];
  C x0[ITEMS], x1[ITEMS];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint64_t g = g0 + (uint64_t)it * kThreads;
    base[it] = ~0ull;
    if (g < p.n_groups) {
      base[it] = insert_zero_bits(g, p.occ) | p.cmask;
      x0[it] = a[base[it]];
      x1[it] = a[base[it] | p.off[1]];
    }
  }
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    if (base[it] == ~0ull) continue;
    C y0 = cmad(p.m[1], x1[it], cmul(p.m[0], x0[it]));
    C y1 = cmad(p.m[3], x1[it], cmul(p.m[2], x0[it]));
    a[base[it]] = y0;
    a[base[it] | p.off[1]] = y1;
  }
}

template <typename R, int ITEMS>
__global__ void __launch_bounds__(kThreads) k_general2(cplx<R>* __restrict__ a, const GateArgs<R> p) {
  using C = cplx<R>;
  const uint64_t g0 = (uint64_t)blockIdx.x * (kThreads * ITEMS) + threadIdx.x;
  uint64_t base[ITEMS];
  C x[ITEMS][4];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint64_t g = g0 + (uint64_t)it * kThreads;
    base[it] = ~0ull;
    if (g < p.n_groups) {
      base[it] = insert_zero_bits(g, p.occ) | p.cmask;
#pragma unroll
      for (int j = 0; j < 4; ++j) x[it][j] = a[base[it] | p.off[j]];
    }
  }
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    if (base[it] == ~0ull) continue;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      C y = cmul(p.m[4 * r], x[it][0]);
      y = cmad(p.m[4 * r + 1], x[it][1], y);
      y = cmad(p.m[4 * r + 2], x[it][2], y);
      y = cmad(p.m[4 * r + 3], x[it][3], y);
      a[base[it] | p.off[r]] = y;
    }
  }
}

// diagonal body (gates.py:431-441): only rows whose complex128 entry differs from 1.0
template <typename R, int ITEMS>
__global__ void __launch_bounds__(kThreads) k_diag(cplx<R>* __restrict__ a, const GateArgs<R> p) {
  using C = cplx<R>;
  const uint64_t g0 = (uint64_t)blockIdx.x * (kThreads * ITEMS) + threadIdx.x;
  uint64_t base[ITEMS];
  C x[ITEMS][4];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint64_t g = g0 + (uint64_t)it * kThreads;
    base[it] = ~0ull;
    if (g < p.n_groups) {
      base[it] = insert_zero_bits(g, p.occ) | p.cmask;
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (r < p.nrows) x[it][r] = a[base[it] | p.off[p.rows[r]]];
    }
  }
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    if (base[it] == ~0ull) continue;
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (r < p.nrows) a[base[it] | p.off[p.rows[r]]] = cmul(x[it][r], p.m[r]);
  }
}

// permutation body (gates.py:443-459): gather every moved row first, then scatter
template <typename R, int ITEMS>
__global__ void __launch_bounds__(kThreads) k_perm(cplx<R>* __restrict__ a, const GateArgs<R> p) {
  using C = cplx<R>;
  const uint64_t g0 = (uint64_t)blockIdx.x * (kThreads * ITEMS) + threadIdx.x;
  uint64_t base[ITEMS];
  C x[ITEMS][4];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint64_t g = g0 + (uint64_t)it * kThreads;
    base[it] = ~0ull;
    if (g < p.n_groups) {
      base[it] = insert_zero_bits(g, p.occ) | p.cmask;
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (r < p.nrows) x[it][r] = a[base[it] | p.off[p.src[r]]];
    }
  }
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    if (base[it] == ~0ull) continue;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (r < p.nrows) {
        C v = x[it][r];
        if (p.use_phase & (1u << r)) v = cmul(v, p.m[r]);
        a[base[it] | p.off[p.rows[r]]] = v;
      }
    }
  }
}

template <typename R>
static void to_dtype(const double* re_im, cplx<R>* out) {
  out->x = (R)re_im[0];
  out->y = (R)re_im[1];
}

static bool is_one(const double* z) { return z[0] == 1.0 && z[1] == 0.0; }
static bool is_nonzero(const double* z) { return z[0] != 0.0 || z[1] != 0.0; }

// Which body a prepared gate runs (0: nothing to do).
enum GateBody { kBodyNone = 0, kBodyDiag = 1, kBodyPerm = 2, kBodyGeneral1 = 3, kBodyGeneral2 = 4 };

// Host side of one apply_matrix call: group geometry + the body's rows/coefficients, the
// classification of gates.py:431-467 (diagonal rows != 1.0, permutation argmax sources,
// general matrix cast to the state dtype).
template <typename R>
static int prepare_gate(int n_qubits, int t, const int* tbits, int nc, const int* cbits, const double* mat,
                        int kclass, GateArgs<R>& p) {
  memset(&p, 0, sizeof p);
  const int dim = 1 << t;
  // occupied bits, ascending
  int occ[kMaxOcc];
  int nocc = 0;
  for (int i = 0; i < t; ++i) occ[nocc++] = tbits[i];
  for (int i = 0; i < nc; ++i) occ[nocc++] = cbits[i];
  for (int i = 1; i < nocc; ++i)
    for (int j = i; j > 0 && occ[j - 1] > occ[j]; --j) {
      int tmp = occ[j];
      occ[j] = occ[j - 1];
      occ[j - 1] = tmp;
    }
  p.occ.n = nocc;
  for (int i = 0; i < nocc; ++i) p.occ.pos[i] = (uint8_t)occ[i];
  p.cmask = 0;
  for (int i = 0; i < nc; ++i) p.cmask |= 1ull << cbits[i];
  for (int j = 0; j < dim; ++j) {
    uint64_t off = 0;
    for (int b = 0; b < t; ++b)
      if ((j >> (t - 1 - b)) & 1) off |= 1ull << tbits[b];
    p.off[j] = off;
  }
  p.n_groups = 1ull << (n_qubits - nocc);

  if (kclass == QSB_KERNEL_DIAGONAL) {
    int nr = 0;
    for (int j = 0; j < dim; ++j) {
      const double* d = mat + 2 * (j * dim + j);
      if (!is_one(d)) {
        p.rows[nr] = j;
        to_dtype<R>(d, &p.m[nr]);
        ++nr;
      }
    }
    p.nrows = nr;
    return nr == 0 ? kBodyNone : kBodyDiag;
  }
  if (kclass == QSB_KERNEL_PERMUTATION) {
    int nr = 0;
    for (int j = 0; j < dim; ++j) {
      int s = 0;  // np.argmax(mat != 0): first non-zero column (0 if the row is all zero)
      for (int c = 0; c < dim; ++c)
        if (is_nonzero(mat + 2 * (j * dim + c))) {
          s = c;
          break;
        }
      const double* ph = mat + 2 * (j * dim + s);
      const bool phase = !is_one(ph);
      if (s != j || phase) {
        p.rows[nr] = j;
        p.src[nr] = s;
        if (phase) p.use_phase |= 1u << nr;
        to_dtype<R>(ph, &p.m[nr]);
        ++nr;
      }
    }
    p.nrows = nr;
    return nr == 0 ? kBodyNone : kBodyPerm;
  }
  for (int k = 0; k < dim * dim; ++k) to_dtype<R>(mat + 2 * k, &p.m[k]);
  return t == 1 ? kBodyGeneral1 : kBodyGeneral2;
}

// ---- 3..5-target matrices (apply_matrix takes any 2^t x 2^t matrix, gates.py:380-469) -------
// One thread per group of 2^T amplitudes; the matrix travels as a kernel parameter (<= 16 KB at
// T = 5, complex128).  mode 0: general (every row = M x), 1: diagonal (rows in `rowmask` times
// m[r]), 2: permutation (row r <- m[r] * x[src[r]] for rows in `rowmask`; all loads first).
constexpr int kMaxWideTargets = 5;

template <typename R, int T>
struct WideArgs {
  uint64_t n_groups;
  uint64_t cmask;
  uint64_t off[1 << T];
  OccBits occ;
  int mode;
  uint32_t rowmask;
  uint32_t phasemask;  // permutation: rows whose entry is not exactly 1 (multiplied)
  uint8_t src[1 << T];
  cplx<R> m[(1 << T) * (1 << T)];
};

template <typename R, int T>
__global__ void __launch_bounds__(128) k_wide(cplx<R>* __restrict__ a, const __grid_constant__ WideArgs<R, T> p) {
  using C = cplx<R>;
  constexpr int D = 1 << T;
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= p.n_groups) return;
  const uint64_t base = insert_zero_bits(g, p.occ) | p.cmask;
  C x[D];
  if (p.mode == 1) {
#pragma unroll
    for (int r = 0; r < D; ++r)
      if ((p.rowmask >> r) & 1u) x[r] = a[base | p.off[r]];
#pragma unroll
    for (int r = 0; r < D; ++r)
      if ((p.rowmask >> r) & 1u) a[base | p.off[r]] = cmul(x[r], p.m[r]);
    return;
  }
  if (p.mode == 2) {
#pragma unroll
    for (int r = 0; r < D; ++r)
      if ((p.rowmask >> r) & 1u) x[r] = a[base | p.off[p.src[r]]];
#pragma unroll
    for (int r = 0; r < D; ++r)
      if ((p.rowmask >> r) & 1u) a[base | p.off[r]] = ((p.phasemask >> r) & 1u) ? cmul(x[r], p.m[r]) : x[r];
    return;
  }
#pragma unroll
  for (int c = 0; c < D; ++c) x[c] = a[base | p.off[c]];
#pragma unroll
  for (int r = 0; r < D; ++r) {
    C y = cmul(p.m[r * D], x[0]);
#pragma unroll
    for (int c = 1; c < D; ++c) y = cmad(p.m[r * D + c], x[c], y);
    a[base | p.off[r]] = y;
  }
}

template <typename R, int T>
static int launch_wide(cplx<R>* a, int n_qubits, const int* tbits, int nc, const int* cbits, const double* mat,
                       int kclass, cudaStream_t st) {
  constexpr int D = 1 << T;
  WideArgs<R, T> p;
  memset(&p, 0, sizeof p);
  int occ[kMaxOcc];
  int nocc = 0;
  for (int i = 0; i < T; ++i) occ[nocc++] = tbits[i];
  for (int i = 0; i < nc; ++i) occ[nocc++] = cbits[i];
  for (int i = 1; i < nocc; ++i)
    for (int j = i; j > 0 && occ[j - 1] > occ[j]; --j) {
      int tmp = occ[j];
      occ[j] = occ[j - 1];
      occ[j - 1] = tmp;
    }
  p.occ.n = nocc;
  for (int i = 0; i < nocc; ++i) p.occ.pos[i] = (uint8_t)occ[i];
  for (int i = 0; i < nc; ++i) p.cmask |= 1ull << cbits[i];
  for (int j = 0; j < D; ++j)
    for (int b = 0; b < T; ++b)
      if ((j >> (T - 1 - b)) & 1) p.off[j] |= 1ull << tbits[b];
  p.n_groups = 1ull << (n_qubits - nocc);
  if (kclass == QSB_KERNEL_DIAGONAL) {
    p.mode = 1;
    for (int j = 0; j < D; ++j) {
      const double* d = mat + 2 * (j * D + j);
      if (!is_one(d)) {
        p.rowmask |= 1u << j;
        to_dtype<R>(d, &p.m[j]);
      }
    }
  } else if (kclass == QSB_KERNEL_PERMUTATION) {
    p.mode = 2;
    for (int j = 0; j < D; ++j) {
      int s = 0;  // np.argmax(mat != 0)
      for (int c = 0; c < D; ++c)
        if (is_nonzero(mat + 2 * (j * D + c))) {
          s = c;
          break;
        }
      const double* ph = mat + 2 * (j * D + s);
      if (s != j || !is_one(ph)) {
        p.rowmask |= 1u << j;
        p.src[j] = (uint8_t)s;
        if (!is_one(ph)) p.phasemask |= 1u << j;
        to_dtype<R>(ph, &p.m[j]);
      }
    }
  } else {
    p.mode = 0;
    for (int k = 0; k < D * D; ++k) to_dtype<R>(mat + 2 * k, &p.m[k]);
  }
  if (p.mode != 0 && p.rowmask == 0) return QSB_OK;
  k_wide<R, T><<<blocks_for(p.n_groups, 128), 128, 0, st>>>(a, p);
  QSB_CHECK_LAUNCH("qsb_apply_matrix(3-5 targets)");
  return QSB_OK;
}

// 6-10 targets (the reference's apply_matrix takes any 2^t x 2^t matrix): one CTA of 2^t
// threads per group of 2^t amplitudes, staged in shared memory; thread r forms row r of the
// product, y_r = sum_c M[r][c] x_c in column order, reading the matrix transposed (coalesced
// across the rows, L2-resident across the groups: at most 1024 x 1024 complex128 = 16 MB).
// Diagonal and permutation matrices take the same dense body (exact zeros and ones change no
// bits of a sum).  A drop-in completeness path, not a hot one.
constexpr int kMaxDenseTargets = 10;

template <typename R>
__global__ void __launch_bounds__(1024) k_dense_big(cplx<R>* __restrict__ a, const double2* __restrict__ mt, int t,
                                                    OccBits occ, uint64_t cmask, uint64_t n_groups,
                                                    const int* __restrict__ tbits_dev) {
  using C = cplx<R>;
  extern __shared__ __align__(16) unsigned char big_raw[];
  C* xs = reinterpret_cast<C*>(big_raw);
  const int D = 1 << t;
  const int r = threadIdx.x;
  uint64_t off = 0;
  for (int b = 0; b < t; ++b)
    if ((r >> (t - 1 - b)) & 1) off |= 1ull << tbits_dev[b];
  for (uint64_t g = blockIdx.x; g < n_groups; g += gridDim.x) {
    const uint64_t base = insert_zero_bits(g, occ) | cmask;
    xs[r] = a[base | off];
    __syncthreads();
    const double2 m0 = mt[r];
    C m;
    m.x = (R)m0.x;
    m.y = (R)m0.y;
    C y = cmul(m, xs[0]);
    for (int c = 1; c < D; ++c) {
      const double2 mc = mt[(uint64_t)c * D + r];
      m.x = (R)mc.x;
      m.y = (R)mc.y;
      y = cmad(m, xs[c], y);
    }
    __syncthreads();
    a[base | off] = y;
  }
}

template <typename R>
static int launch_dense_big(void* amps, int n_qubits, int t, const int* tbits, int nc, const int* cbits,
                            const double* mat, cudaStream_t st) {
  const int D = 1 << t;
  OccBits occ;
  int pos[64];
  int np = 0;
  for (int i = 0; i < t; ++i) pos[np++] = tbits[i];
  for (int i = 0; i < nc; ++i) pos[np++] = cbits[i];
  for (int i = 1; i < np; ++i)
    for (int j = i; j > 0 && pos[j - 1] > pos[j]; --j) {
      const int tmp = pos[j];
      pos[j] = pos[j - 1];
      pos[j - 1] = tmp;
    }
  occ.n = np;
  for (int i = 0; i < np; ++i) occ.pos[i] = (uint8_t)pos[i];
  uint64_t cmask = 0;
  for (int i = 0; i < nc; ++i) cmask |= 1ull << cbits[i];
  const uint64_t n_groups = 1ull << (n_qubits - np);
  // the transposed matrix (mt[c][r] = M[r][c]) and the target bits on the device, freed in order
  const size_t mbytes = (size_t)D * D * sizeof(double2);
  double2* h = static_cast<double2*>(malloc(mbytes));
  if (!h) {
    set_error("apply_matrix: host staging of a %d x %d matrix", D, D);
    return QSB_ERR_CAPACITY;
  }
  for (int r = 0; r < D; ++r)
    for (int c = 0; c < D; ++c) h[(size_t)c * D + r] = make_double2(mat[2 * ((size_t)r * D + c)], mat[2 * ((size_t)r * D + c) + 1]);
  void* dbuf = nullptr;
  cudaError_t e = cudaMallocAsync(&dbuf, mbytes + 64 * sizeof(int), st);
  if (e != cudaSuccess) {
    free(h);
    return cuda_status(e, "apply_matrix matrix buffer");
  }
  double2* mt = static_cast<double2*>(dbuf);
  int* tb = reinterpret_cast<int*>(static_cast<char*>(dbuf) + mbytes);
  e = cudaMemcpyAsync(mt, h, mbytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(tb, tbits, t * sizeof(int), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // the pageable staging is reused below
  free(h);
  if (e != cudaSuccess) {
    cudaFreeAsync(dbuf, st);
    return cuda_status(e, "apply_matrix matrix upload");
  }
  const uint64_t grid = n_groups < 148ull * 4 ? n_groups : 148ull * 4;
  k_dense_big<R><<<(int)grid, D, D * sizeof(cplx<R>), st>>>(static_cast<cplx<R>*>(amps), mt, t, occ, cmask, n_groups,
                                                              tb);
  e = cudaGetLastError();
  cudaFreeAsync(dbuf, st);
  if (e != cudaSuccess) return cuda_status(e, "qsb_apply_matrix(6-10 targets)");
  return QSB_OK;
}

template <typename R>
static int launch_gate(void* amps, int n_qubits, int t, const int* tbits, int nc, const int* cbits,
                       const double* mat, int kclass, cudaStream_t st) {
  cplx<R>* a = static_cast<cplx<R>*>(amps);
  if (t > kMaxWideTargets) return launch_dense_big<R>(amps, n_qubits, t, tbits, nc, cbits, mat, st);
  switch (t) {
    case 3:
      return launch_wide<R, 3>(a, n_qubits, tbits, nc, cbits, mat, kclass, st);
    case 4:
      return launch_wide<R, 4>(a, n_qubits, tbits, nc, cbits, mat, kclass, st);
    case 5:
      return launch_wide<R, 5>(a, n_qubits, tbits, nc, cbits, mat, kclass, st);
    default:
      break;
  }
  GateArgs<R> p;
  const int body = prepare_gate<R>(n_qubits, t, tbits, nc, cbits, mat, kclass, p);
  switch (body) {
    case kBodyDiag:
      k_diag<R, 4><<<blocks_for(p.n_groups, kThreads * 4), kThreads, 0, st>>>(a, p);
      QSB_CHECK_LAUNCH("qsb_apply_matrix(diagonal)");
      break;
    case kBodyPerm:
      k_perm<R, 4><<<blocks_for(p.n_groups, kThreads * 4), kThreads, 0, st>>>(a, p);
      QSB_CHECK_LAUNCH("qsb_apply_matrix(permutation)");
      break;
    case kBodyGeneral1:
      k_general1<R, 4><<<blocks_for(p.n_groups, kThreads * 4), kThreads, 0, st>>>(a, p);
      QSB_CHECK_LAUNCH("qsb_apply_matrix(general)");
      break;
    case kBodyGeneral2:
      k_general2<R, 2><<<blocks_for(p.n_groups, kThreads * 2), kThreads, 0, st>>>(a, p);
      QSB_CHECK_LAUNCH("qsb_apply_matrix(general)");
      break;
    default:
      break;
  }
  return QSB_OK;
}

// ------------------------------------------------------------------------------------------
// deterministic reductions: fixed grid, per-block tree, then one block folds the partials
// ------------------------------------------------------------------------------------------
constexpr int kRedBlocks = 1184;  // 148 SMs x 8

template <typename R>
__global__ void __launch_bounds__(kThreads) k_norm2_partial(const cplx<R>* __restrict__ a, uint64_t n,
                                                            double* __restrict__ part) {
  __shared__ double sh[kThreads];
  double acc = 0.0;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const cplx<R> v = a[i];
    acc = fma((double)v.x, (double)v.x, acc);
    acc = fma((double)v.y, (double)v.y, acc);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

template <typename R>
__global__ void __launch_bounds__(kThreads) k_vdot_partial(const cplx<R>* __restrict__ a,
                                                           const cplx<R>* __restrict__ b, uint64_t n,
                                                           double2* __restrict__ part) {
  __shared__ double2 sh[kThreads];
  double2 acc = make_double2(0.0, 0.0);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const cplx<R> u = a[i];
    const cplx<R> v = b[i];
    // conj(u) * v
    acc.x = fma((double)u.x, (double)v.x, acc.x);
    acc.x = fma((double)u.y, (double)v.y, acc.x);
    acc.y = fma((double)u.x, (double)v.y, acc.y);
    acc.y = fma(-(double)u.y, (double)v.x, acc.y);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sh[threadIdx.x].x += sh[threadIdx.x + s].x;
      sh[threadIdx.x].y += sh[threadIdx.x + s].y;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

template <typename T>
__global__ void __launch_bounds__(1024) k_fold(const T* __restrict__ part, int n, T* out);

template <>
__global__ void __launch_bounds__(1024) k_fold<double>(const double* __restrict__ part, int n, double* out) {
  __shared__ double sh[1024];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) acc += part[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 512; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sh[0];
}

template <>
__global__ void __launch_bounds__(1024) k_fold<double2>(const double2* __restrict__ part, int n, double2* out) {
  __shared__ double2 sh[1024];
  double2 acc = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < n; i += 1024) {
    acc.x += part[i].x;
    acc.y += part[i].y;
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 512; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sh[threadIdx.x].x += sh[threadIdx.x + s].x;
      sh[threadIdx.x].y += sh[threadIdx.x + s].y;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sh[0];
}

// <psi| M_t |psi> summed over up to kExpMax 1- or 2-qubit terms in one launch: per term one
// read-only sweep of the state (no copy, no scratch state), the term matrices are kernel
// parameters (constant-bank operands), accumulation in double, fixed grid => deterministic.
constexpr int kExpMax = 64;
struct ExpTerm {
  int k;       // 1 or 2 target bits
  int hi, lo;  // bit positions: hi = matrix MSB (targets[0]); lo = targets[1] (k = 2)
  int pad;
  double m[32];  // row-major complex (re, im) of the 2^k x 2^k matrix
};
struct ExpTerms {
  int count;
  int pad;
  ExpTerm t[kExpMax];
};

// one term, K target bits: kItems groups per thread per round with all loads issued before any
// math; fully unrolled so the amplitudes stay in registers
template <typename R, int K>
__device__ __forceinline__ void expect_term(const cplx<R>* __restrict__ a, int n, const ExpTerm& e, uint64_t stride,
                                            double2& acc) {
  constexpr int kItems = 4;
  constexpr int D = 1 << K;
  const uint64_t groups = 1ull << (n - K);
  const int b1 = e.hi, b0 = (K == 2) ? e.lo : e.hi;
  const int lo = b1 < b0 ? b1 : b0, hi = b1 < b0 ? b0 : b1;
  const uint64_t off1 = 1ull << e.hi;
  const uint64_t off0 = (K == 2) ? (1ull << e.lo) : 0ull;
  for (uint64_t g0 = (uint64_t)blockIdx.x * kThreads * kItems + threadIdx.x; g0 < groups; g0 += stride * kItems) {
    double xr[kItems][D], xi[kItems][D];
    bool ok[kItems];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const uint64_t g = g0 + (uint64_t)it * kThreads;
      ok[it] = g < groups;
      uint64_t i = ok[it] ? g : 0;
      {
        const uint64_t l = i & ((1ull << lo) - 1ull);
        i = ((i ^ l) << 1) | l;
      }
      if (K == 2) {
        const uint64_t l = i & ((1ull << hi) - 1ull);
        i = ((i ^ l) << 1) | l;
      }
      // matrix row r: bit (K-1) <-> targets[0] (hi), bit 0 <-> targets[1]
#pragma unroll
      for (int r = 0; r < D; ++r) {
        const uint64_t idx = i | ((K == 1) ? ((r & 1) ? off1 : 0ull)
                                           : (((r & 2) ? off1 : 0ull) | ((r & 1) ? off0 : 0ull)));
        const cplx<R> v = a[idx];
        xr[it][r] = (double)v.x;
        xi[it][r] = (double)v.y;
      }
    }
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      if (!ok[it]) continue;
#pragma unroll
      for (int r = 0; r < D; ++r) {
        double yr = 0.0, yi = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const double mr = e.m[2 * (r * D + c)], mi = e.m[2 * (r * D + c) + 1];
          yr = fma(mr, xr[it][c], yr);
          yr = fma(-mi, xi[it][c], yr);
          yi = fma(mr, xi[it][c], yi);
          yi = fma(mi, xr[it][c], yi);
        }
        // conj(x_r) * y_r
        acc.x = fma(xr[it][r], yr, acc.x);
        acc.x = fma(xi[it][r], yi, acc.x);
        acc.y = fma(xr[it][r], yi, acc.y);
        acc.y = fma(-xi[it][r], yr, acc.y);
      }
    }
  }
}

template <typename R>
__global__ void __launch_bounds__(kThreads) k_expect_partial(const cplx<R>* __restrict__ a, int n,
                                                             const __grid_constant__ ExpTerms T,
                                                             double2* __restrict__ part) {
  __shared__ double2 sh[kThreads];
  double2 acc = make_double2(0.0, 0.0);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (int t = 0; t < T.count; ++t) {
    if (T.t[t].k == 1)
      expect_term<R, 1>(a, n, T.t[t], stride, acc);
    else
      expect_term<R, 2>(a, n, T.t[t], stride, acc);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sh[threadIdx.x].x += sh[threadIdx.x + s].x;
      sh[threadIdx.x].y += sh[threadIdx.x + s].y;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void k_add2(double2* out, const double2* v) {
  out->x += v->x;
  out->y += v->y;
}

// scratch for the partials: one lazily grown device buffer per process (tiny)
static void* g_red_scratch = nullptr;
static int ensure_red_scratch() {
  if (g_red_scratch) return QSB_OK;
  cudaError_t e = cudaMalloc(&g_red_scratch, kRedBlocks * sizeof(double2));
  if (e != cudaSuccess) return cuda_status(e, "reduction scratch");
  return QSB_OK;
}

// ------------------------------------------------------------------------------------------
// half-shard staging for the global<->local exchange
// ------------------------------------------------------------------------------------------
template <typename R>
__global__ void k_pack_half(const cplx<R>* __restrict__ s, int bit, int half, uint64_t first, uint64_t count,
                            cplx<R>* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t lowm = (1ull << bit) - 1ull;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += stride) {
    const uint64_t h = first + e;
    const uint64_t i = ((h & ~lowm) << 1) | ((uint64_t)half << bit) | (h & lowm);
    out[e] = s[i];
  }
}

template <typename R>
__global__ void k_unpack_half(cplx<R>* __restrict__ s, int bit, int half, uint64_t first, uint64_t count,
                              const cplx<R>* __restrict__ in) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t lowm = (1ull << bit) - 1ull;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += stride) {
    const uint64_t h = first + e;
    const uint64_t i = ((h & ~lowm) << 1) | ((uint64_t)half << bit) | (h & lowm);
    s[i] = in[e];
  }
}

// k-qubit parts for the batched global<->local exchange: part `bits` of a shard = the
// amplitudes whose local bits at `occ` (ascending) spell `bits` (already placed at those
// positions).  Element e of a part is the e-th such amplitude in index order, so a part whose
// bits are high positions is a few long contiguous runs.
template <typename R>
__global__ void __launch_bounds__(kThreads) k_pack_part(const cplx<R>* __restrict__ s, const OccBits occ,
                                                        uint64_t bits, uint64_t first, uint64_t count,
                                                        cplx<R>* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e < count; e += stride)
    out[e] = s[insert_zero_bits(first + e, occ) | bits];
}

template <typename R>
__global__ void __launch_bounds__(kThreads) k_unpack_part(cplx<R>* __restrict__ s, const OccBits occ,
                                                          uint64_t bits, uint64_t first, uint64_t count,
                                                          const cplx<R>* __restrict__ in) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e < count; e += stride)
    s[insert_zero_bits(first + e, occ) | bits] = in[e];
}

// in-process form: a's part `a_bits` <-> b's part `b_bits`
template <typename R>
__global__ void __launch_bounds__(kThreads) k_exchange_parts(cplx<R>* __restrict__ a, cplx<R>* __restrict__ b,
                                                             const OccBits occ, uint64_t a_bits, uint64_t b_bits,
                                                             uint64_t count) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e < count; e += stride) {
    const uint64_t base = insert_zero_bits(e, occ);
    const cplx<R> t = a[base | a_bits];
    a[base | a_bits] = b[base | b_bits];
    b[base | b_bits] = t;
  }
}

// ------------------------------------------------------------------------------------------
// bit-permuting copy (partition / gather) and half exchange between two shards
// ------------------------------------------------------------------------------------------
struct BitPerm {
  int n;
  uint8_t dst_bit[64];  // destination bit of every source bit
};

// dst[perm(i)] = src[i]; consecutive threads read consecutive source amplitudes
template <typename R>
__global__ void __launch_bounds__(kThreads) k_permute(const cplx<R>* __restrict__ src, cplx<R>* __restrict__ dst,
                                                      uint64_t total, const BitPerm p) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < total; i += stride) {
    uint64_t j = 0;
    for (int b = 0; b < p.n; ++b) j |= ((i >> b) & 1ull) << p.dst_bit[b];
    dst[j] = src[i];
  }
}

// Tiled form (both sides coalesced): a tile is the 2^T elements spanned by the bit set S = the
// low source bits {0..t-1} plus the source bits that land on destination bits {0..t-1}; the
// remaining bits pick the tile.  A CTA reads its tile with the low source bits varying
// fastest into shared memory, then writes it with the low destination bits varying fastest.
constexpr int kPermTileBits = 10;
struct TilePerm {
  int n, T, E;                    // index bits, tile bits, tile-selecting bits
  uint8_t src_s[kPermTileBits];   // source position of tile bit j (ascending)
  uint8_t dst_s[kPermTileBits];   // destination position of the j-th destination tile bit (ascending)
  uint8_t pi[kPermTileBits];      // destination tile bit j carries source tile bit pi[j]
  uint8_t src_e[64], dst_e[64];   // tile-selecting bit k: source / destination position
};

template <typename R>
__global__ void __launch_bounds__(kThreads) k_permute_tiled(const cplx<R>* __restrict__ src,
                                                            cplx<R>* __restrict__ dst, uint64_t n_tiles,
                                                            const TilePerm p) {
  constexpr int kPer = (1 << kPermTileBits) / kThreads;  // elements per thread and tile (4)
  __shared__ cplx<R> tile[1 << kPermTileBits];
  const int size = 1 << p.T;
  // this thread's tile elements: source offsets (read phase) and destination offsets plus the
  // tile slot they come from (write phase), computed once for every tile
  uint64_t soff[kPer], doff[kPer];
  int sslot[kPer], dslot[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int e = threadIdx.x + k * kThreads;
    uint64_t si = 0, di = 0;
    int eo = 0;
    for (int j = 0; j < p.T; ++j) {
      si |= (uint64_t)((e >> j) & 1) << p.src_s[j];
      const int b = (e >> j) & 1;  // as destination tile index f = e
      eo |= b << p.pi[j];
      di |= (uint64_t)b << p.dst_s[j];
    }
    soff[k] = si;
    sslot[k] = e ^ ((e >> 5) & 7);  // xor: spread the 8 x 16 B rows of a later column read
    doff[k] = di;
    dslot[k] = eo ^ ((eo >> 5) & 7);
  }
  for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    uint64_t sb = 0, db = 0;
    for (int k = 0; k < p.E; ++k) {
      const uint64_t b = (t >> k) & 1ull;
      sb |= b << p.src_e[k];
      db |= b << p.dst_e[k];
    }
    cplx<R> v[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if (threadIdx.x + k * kThreads < size) v[k] = src[sb | soff[k]];
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if (threadIdx.x + k * kThreads < size) tile[sslot[k]] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if (threadIdx.x + k * kThreads < size) dst[db | doff[k]] = tile[dslot[k]];
    __syncthreads();
  }
}

// swap a's half with bit=1 and b's half with bit=0 (sharding.py:100-111 _exchange_halves)
template <typename R>
__global__ void __launch_bounds__(kThreads) k_exchange_halves(cplx<R>* __restrict__ a, cplx<R>* __restrict__ b,
                                                              uint64_t half, int bit) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  const uint64_t lowm = (1ull << bit) - 1ull;
  for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e < half; e += stride) {
    const uint64_t base = ((e & ~lowm) << 1) | (e & lowm);
    const uint64_t ia = base | (1ull << bit);
    const cplx<R> t = a[ia];
    a[ia] = b[base];
    b[base] = t;
  }
}

}  // namespace qsb

using namespace qsb;

static int check_dtype(int dtype) {
  if (dtype != QSB_C64 && dtype != QSB_C128) {
    set_error("unknown dtype %d", dtype);
    return QSB_ERR_ARG;
  }
  return QSB_OK;
}

// ------------------------------------------------------------------------------------------
// gate lists in one launch: small states in shared memory, mid-size states grid-synchronised
// ------------------------------------------------------------------------------------------
// Below the fused-pass threshold every gate would otherwise be its own launch of a few
// microseconds.  Up to kBatchMaxGates gates travel as one __grid_constant__ kernel parameter
// (no staging copy; the launch is capturable in a CUDA graph) and run back to back with the
// bodies and operand order of k_general1/k_general2/k_diag/k_perm, so the result has the
// per-gate kernels' bits:
//   * k_small_batch: states <= QSB_BATCH_MAX_STATE_BYTES; one CTA holds the state in shared
//     memory, __syncthreads between gates.
//   * k_grid_batch: states <= QSB_GRID_BATCH_MAX_STATE_BYTES; a co-resident
//     (cooperative) grid walks each gate over global memory with L2-only loads/stores (L1 is not
//     coherent across SMs) and a grid barrier between gates.
constexpr int kSmallThreads = 512;
constexpr int kGridThreads = 256;
constexpr int kBatchMaxGates = 64;

template <typename R>
struct SmallBatch {
  int n_amps;
  int n_gates;
  uint8_t body[kBatchMaxGates];
  GateArgs<R> g[kBatchMaxGates];
};

// shared memory: plain accesses; global memory: cache-global (L2) accesses
template <bool kGlobal, typename C>
__device__ __forceinline__ C bload(const C* p) {
  if constexpr (kGlobal) return __ldcg(p);
  else return *p;
}
template <bool kGlobal, typename C>
__device__ __forceinline__ void bstore(C* p, C v) {
  if constexpr (kGlobal) __stcg(p, v);
  else *p = v;
}

// one group of one gate (the bodies of k_general1 / k_general2 / k_diag / k_perm)
template <bool kGlobal, typename R, typename I>
__device__ __forceinline__ void gate_group(cplx<R>* s, const GateArgs<R>& p, int body, I base) {
  using C = cplx<R>;
  if (body == kBodyGeneral1) {
    const I o1 = base | (I)p.off[1];
    const C x0 = bload<kGlobal>(s + base), x1 = bload<kGlobal>(s + o1);
    bstore<kGlobal>(s + base, cmad(p.m[1], x1, cmul(p.m[0], x0)));
    bstore<kGlobal>(s + o1, cmad(p.m[3], x1, cmul(p.m[2], x0)));
  } else if (body == kBodyGeneral2) {
    C x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = bload<kGlobal>(s + (base | (I)p.off[j]));
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      C y = cmul(p.m[4 * r], x[0]);
      y = cmad(p.m[4 * r + 1], x[1], y);
      y = cmad(p.m[4 * r + 2], x[2], y);
      y = cmad(p.m[4 * r + 3], x[3], y);
      bstore<kGlobal>(s + (base | (I)p.off[r]), y);
    }
  } else if (body == kBodyDiag) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (r < p.nrows) {
        C* q = s + (base | (I)p.off[p.rows[r]]);
        bstore<kGlobal>(q, cmul(bload<kGlobal>(q), p.m[r]));
      }
    }
  } else {  // permutation: gather every moved row, then scatter
    C x[4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (r < p.nrows) x[r] = bload<kGlobal>(s + (base | (I)p.off[p.src[r]]));
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (r < p.nrows) {
        C v = x[r];
        if (p.use_phase & (1u << r)) v = cmul(v, p.m[r]);
        bstore<kGlobal>(s + (base | (I)p.off[p.rows[r]]), v);
      }
    }
  }
}

template <typename R>
__global__ void __launch_bounds__(kSmallThreads, 1)
    k_small_batch(cplx<R>* __restrict__ a, const __grid_constant__ SmallBatch<R> b) {
  using C = cplx<R>;
  extern __shared__ __align__(16) unsigned char small_smem[];
  C* s = reinterpret_cast<C*>(small_smem);
  for (int i = threadIdx.x; i < b.n_amps; i += kSmallThreads) s[i] = a[i];
  __syncthreads();
  for (int k = 0; k < b.n_gates; ++k) {
    const GateArgs<R>& p = b.g[k];
    const int body = b.body[k];
    const uint32_t ng = (uint32_t)p.n_groups;
    for (uint32_t g = threadIdx.x; g < ng; g += kSmallThreads)
      gate_group<false, R, uint32_t>(s, p, body, (uint32_t)(insert_zero_bits(g, p.occ) | p.cmask));
    __syncthreads();
  }
  for (int i = threadIdx.x; i < b.n_amps; i += kSmallThreads) a[i] = s[i];
}

// Sense-by-generation grid barrier on two words {arrived, generation}; the grid is co-resident
// (cooperative launch).  Each launch gets its own slot, so launches on different streams never
// share one.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned n_blocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == n_blocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

template <typename R>
__global__ void __launch_bounds__(kGridThreads)
    k_grid_batch(cplx<R>* a, const __grid_constant__ SmallBatch<R> b, unsigned* bar) {
  const uint32_t tid = blockIdx.x * kGridThreads + threadIdx.x;
  const uint32_t nth = gridDim.x * kGridThreads;
  for (int k = 0; k < b.n_gates; ++k) {
    const GateArgs<R>& p = b.g[k];
    const int body = b.body[k];
    const uint32_t ng = (uint32_t)p.n_groups;
    for (uint32_t g = tid; g < ng; g += nth)
      gate_group<true, R, uint64_t>(a, p, body, insert_zero_bits(g, p.occ) | p.cmask);
    if (k + 1 < b.n_gates) grid_barrier(bar, gridDim.x);
  }
}

static int validate_gate(int n_qubits, int n_targets, const int* target_bits, int n_controls,
                         const int* control_bits) {
  if (n_targets < 1 || n_targets > kMaxWideTargets) {
    set_error("apply_matrix supports 1 to %d targets, got %d", kMaxWideTargets, n_targets);
    return QSB_ERR_SHAPE;
  }
  if (n_qubits < 1 || n_qubits > 40 || n_controls < 0 || n_targets + n_controls > n_qubits) {
    set_error("bad qubit counts (n=%d, targets=%d, controls=%d)", n_qubits, n_targets, n_controls);
    return QSB_ERR_SHAPE;
  }
  uint64_t seen = 0;
  for (int i = 0; i < n_targets + n_controls; ++i) {
    const int b = i < n_targets ? target_bits[i] : control_bits[i - n_targets];
    if (b < 0 || b >= n_qubits) {
      set_error("bit %d out of range for %d qubits", b, n_qubits);
      return QSB_ERR_SHAPE;
    }
    if (seen & (1ull << b)) {
      set_error("targets and controls must be distinct");
      return QSB_ERR_SHAPE;
    }
    seen |= 1ull << b;
  }
  return QSB_OK;
}

constexpr int kBarrierSlots = 256;

template <typename R>
static int launch_batch(void* amps, int n_qubits, int n_gates, const int* n_targets, const int* target_bits,
                        const int* n_controls, const int* control_bits, const double* matrices,
                        const int* kernels, cudaStream_t st) {
  // per-device, per-precision setup (function attribute, grid size, barrier slots), once
  constexpr int kMaxDevices = 64;
  static std::mutex mu;
  static bool smem_set[kMaxDevices] = {};
  static int grid_blocks[kMaxDevices] = {};  // full co-resident grid
  static unsigned* barriers[kMaxDevices] = {};  // kBarrierSlots x {arrived, generation}
  static std::atomic<unsigned> next_slot{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "qsb_apply_batch(device)");
  if (dev < 0 || dev >= kMaxDevices) {
    set_error("apply_batch: device %d out of range", dev);
    return QSB_ERR_ARG;
  }
  const size_t bytes = sizeof(cplx<R>) << n_qubits;
  const bool in_smem = bytes <= QSB_BATCH_MAX_STATE_BYTES;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (in_smem && !smem_set[dev]) {
      e = cudaFuncSetAttribute(k_small_batch<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               QSB_BATCH_MAX_STATE_BYTES);
      if (e != cudaSuccess) return cuda_status(e, "qsb_apply_batch(smem attribute)");
      smem_set[dev] = true;
    }
    if (!in_smem && grid_blocks[dev] == 0) {
      int sms = 0, per_sm = 0;
      e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_grid_batch<R>, kGridThreads, 0);
      if (e == cudaSuccess) e = cudaMalloc(&barriers[dev], sizeof(unsigned) * 2 * kBarrierSlots);
      if (e == cudaSuccess) e = cudaMemset(barriers[dev], 0, sizeof(unsigned) * 2 * kBarrierSlots);
      if (e != cudaSuccess) return cuda_status(e, "qsb_apply_batch(grid setup)");
      grid_blocks[dev] = sms * (per_sm < 1 ? 1 : per_sm);
    }
  }
  // ~27 KB gate table: off the host stack, one per calling thread (ctypes drops the GIL)
  static thread_local SmallBatch<R> b;
  b.n_amps = 1 << n_qubits;
  b.n_gates = 0;
  cplx<R>* a = static_cast<cplx<R>*>(amps);
  auto flush = [&]() -> int {
    if (in_smem) {
      k_small_batch<R><<<1, kSmallThreads, bytes, st>>>(a, b);
    } else {
      unsigned* bar = barriers[dev] + 2 * (next_slot.fetch_add(1) % kBarrierSlots);
      uint64_t widest = b.g[0].n_groups;  // the widest gate bounds the useful grid
      for (int k = 1; k < b.n_gates; ++k) widest = b.g[k].n_groups > widest ? b.g[k].n_groups : widest;
      uint64_t want = (widest + kGridThreads - 1) / kGridThreads;
      // the full co-resident grid (measured: capping it at two CTAs per SM for L2-resident
      // states does not shorten the ~3 us per-gate floor and loses bandwidth at 64 MB+)
      const int cap = grid_blocks[dev];
      const int blocks = (int)(want < (uint64_t)cap ? (want < 1 ? 1 : want) : cap);
      void* args[] = {(void*)&a, (void*)&b, (void*)&bar};
      cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_grid_batch<R>, dim3(blocks), dim3(kGridThreads),
                                                  args, 0, st);
      if (e != cudaSuccess) return cuda_status(e, "qsb_apply_batch(cooperative launch)");
    }
    QSB_CHECK_LAUNCH("qsb_apply_batch");
    b.n_gates = 0;
    return QSB_OK;
  };
  int coff = 0;
  for (int i = 0; i < n_gates; ++i) {
    int kc = kernels[i];
    if (kc == QSB_KERNEL_AUTO) kc = qsb_classify(matrices + 32 * i, n_targets[i]);
    const int body = prepare_gate<R>(n_qubits, n_targets[i], target_bits + 2 * i, n_controls[i], control_bits + coff,
                                     matrices + 32 * i, kc, b.g[b.n_gates]);
    coff += n_controls[i];
    if (body == kBodyNone) continue;
    b.body[b.n_gates++] = (uint8_t)body;
    if (b.n_gates == kBatchMaxGates)
      if (int s = flush()) return s;
  }
  if (b.n_gates)
    if (int s = flush()) return s;
  return QSB_OK;
}

extern "C" {

int qsb_abi_version(void) { return QSB_ABI_VERSION; }
const char* qsb_last_error(void) { return g_err; }

int qsb_init_basis(void* amps, int n_qubits, int dtype, uint64_t basis_index, void* stream) {
  if (int s = check_dtype(dtype)) return s;
  if (n_qubits < 1 || n_qubits > 40) {
    set_error("n_qubits %d out of range", n_qubits);
    return QSB_ERR_CAPACITY;
  }
  const uint64_t n = 1ull << n_qubits;
  if (basis_index >= n) {
    set_error("basis index %llu out of range", (unsigned long long)basis_index);
    return QSB_ERR_SHAPE;
  }
  cudaStream_t st = as_stream(stream);
  const size_t bytes = n * (dtype == QSB_C128 ? 16 : 8);
  cudaError_t e = cudaMemsetAsync(amps, 0, bytes, st);
  if (e != cudaSuccess) return cuda_status(e, "qsb_init_basis(memset)");
  if (dtype == QSB_C128)
    k_set_one<double><<<1, 1, 0, st>>>(static_cast<double2*>(amps), basis_index);
  else
    k_set_one<float><<<1, 1, 0, st>>>(static_cast<float2*>(amps), basis_index);
  QSB_CHECK_LAUNCH("qsb_init_basis");
  return QSB_OK;
}

int qsb_init_uniform(void* amps, int n_qubits, int dtype, double re, double im, void* stream) {
  if (int s = check_dtype(dtype)) return s;
  if (n_qubits < 1 || n_qubits > 40) {
    set_error("n_qubits %d out of range", n_qubits);
    return QSB_ERR_CAPACITY;
  }
  const uint64_t n = 1ull << n_qubits;
  cudaStream_t st = as_stream(stream);
  if (dtype == QSB_C128)
    k_fill<double><<<stream_grid(n), kThreads, 0, st>>>(static_cast<double2*>(amps), n, re, im);
  else
    k_fill<float><<<stream_grid(n), kThreads, 0, st>>>(static_cast<float2*>(amps), n, (float)re, (float)im);
  QSB_CHECK_LAUNCH("qsb_init_uniform");
  return QSB_OK;
}

int qsb_classify(const double* m, int t) {
  const int dim = 1 << t;
  bool off_nz = false;
  for (int r = 0; r < dim; ++r)
    for (int c = 0; c < dim; ++c)
      if (r != c && is_nonzero(m + 2 * (r * dim + c))) off_nz = true;
  if (!off_nz) return QSB_KERNEL_DIAGONAL;
  for (int r = 0; r < dim; ++r) {
    int row_nz = 0, col_nz = 0;
    for (int c = 0; c < dim; ++c) {
      row_nz += is_nonzero(m + 2 * (r * dim + c));
      col_nz += is_nonzero(m + 2 * (c * dim + r));
    }
    if (row_nz != 1 || col_nz != 1) return QSB_KERNEL_GENERAL;
  }
  for (int k = 0; k < dim * dim; ++k) {
    const double* z = m + 2 * k;
    if (is_nonzero(z) && fabs(hypot(z[0], z[1]) - 1.0) > 1e-12) return QSB_KERNEL_GENERAL;
  }
  return QSB_KERNEL_PERMUTATION;
}

int qsb_apply_matrix(void* amps, int n_qubits, int dtype, int n_targets, const int* target_bits,
                     int n_controls, const int* control_bits, const double* matrix, int kernel,
                     void* stream) {
  if (int s = check_dtype(dtype)) return s;
  if (n_targets < 1 || n_targets > kMaxDenseTargets) {
    set_error("apply_matrix supports 1 to %d targets, got %d", kMaxDenseTargets, n_targets);
    return QSB_ERR_SHAPE;
  }
  if (n_qubits < 1 || n_qubits > 40 || n_controls < 0 || n_targets + n_controls > n_qubits) {
    set_error("bad qubit counts (n=%d, targets=%d, controls=%d)", n_qubits, n_targets, n_controls);
    return QSB_ERR_SHAPE;
  }
  uint64_t seen = 0;
  for (int i = 0; i < n_targets + n_controls; ++i) {
    const int b = i < n_targets ? target_bits[i] : control_bits[i - n_targets];
    if (b < 0 || b >= n_qubits) {
      set_error("bit %d out of range for %d qubits", b, n_qubits);
      return QSB_ERR_SHAPE;
    }
    if (seen & (1ull << b)) {
      set_error("targets and controls must be distinct");
      return QSB_ERR_SHAPE;
    }
    seen |= 1ull << b;
  }
  if (kernel == QSB_KERNEL_AUTO) kernel = qsb_classify(matrix, n_targets);
  if (kernel < 0 || kernel > 2) {
    set_error("unknown kernel class %d", kernel);
    return QSB_ERR_ARG;
  }
  cudaStream_t st = as_stream(stream);
  if (dtype == QSB_C128)
    return launch_gate<double>(amps, n_qubits, n_targets, target_bits, n_controls, control_bits, matrix, kernel, st);
  return launch_gate<float>(amps, n_qubits, n_targets, target_bits, n_controls, control_bits, matrix, kernel, st);
}

int qsb_apply_batch(void* amps, int n_qubits, int dtype, int n_gates, const int* n_targets, const int* target_bits,
                    const int* n_controls, const int* control_bits, const double* matrices, const int* kernels,
                    void* stream) {
  if (int s = check_dtype(dtype)) return s;
  const size_t isz = dtype == QSB_C128 ? 16 : 8;
  if (n_qubits < 1 || n_qubits > 32 || (isz << n_qubits) > QSB_GRID_BATCH_MAX_STATE_BYTES) {
    set_error("apply_batch keeps the state on chip: %d qubits exceed %d bytes", n_qubits,
              QSB_GRID_BATCH_MAX_STATE_BYTES);
    return QSB_ERR_CAPACITY;
  }
  if (n_gates < 0) {
    set_error("negative gate count");
    return QSB_ERR_ARG;
  }
  int coff = 0;
  for (int i = 0; i < n_gates; ++i) {  // validate the whole list before any work is enqueued
    if (int s = validate_gate(n_qubits, n_targets[i], target_bits + 2 * i, n_controls[i], control_bits + coff))
      return s;
    coff += n_controls[i];
    if (kernels[i] < QSB_KERNEL_AUTO || kernels[i] > QSB_KERNEL_PERMUTATION) {
      set_error("unknown kernel class %d", kernels[i]);
      return QSB_ERR_ARG;
    }
  }
  if (n_gates == 0) return QSB_OK;
  cudaStream_t st = as_stream(stream);
  if (dtype == QSB_C128)
    return launch_batch<double>(amps, n_qubits, n_gates, n_targets, target_bits, n_controls, control_bits, matrices,
                                kernels, st);
  return launch_batch<float>(amps, n_qubits, n_gates, n_targets, target_bits, n_controls, control_bits, matrices,
                             kernels, st);
}

int qsb_scale(void* amps, uint64_t n, int dtype, double re, double im, void* stream) {
  if (int s = check_dtype(dtype)) return s;
  cudaStream_t st = as_stream(stream);
  if (dtype == QSB_C128)
    k_scale<double><<<stream_grid(n), kThreads, 0, st>>>(static_cast<double2*>(amps), n, make_double2(re, im));
  else
    k_scale<float><<<stream_grid(n), kThreads, 0, st>>>(static_cast<float2*>(amps), n,
                                                        make_float2((float)re, (float)im));
  QSB_CHECK_LAUNCH("qsb_scale");
  return QSB_OK;
}

int qsb_expect_terms(const void* amps, int n_qubits, int dtype, int n_terms, const int* ks, const int* bits,
                     const double* mats, double* out, void* stream) {
  if (int s = check_dtype(dtype)) return s;
  if (n_terms < 0 || (n_terms > 0 && (!ks || !bits || !mats))) {
    set_error("qsb_expect_terms: bad term arrays");
    return QSB_ERR_ARG;
  }
  if (int s = ensure_red_scratch()) return s;
  cudaStream_t st = as_stream(stream);
  double2* part = static_cast<double2*>(g_red_scratch);
  static double2* acc = nullptr;  // running (re, im) over term chunks
  if (!acc) {
    cudaError_t e = cudaMalloc(&acc, 2 * sizeof(double2));
    if (e != cudaSuccess) return cuda_status(e, "expectation accumulator");
  }
  const uint64_t n = 1ull << n_qubits;
  cudaMemsetAsync(out, 0, 2 * sizeof(double), st);
  for (int t0 = 0; t0 < n_terms || (t0 == 0 && n_terms == 0); t0 += kExpMax) {
    ExpTerms T;
    memset(&T, 0, sizeof T);
    T.count = n_terms - t0 < kExpMax ? n_terms - t0 : kExpMax;
    for (int j = 0; j < T.count; ++j) {
      const int t = t0 + j;
      const int k = ks[t];
      if (k != 1 && k != 2) {
        set_error("qsb_expect_terms: terms act on 1 or 2 qubits, got %d", k);
        return QSB_ERR_SHAPE;
      }
      const int hi = bits[2 * t], lo = bits[2 * t + 1];
      if (hi < 0 || hi >= n_qubits || (k == 2 && (lo < 0 || lo >= n_qubits || lo == hi))) {
        set_error("qsb_expect_terms: bad bit positions");
        return QSB_ERR_SHAPE;
      }
      T.t[j].k = k;
      T.t[j].hi = hi;
      T.t[j].lo = k == 2 ? lo : hi;
      memcpy(T.t[j].m, mats + 32 * (size_t)t, sizeof(double) * 2 * (1 << k) * (1 << k));
    }
    if (T.count == 0) break;
    if (dtype == QSB_C128)
      k_expect_partial<double><<<kRedBlocks, kThreads, 0, st>>>(static_cast<const double2*>(amps), n_qubits, T, part);
    else
      k_expect_partial<float><<<kRedBlocks, kThreads, 0, st>>>(static_cast<const float2*>(amps), n_qubits, T, part);
    k_fold<double2><<<1, 1024, 0, st>>>(part, kRedBlocks, acc);
    k_add2<<<1, 1, 0, st>>>(reinterpret_cast<double2*>(out), acc);
  }
  (void)n;
  QSB_CHECK_LAUNCH("qsb_expect_terms");
  return QSB_OK;
}

int qsb_collapse(void* amps, uint64_t n, int dtype, uint64_t mask, uint64_t value, double scale, void* stream) {
  if (int s = check_dtype(dtype)) return s;
  if ((value & ~mask) != 0) {
    set_error("qsb_collapse: value has bits outside the mask");
    return QSB_ERR_ARG;
  }
  cudaStream_t st = as_stream(stream);
  if (dtype == QSB_C128)
    k_collapse<double><<<stream_grid(n), kThreads, 0, st>>>(static_cast<double2*>(amps), n, mask, value, scale);
  else
    k_collapse<float><<<stream_grid(n), kThreads, 0, st>>>(static_cast<float2*>(amps), n, mask, value,
                                                           (float)scale);
  QSB_CHECK_LAUNCH("qsb_collapse");
  return QSB_OK;
}

int qsb_norm2(const void* amps, uint64_t n, int dtype, double* out, void* stream) {
  if (int s = check_dtype(dtype)) return s;
  if (int s = ensure_red_scratch()) return s;
  cudaStream_t st = as_stream(stream);
  double* part = static_cast<double*>(g_red_scratch);
  if (dtype == QSB_C128)
    k_norm2_partial<double><<<kRedBlocks, kThreads, 0, st>>>(static_cast<const double2*>(amps), n, part);
  else
    k_norm2_partial<float><<<kRedBlocks, kThreads, 0, st>>>(static_cast<const float2*>(amps), n, part);
  k_fold<double><<<1, 1024, 0, st>>>(part, kRedBlocks, out);
  QSB_CHECK_LAUNCH("qsb_norm2");
  return QSB_OK;
}

int qsb_vdot(const void* a, const void* b, uint64_t n, int dtype, double* out, void* stream) {
  if (int s = check_dtype(dtype)) return s;
  if (int s = ensure_red_scratch()) return s;
  cudaStream_t st = as_stream(stream);
  double2* part = static_cast<double2*>(g_red_scratch);
  if (dtype == QSB_C128)
    k_vdot_partial<double><<<kRedBlocks, kThreads, 0, st>>>(static_cast<const double2*>(a),
                                                           static_cast<const double2*>(b), n, part);
  else
    k_vdot_partial<float><<<kRedBlocks, kThreads, 0, st>>>(static_cast<const float2*>(a),
                                                          static_cast<const float2*>(b), n, part);
  k_fold<double2><<<1, 1024, 0, st>>>(part, kRedBlocks, reinterpret_cast<double2*>(out));
  QSB_CHECK_LAUNCH("qsb_vdot");
  return QSB_OK;
}

int qsb_permute_qubits(const void* src, void* dst, int n_bits, int dtype, const int* dst_bit, void* stream) {
  if (int s = check_dtype(dtype)) return s;
  if (n_bits < 1 || n_bits > 40) {
    set_error("qsb_permute_qubits: bad size");
    return QSB_ERR_SHAPE;
  }
  BitPerm p;
  p.n = n_bits;
  uint64_t seen = 0;
  int src_of[64];
  for (int b = 0; b < n_bits; ++b) {
    if (dst_bit[b] < 0 || dst_bit[b] >= n_bits || ((seen >> dst_bit[b]) & 1ull)) {
      set_error("qsb_permute_qubits: not a permutation");
      return QSB_ERR_SHAPE;
    }
    seen |= 1ull << dst_bit[b];
    p.dst_bit[b] = (uint8_t)dst_bit[b];
    src_of[dst_bit[b]] = b;
  }
  const uint64_t total = 1ull << n_bits;
  cudaStream_t st = as_stream(stream);
  // tile set: low source bits 0..t-1 and the sources of destination bits 0..t-1, as many as fit
  uint64_t S = 0;
  int t = 0;
  while (t < n_bits) {
    const uint64_t add = (1ull << t) | (1ull << src_of[t]);
    if (__builtin_popcountll(S | add) > kPermTileBits) break;
    S |= add;
    ++t;
  }
  if (t >= 4 && n_bits > kPermTileBits) {
    TilePerm tp;
    tp.n = n_bits;
    tp.T = 0;
    tp.E = 0;
    int idx_of[64];
    for (int b = 0; b < n_bits; ++b) {
      if ((S >> b) & 1ull) {
        idx_of[b] = tp.T;
        tp.src_s[tp.T++] = (uint8_t)b;
      } else {
        tp.src_e[tp.E] = (uint8_t)b;
        tp.dst_e[tp.E++] = (uint8_t)dst_bit[b];
      }
    }
    // destination tile bits in ascending destination order, each with its source tile bit
    int j = 0;
    for (int d = 0; d < n_bits; ++d) {
      const int b = src_of[d];
      if ((S >> b) & 1ull) {
        tp.dst_s[j] = (uint8_t)d;
        tp.pi[j] = (uint8_t)idx_of[b];
        ++j;
      }
    }
    const uint64_t n_tiles = total >> tp.T;
    const int grid = (int)(n_tiles < 148ull * 16ull ? n_tiles : 148ull * 16ull);
    if (dtype == QSB_C128)
      k_permute_tiled<double><<<grid, kThreads, 0, st>>>(static_cast<const double2*>(src), static_cast<double2*>(dst),
                                                         n_tiles, tp);
    else
      k_permute_tiled<float><<<grid, kThreads, 0, st>>>(static_cast<const float2*>(src), static_cast<float2*>(dst),
                                                        n_tiles, tp);
    QSB_CHECK_LAUNCH("qsb_permute_qubits");
    return QSB_OK;
  }
  if (dtype == QSB_C128)
    k_permute<double><<<stream_grid(total), kThreads, 0, st>>>(static_cast<const double2*>(src),
                                                               static_cast<double2*>(dst), total, p);
  else
    k_permute<float><<<stream_grid(total), kThreads, 0, st>>>(static_cast<const float2*>(src),
                                                              static_cast<float2*>(dst), total, p);
  QSB_CHECK_LAUNCH("qsb_permute_qubits");
  return QSB_OK;
}

int qsb_exchange_halves(void* a, void* b, int n_local_bits, int dtype, int bit, void* stream) {
  if (int s = check_dtype(dtype)) return s;
  if (bit < 0 || bit >= n_local_bits) {
    set_error("qsb_exchange_halves: bad bit");
    return QSB_ERR_SHAPE;
  }
  const uint64_t half = 1ull << (n_local_bits - 1);
  cudaStream_t st = as_stream(stream);
  if (dtype == QSB_C128)
    k_exchange_halves<double><<<stream_grid(half), kThreads, 0, st>>>(static_cast<double2*>(a),
                                                                      static_cast<double2*>(b), half, bit);
  else
    k_exchange_halves<float><<<stream_grid(half), kThreads, 0, st>>>(static_cast<float2*>(a),
                                                                     static_cast<float2*>(b), half, bit);
  QSB_CHECK_LAUNCH("qsb_exchange_halves");
  return QSB_OK;
}

int qsb_pack_half(const void* shard, int n_local_bits, int dtype, int bit, int half, uint64_t first,
                  uint64_t count, void* staging, void* stream) {
  if (int s = check_dtype(dtype)) return s;
  if (bit < 0 || bit >= n_local_bits || (half != 0 && half != 1) ||
      first + count > (1ull << (n_local_bits - 1))) {
    set_error("qsb_pack_half: bad bit/half/range");
    return QSB_ERR_SHAPE;
  }
  if (count == 0) return QSB_OK;
  cudaStream_t st = as_stream(stream);
  if (dtype == QSB_C128)
    k_pack_half<double><<<stream_grid(count), kThreads, 0, st>>>(static_cast<const double2*>(shard), bit, half,
                                                                 first, count, static_cast<double2*>(staging));
  else
    k_pack_half<float><<<stream_grid(count), kThreads, 0, st>>>(static_cast<const float2*>(shard), bit, half,
                                                                first, count, static_cast<float2*>(staging));
  QSB_CHECK_LAUNCH("qsb_pack_half");
  return QSB_OK;
}

int qsb_unpack_half(void* shard, int n_local_bits, int dtype, int bit, int half, uint64_t first, uint64_t count,
                    const void* staging, void* stream) {
  if (int s = check_dtype(dtype)) return s;
  if (bit < 0 || bit >= n_local_bits || (half != 0 && half != 1) ||
      first + count > (1ull << (n_local_bits - 1))) {
    set_error("qsb_unpack_half: bad bit/half/range");
    return QSB_ERR_SHAPE;
  }
  if (count == 0) return QSB_OK;
  cudaStream_t st = as_stream(stream);
  if (dtype == QSB_C128)
    k_unpack_half<double><<<stream_grid(count), kThreads, 0, st>>>(static_cast<double2*>(shard), bit, half, first,
                                                                   count, static_cast<const double2*>(staging));
  else
    k_unpack_half<float><<<stream_grid(count), kThreads, 0, st>>>(static_cast<float2*>(shard), bit, half, first,
                                                                  count, static_cast<const float2*>(staging));
  QSB_CHECK_LAUNCH("qsb_unpack_half");
  return QSB_OK;
}

// k local bits (any order) -> sorted OccBits; the part's bit pattern at those positions
static int part_args(int n_local_bits, int k, const int* bits, OccBits* occ, const char* where) {
  if (k < 1 || k > 16 || k >= n_local_bits) {
    set_error("%s: need 1 <= k <= 16 and k < n_local_bits (k=%d)", where, k);
    return QSB_ERR_SHAPE;
  }
  uint64_t seen = 0;
  for (int i = 0; i < k; ++i) {
    if (bits[i] < 0 || bits[i] >= n_local_bits || ((seen >> bits[i]) & 1ull)) {
      set_error("%s: bad or duplicate bit %d", where, bits[i]);
      return QSB_ERR_SHAPE;
    }
    seen |= 1ull << bits[i];
  }
  occ->n = 0;
  for (int b = 0; b < n_local_bits; ++b)
    if ((seen >> b) & 1ull) occ->pos[occ->n++] = (uint8_t)b;
  return QSB_OK;
}

static int check_part_bits(int k, const int* bits, uint64_t part, const char* where) {
  uint64_t mask = 0;
  for (int i = 0; i < k; ++i) mask |= 1ull << bits[i];
  if (part & ~mask) {
    set_error("%s: part bits 0x%llx outside the part positions", where, (unsigned long long)part);
    return QSB_ERR_SHAPE;
  }
  return QSB_OK;
}

int qsb_pack_part(const void* shard, int n_local_bits, int dtype, int k, const int* bits, uint64_t part_bits,
                  uint64_t first, uint64_t count, void* staging, void* stream) {
  if (int s = check_dtype(dtype)) return s;
  OccBits occ;
  if (int s = part_args(n_local_bits, k, bits, &occ, "qsb_pack_part")) return s;
  if (int s = check_part_bits(k, bits, part_bits, "qsb_pack_part")) return s;
  if (first + count > (1ull << (n_local_bits - k))) {
    set_error("qsb_pack_part: range past the part");
    return QSB_ERR_SHAPE;
  }
  if (count == 0) return QSB_OK;
  cudaStream_t st = as_stream(stream);
  if (dtype == QSB_C128)
    k_pack_part<double><<<stream_grid(count), kThreads, 0, st>>>(static_cast<const double2*>(shard), occ, part_bits,
                                                                 first, count, static_cast<double2*>(staging));
  else
    k_pack_part<float><<<stream_grid(count), kThreads, 0, st>>>(static_cast<const float2*>(shard), occ, part_bits,
                                                                first, count, static_cast<float2*>(staging));
  QSB_CHECK_LAUNCH("qsb_pack_part");
  return QSB_OK;
}

int qsb_unpack_part(void* shard, int n_local_bits, int dtype, int k, const int* bits, uint64_t part_bits,
                    uint64_t first, uint64_t count, const void* staging, void* stream) {
  if (int s = check_dtype(dtype)) return s;
  OccBits occ;
  if (int s = part_args(n_local_bits, k, bits, &occ, "qsb_unpack_part")) return s;
  if (int s = check_part_bits(k, bits, part_bits, "qsb_unpack_part")) return s;
  if (first + count > (1ull << (n_local_bits - k))) {
    set_error("qsb_unpack_part: range past the part");
    return QSB_ERR_SHAPE;
  }
  if (count == 0) return QSB_OK;
  cudaStream_t st = as_stream(stream);
  if (dtype == QSB_C128)
    k_unpack_part<double><<<stream_grid(count), kThreads, 0, st>>>(static_cast<double2*>(shard), occ, part_bits,
                                                                   first, count, static_cast<const double2*>(staging));
  else
    k_unpack_part<float><<<stream_grid(count), kThreads, 0, st>>>(static_cast<float2*>(shard), occ, part_bits,
                                                                  first, count, static_cast<const float2*>(staging));
  QSB_CHECK_LAUNCH("qsb_unpack_part");
  return QSB_OK;
}

int qsb_exchange_parts(void* a, void* b, int n_local_bits, int dtype, int k, const int* bits, uint64_t a_bits,
                       uint64_t b_bits, void* stream) {
  if (int s = check_dtype(dtype)) return s;
  OccBits occ;
  if (int s = part_args(n_local_bits, k, bits, &occ, "qsb_exchange_parts")) return s;
  if (int s = check_part_bits(k, bits, a_bits, "qsb_exchange_parts")) return s;
  if (int s = check_part_bits(k, bits, b_bits, "qsb_exchange_parts")) return s;
  if (a == b && a_bits == b_bits) return QSB_OK;
  if (a == b) {
    set_error("qsb_exchange_parts: a part cannot be exchanged within one shard");
    return QSB_ERR_ARG;
  }
  const uint64_t count = 1ull << (n_local_bits - k);
  cudaStream_t st = as_stream(stream);
  if (dtype == QSB_C128)
    k_exchange_parts<double><<<stream_grid(count), kThreads, 0, st>>>(static_cast<double2*>(a), static_cast<double2*>(b),
                                                                      occ, a_bits, b_bits, count);
  else
    k_exchange_parts<float><<<stream_grid(count), kThreads, 0, st>>>(static_cast<float2*>(a), static_cast<float2*>(b),
                                                                     occ, a_bits, b_bits, count);
  QSB_CHECK_LAUNCH("qsb_exchange_parts");
  return QSB_OK;
}

}  // extern "C"
