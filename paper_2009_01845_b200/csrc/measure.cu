// Measurement kernels: probabilities, marginals, the exact sequential CDF and PCG64 sampling.
//
// Reference path: qsim.measurement.sample -> marginal_probabilities
// (/root/reference/pkg/src/qsim/measurement.py:36-87).  Samples must be bit-identical to the
// reference for identical RNG draws, so every step reproduces numpy's floating-point order:
//   probabilities   np.abs(a.astype(c128))**2 == (M*sqrt(fma(r,r,1)))^2
//   marginal        numpy add.reduce: pairwise_sum over the innermost reduced run, sequential
//                   accumulation over the outer rows (App. B.2)
//   cumsum          strictly sequential fl(c + p): reproduced EXACTLY in parallel by the
//                   binade-integer scan below (App. B.3)
//   draws           numpy PCG64 (XSL-RR 128/64), u = (raw >> 11) * 2^-53 (App. B.4)
//   search          np.searchsorted(cum, u, side="right"), clipped (App. B.5)
#include <math.h>
#include <string.h>

#include "qsb_common.cuh"

namespace qsb {

constexpr int kMT = 256;

static int grid_for(uint64_t n, int per = kMT) {
  uint64_t b = (n + per - 1) / per;
  if (b < 1) b = 1;
  if (b > 148ull * 32ull) b = 148ull * 32ull;
  return (int)b;
}

// numpy's SIMD complex absolute value, squared (no contraction: explicit _rn intrinsics)
__device__ __forceinline__ double np_abs2(double re, double im) {
  const double ar = fabs(re), ai = fabs(im);
  const double big = fmax(ar, ai), small = fmin(ar, ai);
  if (big == 0.0) return 0.0;
  const double r = __ddiv_rn(small, big);
  const double h = __dmul_rn(big, __dsqrt_rn(__fma_rn(r, r, 1.0)));
  return __dmul_rn(h, h);
}

template <typename R>
__global__ void __launch_bounds__(kMT) k_probs(const cplx<R>* __restrict__ a, uint64_t n, double* __restrict__ p) {
  const uint64_t stride = (uint64_t)gridDim.x * kMT;
  for (uint64_t i = (uint64_t)blockIdx.x * kMT + threadIdx.x; i < n; i += stride) {
    const cplx<R> v = a[i];
    p[i] = np_abs2((double)v.x, (double)v.y);
  }
}

// ---- numpy pairwise_sum (loops_utils.h: PW_BLOCKSIZE 128, 8-way unroll) -------------------
// Leaf: a run of L <= 128 contiguous doubles.
__device__ __forceinline__ double np_pairwise_leaf(const double* a, int L) {
  if (L < 8) {
    double res = 0.0;
    for (int i = 0; i < L; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < L - (L % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < L; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

// leaf sums of 128-element blocks (rows longer than 128 are power-of-two long, so numpy's
// recursion splits them into a perfect binary tree of 128-element leaves)
// Four leaves per warp: lane 8g + j keeps numpy's accumulator r[j] of leaf g (r[j] = a[j] +
// a[j+8] + ... in order), so every load instruction reads four 64-byte runs (one thread per
// leaf strided its loads 1 KB apart and re-read each sector ~3x from DRAM); the eight
// accumulators then combine as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) through xor shuffles
// (IEEE addition is commutative, so each pair sums to the same bits on both lanes).
__global__ void __launch_bounds__(kMT) k_leaf128(const double* __restrict__ p, uint64_t n_leaves,
                                                 double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 3, j = lane & 7;
  const uint64_t warps = (uint64_t)gridDim.x * (kMT / 32);
  for (uint64_t w = (uint64_t)blockIdx.x * (kMT / 32) + (threadIdx.x >> 5); w * 4 < n_leaves; w += warps) {
    const uint64_t leaf = w * 4 + g;
    const bool valid = leaf < n_leaves;
    const double* a = p + leaf * 128;
    double r = valid ? a[j] : 0.0;
#pragma unroll
    for (int i = 8; i < 128; i += 8) r = __dadd_rn(r, valid ? a[i + j] : 0.0);
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
    if (valid && j == 0) out[leaf] = r;
  }
}

// k_leaf128 straight from the amplitudes: p = numpy's |z|^2 formed in registers (no 2^n
// probability array written and read back), then the same warp-cooperative leaf sums.
template <typename R>
__global__ void __launch_bounds__(kMT) k_leaf128_amps(const cplx<R>* __restrict__ amps, uint64_t n_leaves,
                                                      double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 3, j = lane & 7;
  const uint64_t warps = (uint64_t)gridDim.x * (kMT / 32);
  for (uint64_t w = (uint64_t)blockIdx.x * (kMT / 32) + (threadIdx.x >> 5); w * 4 < n_leaves; w += warps) {
    const uint64_t leaf = w * 4 + g;
    const bool valid = leaf < n_leaves;
    const cplx<R>* a = amps + leaf * 128;
    double r = 0.0;
    if (valid) {
      const cplx<R> v = a[j];
      r = np_abs2((double)v.x, (double)v.y);
    }
#pragma unroll
    for (int i = 8; i < 128; i += 8) {
      double x = 0.0;
      if (valid) {
        const cplx<R> v = a[i + j];
        x = np_abs2((double)v.x, (double)v.y);
      }
      r = __dadd_rn(r, x);
    }
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
    if (valid && j == 0) out[leaf] = r;
  }
}

// one level of the pairwise tree: out[i] = in[2i] + in[2i+1]
__global__ void __launch_bounds__(kMT) k_pair_level(const double* __restrict__ in, uint64_t n_out,
                                                    double* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * kMT;
  for (uint64_t i = (uint64_t)blockIdx.x * kMT + threadIdx.x; i < n_out; i += stride)
    out[i] = __dadd_rn(in[2 * i], in[2 * i + 1]);
}

// rows shorter than or equal to 128: one thread per row
__global__ void __launch_bounds__(kMT) k_row_small(const double* __restrict__ p, uint64_t n_rows, int L,
                                                   double* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * kMT;
  for (uint64_t r = (uint64_t)blockIdx.x * kMT + threadIdx.x; r < n_rows; r += stride)
    out[r] = np_pairwise_leaf(p + r * (uint64_t)L, L);
}

__device__ __forceinline__ uint64_t pdep64(uint64_t x, uint64_t mask) {
  uint64_t r = 0;
  for (uint64_t bb = 1; mask; bb <<= 1) {
    const uint64_t low = mask & (~mask + 1);
    if (x & bb) r |= low;
    mask ^= low;
  }
  return r;
}

// Sequential outer accumulation: out[key] = ((0 + v[row_0]) + v[row_1]) + ... over the rows
// (index = pdep(key, keep) | pdep(j, red)) in increasing j.  `v` is indexed by row.
__global__ void __launch_bounds__(kMT) k_fold_rows(const double* __restrict__ v, uint64_t n_keys,
                                                   uint64_t keep_mask, uint64_t red_mask, uint64_t n_red,
                                                   double* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * kMT;
  for (uint64_t key = (uint64_t)blockIdx.x * kMT + threadIdx.x; key < n_keys; key += stride) {
    const uint64_t kb = pdep64(key, keep_mask);
    double acc = 0.0;
    for (uint64_t j = 0; j < n_red; ++j) acc = __dadd_rn(acc, v[kb | pdep64(j, red_mask)]);
    out[key] = acc;
  }
}

// out[j] = in[src(j)] where output bit b (LSB first) takes compressed-index bit rank[b]:
// reorders the kept bits into the requested qubit order
struct BitRanks {
  int k;
  int8_t rank[48];
};
__global__ void __launch_bounds__(kMT) k_permute_out(const double* __restrict__ in, uint64_t n, const BitRanks br,
                                                     double* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * kMT;
  for (uint64_t j = (uint64_t)blockIdx.x * kMT + threadIdx.x; j < n; j += stride) {
    uint64_t src = 0;
    for (int b = 0; b < br.k; ++b) src |= ((j >> b) & 1ull) << br.rank[b];
    out[j] = in[src];
  }
}

// ---- exact sequential cumsum ---------------------------------------------------------------
// Sequential prefix c_i = fl(c_{i-1} + p_i) with p_i >= 0.  Inside one binade [2^e, 2^(e+1))
// every c is an integer multiple K of u = 2^(e-52), and fl(K*u + p) = (K + d)*u where
// d = round(p/u) with ties broken towards the even K+d -- an integer increment that depends on
// the running K only through its parity.  Such maps K -> K + d[K & 1] compose associatively
// ((D0, D1) pairs), so the sequential sum becomes a parallel integer scan.  Elements whose
// approximate prefix lies near a power of two (or that start a new binade) are "serial": their
// value is computed with a real fl(c + p) by a single stitching thread.  Result is bit-identical
// to the strictly sequential loop.

struct Piece {           // composed map over a run inside one binade
  long long d0, d1;      // increment of K when K is even / odd
  int e;                 // binade exponent of the run (INT_MIN: identity / zero run)
  int pad;
};

__device__ __forceinline__ Piece piece_id() {
  Piece q;
  q.d0 = 0;
  q.d1 = 0;
  q.e = -100000;
  q.pad = 0;
  return q;
}

__device__ __forceinline__ Piece piece_then(const Piece& a, const Piece& b) {
  // apply a, then b (same binade, or one of them the identity)
  Piece r;
  r.e = (a.e != -100000) ? a.e : b.e;
  r.d0 = a.d0 + (((a.d0) & 1) ? b.d1 : b.d0);
  r.d1 = a.d1 + (((1 + a.d1) & 1) ? b.d1 : b.d0);
  r.pad = 0;
  return r;
}

// x * 2^k, exact (power-of-two scaling of a value whose result is normal): one multiply when
// 2^k is a normal double, else the library ldexp
__device__ __forceinline__ double pow2_scale(double x, int k) {
  if (k >= -1022 && k <= 1023) return x * __longlong_as_double((long long)(1023 + k) << 52);
  return ldexp(x, k);
}

__device__ __forceinline__ double piece_apply(const Piece& q, double c) {
  if (q.e == -100000 || (q.d0 == 0 && q.d1 == 0)) return c;
  // K = c / 2^(e-52) exactly
  const long long K = (long long)pow2_scale(c, 52 - q.e);
  const long long K2 = K + ((K & 1) ? q.d1 : q.d0);
  return pow2_scale((double)K2, q.e - 52);
}

// Fast single-thread fallback (also the reference semantics): c_i = fl(c_{i-1} + p_i).
__global__ void k_cumsum_serial(const double* __restrict__ p, uint64_t n, double* __restrict__ c) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    acc = __dadd_rn(acc, p[i]);
    c[i] = acc;
  }
}

constexpr int kScanItems = 16;                 // elements per thread
constexpr int kScanBlock = kMT * kScanItems;   // 4096 elements per block

// Exclusive scan of nb values by one CTA walking chunks of 1024 x 8 (each thread 8 consecutive
// values, a block scan of the thread sums, a running carry): used for the block sums (approximate
// doubles, classification only) and the serial-point counts (exact integers).  In place is fine
// (every value is read before it is written, by the same thread).  Replaces a per-thread
// sequential walk whose strided loads took 0.45 ms at 2^18 blocks.
template <typename T>
__global__ void __launch_bounds__(1024) k_scan_chunked(const T* in, uint64_t nb, T* out, T* total) {
  constexpr int kPer = 8;
  __shared__ T wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  T carry = 0;
  for (uint64_t b0 = 0; b0 < nb; b0 += 1024 * kPer) {
    T x[kPer];
    T sum = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const uint64_t i = b0 + (uint64_t)tid * kPer + k;
      x[k] = i < nb ? in[i] : (T)0;
      sum += x[k];
    }
    T incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
      const T t = wsum[lane];
      T u = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, u, o);
        if (lane >= o) u += y;
      }
      wsum[lane] = u - t;  // exclusive over warps
    }
    __syncthreads();
    T run = carry + wsum[w] + (incl - sum);
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const uint64_t i = b0 + (uint64_t)tid * kPer + k;
      if (i < nb) out[i] = run;
      run += x[k];
    }
    // chunk total: the last thread's inclusive value
    __shared__ T chunk_total;
    if (tid == 1023) chunk_total = run - carry;
    __syncthreads();
    carry += chunk_total;
    __syncthreads();
  }
  if (total && tid == 0) *total = carry;
}


// Binade of an approximate prefix value: -100000 for zero.  "risky" when within `margin`
// (relative) of a power of two or in the subnormal-adjacent range.  The strictly sequential
// prefix of n nonnegative terms differs from the exact one by at most (n-1)*2^-53 relative, the
// approximate (blocked) prefix by far less, so margin = 4 * 2^ceil(log2 n) * 2^-53 (at least
// 2^-40, at most 2^-16) classifies every element whose true prefix could sit on the other side
// of a power of two as serial.
__device__ __forceinline__ int approx_binade(double s, double margin, bool* risky) {
  if (s <= 0.0) {
    *risky = false;
    return -100000;
  }
  const unsigned long long b = (unsigned long long)__double_as_longlong(s);
  const int ef = (int)(b >> 52) & 0x7ff;
  if (ef == 0) {  // subnormal (always risky): exponent from frexp
    int e;
    frexp(s, &e);
    *risky = true;
    return e - 1;
  }
  // s = m2 * 2^e with m2 in [1, 2) taken from the bits (exactly frexp's 2m, e = frexp's e - 1)
  const double m2 = __longlong_as_double((long long)((b & 0x000fffffffffffffull) | 0x3ff0000000000000ull));
  const int e = ef - 1023;
  *risky = (m2 < 1.0 + margin) || (m2 > 2.0 - 2.0 * margin) || (e < -1001);
  return e;  // s in [2^e, 2^(e+1))
}

static double risky_margin(uint64_t n) {
  int lg = 0;
  while ((1ull << lg) < n) ++lg;
  int ex = lg + 2 - 53;
  if (ex < -40) ex = -40;
  if (ex > -16) ex = -16;
  return ldexp(1.0, ex);
}

// piece of one safe element p inside binade e: K -> K + round(p / 2^(e-52)) (ties to even K+d)
__device__ __forceinline__ Piece elem_piece(double p, int e) {
  Piece q;
  q.e = e;
  q.pad = 0;
  if (e == -100000) {  // zero run: p == 0
    q.d0 = 0;
    q.d1 = 0;
    return q;
  }
  const double v = pow2_scale(p, 52 - e);  // p / u, exact (< 2^53)
  const long long mi = __double2ll_rd(v);   // floor
  const double f = v - (double)mi;          // exact
  if (f < 0.5) {
    q.d0 = mi;
    q.d1 = mi;
  } else if (f > 0.5) {
    q.d0 = mi + 1;
    q.d1 = mi + 1;
  } else {
    q.d0 = mi + (mi & 1);
    q.d1 = mi + ((~mi) & 1);
  }
  return q;
}


// Pass D (parallel form): the chain visits every block head, but between two serial points
// every map is a piece of one binade, so the heads of consecutive blocks compose with a
// segmented scan (segments start after blocks that contain serial points).  A single thread
// then walks only the serial points: c = fl(c + p_serial), the serial's after-piece, and (for
// the last serial of a block) the composed heads up to the next serial's block.  Finally
// every block start is its run's start value mapped through the run prefix.
struct SegP {
  Piece p;             // composed heads from the segment start through this block
  unsigned int start;  // first block of the segment
  int flag;            // a segment starts inside the combined range
};

__device__ __forceinline__ SegP seg_then(const SegP& a, const SegP& b) {
  if (b.flag) return b;
  SegP r;
  r.p = piece_then(a.p, b.p);
  r.start = a.start;
  r.flag = a.flag;
  return r;
}

constexpr int kSegPer = 4;                    // blocks per thread
constexpr int kSegCta = kMT * kSegPer;        // blocks per CTA

__device__ __forceinline__ SegP seg_leaf(const Piece* head, const unsigned int* cnt, uint64_t b) {
  SegP v;
  v.p = head[b];
  v.start = (unsigned int)b;
  v.flag = (b == 0 || cnt[b - 1] != 0) ? 1 : 0;
  return v;
}

// per-CTA inclusive segmented scan of block heads; CTA aggregate out
__global__ void __launch_bounds__(kMT) k_seg_local(const Piece* __restrict__ head, const unsigned int* __restrict__ cnt,
                                                   uint64_t nb, SegP* __restrict__ out, SegP* __restrict__ agg) {
  __shared__ SegP sh[kMT];
  const uint64_t b0 = (uint64_t)blockIdx.x * kSegCta + (uint64_t)threadIdx.x * kSegPer;
  SegP v[kSegPer];
  SegP acc;
  bool have = false;
  for (int k = 0; k < kSegPer; ++k) {
    const uint64_t b = b0 + k;
    if (b < nb) {
      v[k] = seg_leaf(head, cnt, b);
      acc = have ? seg_then(acc, v[k]) : v[k];
      have = true;
    }
  }
  if (!have) {
    acc.p = piece_id();
    acc.start = 0;
    acc.flag = 0;
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 1; o < kMT; o <<= 1) {
    SegP x = sh[threadIdx.x];
    if ((int)threadIdx.x >= o) x = seg_then(sh[threadIdx.x - o], x);
    __syncthreads();
    sh[threadIdx.x] = x;
    __syncthreads();
  }
  SegP run;
  bool hrun = threadIdx.x > 0;
  if (hrun) run = sh[threadIdx.x - 1];
  for (int k = 0; k < kSegPer; ++k) {
    const uint64_t b = b0 + k;
    if (b >= nb) break;
    run = hrun ? seg_then(run, v[k]) : v[k];
    hrun = true;
    out[b] = run;
  }
  if (threadIdx.x == kMT - 1) agg[blockIdx.x] = sh[kMT - 1];
}

// exclusive scan of the CTA aggregates (one CTA; serial chunks per thread)
__global__ void __launch_bounds__(kMT) k_seg_top(SegP* __restrict__ agg, uint64_t na) {
  __shared__ SegP sh[kMT];
  const uint64_t per = (na + kMT - 1) / kMT;
  const uint64_t lo = threadIdx.x * per;
  SegP acc;
  bool have = false;
  for (uint64_t i = lo; i < lo + per && i < na; ++i) {
    acc = have ? seg_then(acc, agg[i]) : agg[i];
    have = true;
  }
  if (!have) {
    acc.p = piece_id();
    acc.start = 0;
    acc.flag = 0;
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 1; o < kMT; o <<= 1) {
    SegP x = sh[threadIdx.x];
    if ((int)threadIdx.x >= o) x = seg_then(sh[threadIdx.x - o], x);
    __syncthreads();
    sh[threadIdx.x] = x;
    __syncthreads();
  }
  // rewrite as exclusive prefixes: agg[i] = combination of agg[0..i-1] (only read for i > 0)
  SegP run;
  bool hrun = threadIdx.x > 0;
  if (hrun) run = sh[threadIdx.x - 1];
  for (uint64_t i = lo; i < lo + per && i < na; ++i) {
    const SegP x = agg[i];
    if (hrun) agg[i] = run;
    run = hrun ? seg_then(run, x) : x;
    hrun = true;
  }
}

__global__ void __launch_bounds__(kMT) k_seg_fix(SegP* __restrict__ out, uint64_t nb, const SegP* __restrict__ agg) {
  const uint64_t b = (uint64_t)blockIdx.x * kMT + threadIdx.x;
  if (b >= nb) return;
  const uint64_t c = b / kSegCta;
  if (c == 0) return;
  SegP v = out[b];
  if (!v.flag) out[b] = seg_then(agg[c], v);
}

// the serial walk: only serial points (ns of them, sorted by index)
__global__ void k_stitch_serial(const double* __restrict__ p, uint64_t ns, const unsigned long long* __restrict__ sidx,
                                const Piece* __restrict__ after, const SegP* __restrict__ run,
                                double* __restrict__ serial_val, double* __restrict__ run_start) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  run_start[0] = 0.0;
  if (ns == 0) return;
  unsigned long long b = sidx[0] / kScanBlock;
  double c = piece_apply(run[b].p, 0.0);
  for (uint64_t k = 0; k < ns; ++k) {
    c = __dadd_rn(c, p[sidx[k]]);
    serial_val[k] = c;
    c = piece_apply(after[k], c);
    const unsigned long long bn = (k + 1 < ns) ? sidx[k + 1] / kScanBlock : ~0ull;
    if (bn != b) {  // last serial of block b: the next run starts at block b + 1
      run_start[b + 1] = c;
      if (bn != ~0ull) c = piece_apply(run[bn].p, c);
      b = bn;
    }
  }
}

__global__ void __launch_bounds__(kMT) k_block_starts(const SegP* __restrict__ run, uint64_t nb,
                                                      const double* __restrict__ run_start,
                                                      double* __restrict__ block_start) {
  const uint64_t b = (uint64_t)blockIdx.x * kMT + threadIdx.x;
  if (b >= nb) return;
  const unsigned int s = run[b].start;
  const double c0 = run_start[s];
  block_start[b] = (b == s) ? c0 : piece_apply(run[b - 1].p, c0);
}

// ---- coalesced block kernels (round 1b) -----------------------------------------------------
// Each 4096-element block is loaded with coalesced reads into a padded shared array (row of 16
// elements per thread, stride 17 doubles: at most 2-way bank conflicts), every thread then walks
// its 16 consecutive elements.  The classification (approximate prefix -> binade / risky) is a
// shared device function, so the count, pieces and materialize kernels agree bit for bit.
constexpr int kRow = kScanItems + 1;

__device__ __forceinline__ void load_block(const double* __restrict__ p, uint64_t n, uint64_t b0, double* sh) {
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int j = threadIdx.x + k * kMT;
    const uint64_t i = b0 + j;
    sh[(j / kScanItems) * kRow + (j % kScanItems)] = (i < n) ? p[i] : 0.0;
  }
  __syncthreads();
}

// exclusive block scan of one double per thread (warp shuffles + one warp over warp totals)
__device__ __forceinline__ double block_excl_scan(double v, double* wsum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    double t = (lane < kMT / 32) ? wsum[lane] : 0.0;
    double u = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, u, o);
      if (lane >= o) u += y;
    }
    if (lane < kMT / 32) wsum[lane] = u - t;  // exclusive over warps
  }
  __syncthreads();
  return wsum[w] + (x - v);
}

// per-thread classification of its 16 elements: serial bits and binades
struct RowClass {
  unsigned int serial;  // bit k: element k is serial
  int e[kScanItems];
};

__device__ __forceinline__ void classify_row(const double* row, double s, bool first_elem_of_all, double margin,
                                             uint64_t i0, uint64_t n, RowClass& rc) {
  bool prev_risky = false;
  int prev_e = first_elem_of_all ? -100001 : approx_binade(s, margin, &prev_risky);
  rc.serial = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    s += row[k];
    bool risky;
    const int e = approx_binade(s, margin, &risky);
    const bool ser = risky || prev_risky || (e != prev_e && e != -100000) ||
                     (e == -100000 && prev_e != -100000 && prev_e != -100001);
    if (i0 + k < n && ser) rc.serial |= 1u << k;
    rc.e[k] = e;
    prev_e = e;
    prev_risky = risky;
  }
}

// common prologue: block load + approximate thread prefix + classification
__device__ __forceinline__ void block_classify(const double* __restrict__ p, uint64_t n, double margin,
                                               const double* __restrict__ block_prefix, double* sh, double* wsum,
                                               RowClass& rc, uint64_t& i0) {
  const uint64_t b0 = (uint64_t)blockIdx.x * kScanBlock;
  load_block(p, n, b0, sh);
  const double* row = sh + threadIdx.x * kRow;
  double loc = 0.0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) loc += row[k];
  const double s = block_prefix[blockIdx.x] + block_excl_scan(loc, wsum);
  i0 = b0 + (uint64_t)threadIdx.x * kScanItems;
  classify_row(row, s, i0 == 0, margin, i0, n, rc);
}

__global__ void __launch_bounds__(kMT) k_block_sums2(const double* __restrict__ p, uint64_t n,
                                                     double* __restrict__ block_sum) {
  __shared__ double wsum[kMT / 32];
  const uint64_t b0 = (uint64_t)blockIdx.x * kScanBlock;
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint64_t i = b0 + threadIdx.x + (uint64_t)k * kMT;
    if (i < n) acc += p[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kMT / 32; ++w) t += wsum[w];
    block_sum[blockIdx.x] = t;
  }
}

// numpy |z|^2 of every amplitude (k_probs) and, per 4096-element block, the same approximate
// sum k_block_sums2 forms (same per-thread order, same shuffle tree): the sampling pipeline's
// first two passes in one read of the amplitudes
template <typename R>
__global__ void __launch_bounds__(kMT) k_probs_bsums(const cplx<R>* __restrict__ a, uint64_t n,
                                                     double* __restrict__ p, double* __restrict__ block_sum) {
  __shared__ double wsum[kMT / 32];
  const uint64_t b0 = (uint64_t)blockIdx.x * kScanBlock;
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint64_t i = b0 + threadIdx.x + (uint64_t)k * kMT;
    if (i < n) {
      const cplx<R> v = a[i];
      const double x = np_abs2((double)v.x, (double)v.y);
      p[i] = x;
      acc += x;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kMT / 32; ++w) t += wsum[w];
    block_sum[blockIdx.x] = t;
  }
}


// element segments: a serial element starts a new (empty) segment; V_i = composition of the
// safe elements' pieces since the last serial (or the block start).  Thread rows are combined
// with a segmented scan over (has-serial, tail piece) pairs.
struct RowSeg {
  Piece v;   // composition over the combined range since its last serial (or its start)
  int ser;   // the combined range contains a serial element
};

__device__ __forceinline__ RowSeg rowseg_then(const RowSeg& a, const RowSeg& b) {
  if (b.ser) return b;
  RowSeg r;
  r.v = piece_then(a.v, b.v);
  r.ser = a.ser;
  return r;
}

__device__ __forceinline__ RowSeg rowseg_shfl_up(const RowSeg& x, int o) {
  RowSeg r;
  r.v.d0 = __shfl_up_sync(0xffffffffu, x.v.d0, o);
  r.v.d1 = __shfl_up_sync(0xffffffffu, x.v.d1, o);
  r.v.e = __shfl_up_sync(0xffffffffu, x.v.e, o);
  r.v.pad = 0;
  r.ser = __shfl_up_sync(0xffffffffu, x.ser, o);
  return r;
}

// exclusive segmented scan of one RowSeg per thread: warp shuffles, then one warp over the
// warp aggregates (combination order is the serial order, so results equal a serial walk)
__device__ RowSeg block_excl_rowseg(RowSeg mine, RowSeg* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  RowSeg x = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const RowSeg y = rowseg_shfl_up(x, o);
    if (lane >= o) x = rowseg_then(y, x);
  }
  if (lane == 31) sh[w] = x;  // warp aggregate
  __syncthreads();
  if (w == 0) {
    RowSeg t;
    if (lane < kMT / 32) {
      t = sh[lane];
    } else {
      t.v = piece_id();
      t.ser = 0;
    }
    RowSeg u = t;
#pragma unroll
    for (int o = 1; o < kMT / 32; o <<= 1) {
      const RowSeg y = rowseg_shfl_up(u, o);
      if (lane >= o) u = rowseg_then(y, u);
    }
    if (lane < kMT / 32) sh[kMT / 32 + lane] = u;  // inclusive over warps
  }
  __syncthreads();
  // exclusive value for this thread: (warps before) then (lanes before in this warp)
  RowSeg in_warp = rowseg_shfl_up(x, 1);
  RowSeg ex;
  const bool have_w = w > 0;
  const bool have_l = lane > 0;
  if (have_w && have_l) ex = rowseg_then(sh[kMT / 32 + w - 1], in_warp);
  else if (have_w) ex = sh[kMT / 32 + w - 1];
  else if (have_l) ex = in_warp;
  else {
    ex.v = piece_id();
    ex.ser = 0;
  }
  __syncthreads();
  return ex;
}

__device__ __forceinline__ unsigned int block_excl_count(unsigned int c, unsigned int* wsum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned int x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int run = 0;
    for (int k = 0; k < kMT / 32; ++k) {
      const unsigned int t = wsum[k];
      wsum[k] = run;
      run += t;
    }
  }
  __syncthreads();
  const unsigned int r = wsum[w] + (x - c);
  __syncthreads();
  return r;
}

// kLocal: the serial points' indices and after-pieces go to per-block lists of kSerCap entries
// (block-local slots; cnt[b] = the block's serial count, *overflow set when a block has more) and
// are compacted after the count scan -- the count pass then needs no classification of its own.
// !kLocal: straight into the global lists at serial_base[b] + local slot (after a count pass).
constexpr unsigned int kSerCap = 16;

template <bool kLocal>
__global__ void __launch_bounds__(kMT, 3) k_pieces2(const double* __restrict__ p, uint64_t n, double margin,
                                                 const double* __restrict__ block_prefix,
                                                 const unsigned int* __restrict__ serial_base,
                                                 Piece* __restrict__ head, Piece* __restrict__ after,
                                                 unsigned long long* __restrict__ serial_idx,
                                                 unsigned int* __restrict__ cnt, unsigned int* __restrict__ overflow) {
  // !kLocal with cnt given: only the blocks whose serial points overflowed their local lists
  if (!kLocal && cnt && cnt[blockIdx.x] <= kSerCap) return;
  __shared__ double sh[kMT * kRow];
  __shared__ double wsum[kMT / 32];
  __shared__ unsigned int usum[kMT / 32];
  __shared__ RowSeg ssh[kMT];
  RowClass rc;
  uint64_t i0;
  block_classify(p, n, margin, block_prefix, sh, wsum, rc, i0);
  const double* row = sh + threadIdx.x * kRow;
  // thread-local segment of the row (pieces after the last serial in the row)
  RowSeg mine;
  mine.v = piece_id();
  mine.ser = rc.serial ? 1 : 0;
  const int last_ser = rc.serial ? 31 - __clz(rc.serial) : -1;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (k > last_ser && i0 + k < n) mine.v = piece_then(mine.v, elem_piece(row[k], rc.e[k]));
  const RowSeg in = block_excl_rowseg(mine, ssh);
  const unsigned int nser = __popc(rc.serial);
  const unsigned int slot0 = (kLocal ? 0u : serial_base[blockIdx.x]) + block_excl_count(nser, usum);
  if (kLocal && threadIdx.x == kMT - 1) {
    cnt[blockIdx.x] = slot0 + nser;
    if (slot0 + nser > kSerCap) atomicOr(overflow, 1u);
  }
  const uint64_t lbase = kLocal ? (uint64_t)blockIdx.x * kSerCap : 0;
  // walk the row: V = running segment value; at segment ends write head / after
  if (threadIdx.x == 0 && (rc.serial & 1u)) head[blockIdx.x] = piece_id();  // empty head segment
  Piece V = in.v;
  bool seen = in.ser;              // a serial precedes the current element inside the block
  unsigned int slot = slot0;       // slot of the next serial; the current segment's is slot - 1
  const uint64_t bend = min((uint64_t)(blockIdx.x + 1) * kScanBlock, n);
  if (rc.serial == 0) {
    // no serial in the row (nearly every row): the only segment end inside it is the block's
    // last element, and the value there is the incoming segment composed with the whole row
    V = piece_then(V, mine.v);
    if (i0 < bend && bend - 1 - i0 < (uint64_t)kScanItems) {
      if (seen) { if (!kLocal || slot - 1 < kSerCap) after[lbase + slot - 1] = V; }
      else head[blockIdx.x] = V;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const uint64_t i = i0 + k;
      if (i >= n) break;
      if ((rc.serial >> k) & 1u) {
        if (!kLocal || slot < kSerCap) serial_idx[lbase + slot] = i;
        ++slot;
        seen = true;
        V = piece_id();
      } else {
        V = piece_then(V, elem_piece(row[k], rc.e[k]));
      }
      bool end = (i + 1 == bend);
      if (!end) {
        // next element serial?  within the row use the bits, else the next thread's first bit
        end = (k + 1 < kScanItems) ? ((rc.serial >> (k + 1)) & 1u) != 0 : false;
      }
      if (end) {
        if (seen) { if (!kLocal || slot - 1 < kSerCap) after[lbase + slot - 1] = V; }
        else head[blockIdx.x] = V;
      }
    }
  }
  // the row's last element ends a segment when the next row starts with a serial
  __shared__ unsigned int first_bits[kMT];
  first_bits[threadIdx.x] = rc.serial & 1u;
  __syncthreads();
  const bool next_ser = (threadIdx.x + 1 < kMT) ? first_bits[threadIdx.x + 1] != 0 : false;
  const uint64_t ilast = i0 + kScanItems - 1;
  if (next_ser && ilast < n && ilast + 1 != bend) {
    if (seen) { if (!kLocal || slot - 1 < kSerCap) after[lbase + slot - 1] = V; }
    else head[blockIdx.x] = V;
  }
}

// per-block serial lists -> the global lists at the scanned bases (kLocal pieces pass)
__global__ void __launch_bounds__(32) k_compact_serials(const unsigned int* __restrict__ cnt,
                                                        const unsigned int* __restrict__ base,
                                                        const Piece* __restrict__ loc_after,
                                                        const unsigned long long* __restrict__ loc_idx,
                                                        Piece* __restrict__ after,
                                                        unsigned long long* __restrict__ serial_idx) {
  const unsigned int c = cnt[blockIdx.x];
  if (c > kSerCap) return;  // an overflowing block: its own pieces pass writes the global lists
  const uint64_t lb = (uint64_t)blockIdx.x * kSerCap;
  for (unsigned int j = threadIdx.x; j < c; j += 32) {
    after[base[blockIdx.x] + j] = loc_after[lb + j];
    serial_idx[base[blockIdx.x] + j] = loc_idx[lb + j];
  }
}

// total = c[n-1]: the final segment's value (the last block's head, or the last serial's)
__global__ void k_total2(const Piece* __restrict__ head, const unsigned int* __restrict__ cnt, uint64_t nb,
                         const double* __restrict__ block_start, const Piece* __restrict__ after,
                         const double* __restrict__ serial_val, uint64_t ns, double* __restrict__ total) {
  if (threadIdx.x || blockIdx.x) return;
  if (cnt[nb - 1] == 0)
    *total = piece_apply(head[nb - 1], block_start[nb - 1]);
  else
    *total = piece_apply(after[ns - 1], serial_val[ns - 1]);
}

// materialize + normalise: c_i / c_{n-1}, written coalesced through the padded shared row
// Sparse sampling, pass E': the exact value before every row of 16 elements (the row start) of
// the flagged blocks -- the materialise prologue without its per-element walk.  A draw then
// finds its row by the row starts and walks at most 16 elements with fl(c + p) from the row's
// exact start, which is the sequential cumsum itself (k_draw_rows).
__global__ void __launch_bounds__(kMT, 3) k_row_starts(const double* __restrict__ p, uint64_t n, double margin,
                                                    const double* __restrict__ block_prefix,
                                                    const unsigned int* __restrict__ serial_base,
                                                    const double* __restrict__ block_start,
                                                    const double* __restrict__ serial_val,
                                                    double* __restrict__ rs, const unsigned char* __restrict__ only) {
  if (!only[blockIdx.x]) return;
  __shared__ double sh[kMT * kRow];
  __shared__ double wsum[kMT / 32];
  __shared__ unsigned int usum[kMT / 32];
  __shared__ RowSeg ssh[kMT];
  RowClass rc;
  uint64_t i0;
  block_classify(p, n, margin, block_prefix, sh, wsum, rc, i0);
  const double* row = sh + threadIdx.x * kRow;
  RowSeg mine;
  mine.v = piece_id();
  mine.ser = rc.serial ? 1 : 0;
  const int last_ser = rc.serial ? 31 - __clz(rc.serial) : -1;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (k > last_ser && i0 + k < n) mine.v = piece_then(mine.v, elem_piece(row[k], rc.e[k]));
  const RowSeg in = block_excl_rowseg(mine, ssh);
  const unsigned int slot0 = serial_base[blockIdx.x] + block_excl_count(__popc(rc.serial), usum);
  // c before the row's first element: the incoming segment applied to its start value (the last
  // serial before the row, or the block start)
  const double c0 = in.ser ? serial_val[slot0 - 1] : block_start[blockIdx.x];
  rs[(uint64_t)blockIdx.x * kMT + threadIdx.x] = piece_apply(in.v, c0);
}

__global__ void __launch_bounds__(kMT, 3) k_materialize2(const double* __restrict__ p, uint64_t n, double margin,
                                                      const double* __restrict__ block_prefix,
                                                      const unsigned int* __restrict__ serial_base,
                                                      const double* __restrict__ block_start,
                                                      const double* __restrict__ serial_val,
                                                      const double* __restrict__ total,
                                                      double* __restrict__ c_out, int normalize,
                                                      const unsigned char* __restrict__ only) {
  // only != nullptr: materialise just the blocks flagged there (the blocks that hold a draw)
  if (only && !only[blockIdx.x]) return;
  __shared__ double sh[kMT * kRow];
  __shared__ double wsum[kMT / 32];
  __shared__ unsigned int usum[kMT / 32];
  __shared__ RowSeg ssh[kMT];
  RowClass rc;
  uint64_t i0;
  block_classify(p, n, margin, block_prefix, sh, wsum, rc, i0);
  double* row = sh + threadIdx.x * kRow;
  RowSeg mine;
  mine.v = piece_id();
  mine.ser = rc.serial ? 1 : 0;
  const int last_ser = rc.serial ? 31 - __clz(rc.serial) : -1;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (k > last_ser && i0 + k < n) mine.v = piece_then(mine.v, elem_piece(row[k], rc.e[k]));
  const RowSeg in = block_excl_rowseg(mine, ssh);
  const unsigned int slot0 = serial_base[blockIdx.x] + block_excl_count(__popc(rc.serial), usum);
  const double tot = *total;
  // start value of the current segment
  double c0 = in.ser ? serial_val[slot0 - 1] : block_start[blockIdx.x];
  Piece V = in.v;
  unsigned int slot = slot0;
  // the row is private to this thread: each element's result replaces its probability in place
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    double c;
    if ((rc.serial >> k) & 1u) {
      c = serial_val[slot++];
      c0 = c;
      V = piece_id();
    } else {
      V = piece_then(V, elem_piece(row[k], rc.e[k]));
      c = piece_apply(V, c0);
    }
    row[k] = normalize ? __ddiv_rn(c, tot) : c;
  }
  __syncthreads();
  const uint64_t b0 = (uint64_t)blockIdx.x * kScanBlock;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int j = threadIdx.x + k * kMT;
    const uint64_t i = b0 + j;
    if (i < n) c_out[i] = sh[(j / kScanItems) * kRow + (j % kScanItems)];
  }
}


// total is read from a separate copy: c[n-1] itself is overwritten by the normalisation
// ---- PCG64 ---------------------------------------------------------------------------------
typedef unsigned __int128 u128;
__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}
__device__ __forceinline__ uint64_t pcg_out(u128 s) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const unsigned rot = (unsigned)(hi >> 58);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64 - rot) & 63));
}
// LCG jump-ahead by `delta` steps
__device__ u128 pcg_advance(u128 s, u128 inc, uint64_t delta) {
  u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * s + acc_plus;
}

constexpr int kShotsPerThread = 32;

__global__ void __launch_bounds__(kMT) k_sample(const double* __restrict__ cum, uint64_t n, uint64_t s_hi,
                                                uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, uint64_t n_shots,
                                                long long* __restrict__ out, uint64_t clip_max) {
  const uint64_t t = (uint64_t)blockIdx.x * kMT + threadIdx.x;
  const uint64_t first = t * kShotsPerThread;
  if (first >= n_shots) return;
  const u128 inc = ((u128)i_hi << 64) | i_lo;
  u128 s = pcg_advance(((u128)s_hi << 64) | s_lo, inc, first);
  const u128 mult = pcg_mult();
  for (int k = 0; k < kShotsPerThread; ++k) {
    const uint64_t shot = first + k;
    if (shot >= n_shots) break;
    s = s * mult + inc;
    const double u = (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
    // upper_bound: number of cum[i] <= u
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t mid = lo + ((hi - lo) >> 1);
      if (cum[mid] <= u)
        lo = mid + 1;
      else
        hi = mid;
    }
    uint64_t idx = lo;
    if (idx > clip_max) idx = clip_max;
    out[shot] = (long long)idx;
  }
}

}  // namespace qsb

using namespace qsb;

extern "C" {

int qsb_probabilities(const void* amps, uint64_t n, int dtype, double* probs, void* stream) {
  cudaStream_t st = as_stream(stream);
  if (dtype == QSB_C128)
    k_probs<double><<<grid_for(n), kMT, 0, st>>>(static_cast<const double2*>(amps), n, probs);
  else if (dtype == QSB_C64)
    k_probs<float><<<grid_for(n), kMT, 0, st>>>(static_cast<const float2*>(amps), n, probs);
  else {
    set_error("unknown dtype %d", dtype);
    return QSB_ERR_ARG;
  }
  QSB_CHECK_LAUNCH("qsb_probabilities");
  return QSB_OK;
}

}  // extern "C"

// Marginal with explicit output order.  `kept` lists the kept bit positions in output order
// (kept[0] = most significant output bit).  scratch: qsb_marginal_scratch_doubles() doubles.
extern "C" uint64_t qsb_marginal_scratch_doubles(int n_bits, int k) {
  return (1ull << k) + (1ull << (n_bits - 1)) + 256;
}

static int marginal_impl(const double* probs, const void* amps, int dtype, int n_bits, int k, const int* kept,
                         double* out, double* scratch, cudaStream_t st);

extern "C" int qsb_marginal(const double* probs, int n_bits, int k, const int* kept, double* out, double* scratch,
                            void* stream) {
  return marginal_impl(probs, nullptr, 0, n_bits, k, kept, out, scratch, as_stream(stream));
}

extern "C" int qsb_marginal_amps(const void* amps, int dtype, int n_bits, int k, const int* kept, double* out,
                                 double* scratch, void* stream) {
  if (dtype != QSB_C128 && dtype != QSB_C64) {
    set_error("unknown dtype %d", dtype);
    return QSB_ERR_ARG;
  }
  return marginal_impl(nullptr, amps, dtype, n_bits, k, kept, out, scratch, as_stream(stream));
}

static int marginal_impl(const double* probs, const void* amps, int dtype, int n_bits, int k, const int* kept,
                         double* out, double* scratch, cudaStream_t st) {
  if (n_bits < 1 || n_bits > 40 || k < 1 || k > n_bits) {
    set_error("qsb_marginal: bad sizes (n=%d, k=%d)", n_bits, k);
    return QSB_ERR_SHAPE;
  }
  uint64_t keep = 0;
  for (int i = 0; i < k; ++i) {
    if (kept[i] < 0 || kept[i] >= n_bits || ((keep >> kept[i]) & 1ull)) {
      set_error("qsb_marginal: bad kept bit");
      return QSB_ERR_SHAPE;
    }
    keep |= 1ull << kept[i];
  }
  const uint64_t N = 1ull << n_bits;
  const uint64_t red = (N - 1) & ~keep;
  const uint64_t n_keys = 1ull << k;
  const double* asc = scratch;  // 2^k, ascending kept-bit order
  double* work = scratch + n_keys;
  if (amps) {  // the fused form exists for the leaf branch only: >= 8 low bits reduced
    int r = 0;
    while (r < n_bits && ((red >> r) & 1ull)) ++r;
    if (r < 8) {
      set_error("qsb_marginal_amps: needs the 8 lowest bits reduced (use qsb_probabilities + qsb_marginal)");
      return QSB_ERR_ARG;
    }
  }
  if (red == 0) {
    asc = probs;
  } else if (red & 1ull) {
    // innermost run of reduced bits [0, r): numpy pairwise_sum per row
    int r = 0;
    while (r < n_bits && ((red >> r) & 1ull)) ++r;
    const uint64_t L = 1ull << r;
    const uint64_t rows = N >> r;
    const double* rowsum = work;
    if (L <= 128) {
      k_row_small<<<grid_for(rows), kMT, 0, st>>>(probs, rows, (int)L, work);
    } else {
      const uint64_t leaves = N / 128;
      double* a = work;
      double* b = work + leaves;
      if (!amps)
        k_leaf128<<<grid_for(leaves), kMT, 0, st>>>(probs, leaves, a);
      else if (dtype == QSB_C128)
        k_leaf128_amps<double><<<grid_for(leaves), kMT, 0, st>>>(static_cast<const double2*>(amps), leaves, a);
      else
        k_leaf128_amps<float><<<grid_for(leaves), kMT, 0, st>>>(static_cast<const float2*>(amps), leaves, a);
      uint64_t cur = leaves;
      while (cur > rows) {
        k_pair_level<<<grid_for(cur / 2), kMT, 0, st>>>(a, cur / 2, b);
        double* tmp = a;
        a = b;
        b = tmp;
        cur /= 2;
      }
      rowsum = a;
    }
    // sequential accumulation over the outer reduced rows with equal kept bits
    const uint64_t keep_row = keep >> r, red_row = red >> r;
    const uint64_t n_red = 1ull << __builtin_popcountll(red_row);
    k_fold_rows<<<grid_for(n_keys), kMT, 0, st>>>(rowsum, n_keys, keep_row, red_row, n_red, scratch);
  } else {
    // innermost run kept: element-wise sequential accumulation over every reduced row
    const uint64_t n_red = 1ull << __builtin_popcountll(red);
    k_fold_rows<<<grid_for(n_keys), kMT, 0, st>>>(probs, n_keys, keep, red, n_red, scratch);
  }
  // reorder: output bit b (LSB first) is kept[k-1-b], found at its rank among the kept bits
  BitRanks br;
  br.k = k;
  for (int b = 0; b < k; ++b) {
    const int bit = kept[k - 1 - b];
    br.rank[b] = (int8_t)__builtin_popcountll(keep & ((1ull << bit) - 1ull));
  }
  k_permute_out<<<grid_for(n_keys), kMT, 0, st>>>(asc, n_keys, br, out);
  QSB_CHECK_LAUNCH("qsb_marginal");
  return QSB_OK;
}

extern "C" size_t qsb_cumsum_scratch_bytes(uint64_t n) {
  const uint64_t nb = (n + kScanBlock - 1) / kScanBlock;
  size_t b = 0;
  b += nb * sizeof(double);              // block prefix
  b += nb * sizeof(unsigned int) * 2;    // counts, bases
  b = (b + 255) & ~(size_t)255;
  b += nb * sizeof(Piece);               // heads
  b += nb * sizeof(double);              // block starts
  b = (b + 255) & ~(size_t)255;
  b += nb * sizeof(SegP);                // segmented head prefixes
  b += ((nb + kSegCta - 1) / kSegCta + 1) * sizeof(SegP);  // CTA aggregates
  b = (b + 255) & ~(size_t)255;
  b += (nb + 1) * sizeof(double);        // run start values
  b += 256;
  return b;
}

// The serial-point arrays are sized by the number of serial elements, which is data
// dependent; they live in a separately grown buffer.
static void* g_ser_buf = nullptr;
static size_t g_ser_cap = 0;
static void* g_loc_buf = nullptr;  // per-block serial lists (kLocal pieces pass)
static size_t g_loc_cap = 0;

extern "C" int qsb_cumsum_normalized(const double* probs, uint64_t n, double* cum, void* scratch,
                                     size_t scratch_bytes, void* stream) {
  return qsb_cumsum(probs, n, cum, scratch, scratch_bytes, 1, stream);
}

struct CumsumCtx {
  uint64_t n, nb;
  double margin;
  double* bpre;
  unsigned int* base;
  double* bstart;
  double* sval;
  double* d_total;
};

static int cumsum_phases(const double* probs, uint64_t n, void* scratch, size_t scratch_bytes, cudaStream_t st,
                         CumsumCtx* ctx, const double* block_sums = nullptr);

extern "C" int qsb_cumsum(const double* probs, uint64_t n, double* cum, void* scratch, size_t scratch_bytes,
                          int normalize, void* stream) {
  cudaStream_t st = as_stream(stream);
  if (n == 0) return QSB_OK;
  CumsumCtx c;
  if (int rc = cumsum_phases(probs, n, scratch, scratch_bytes, st, &c)) return rc;
  // E: every c_i, divided by c_{n-1}
  k_materialize2<<<(int)c.nb, kMT, 0, st>>>(probs, n, c.margin, c.bpre, c.base, c.bstart, c.sval, c.d_total, cum,
                                            normalize, nullptr);
  QSB_CHECK_LAUNCH("qsb_cumsum");
  return QSB_OK;
}

// phases A-D of the exact cumsum: block classification, serial points, block head pieces and
// the stitch -- everything but the per-element values (k_materialize2)
static int cumsum_phases(const double* probs, uint64_t n, void* scratch, size_t scratch_bytes, cudaStream_t st,
                         CumsumCtx* ctx, const double* block_sums) {
  if (scratch_bytes < qsb_cumsum_scratch_bytes(n)) {
    set_error("qsb_cumsum: scratch too small");
    return QSB_ERR_ARG;
  }
  const uint64_t nb = (n + kScanBlock - 1) / kScanBlock;
  const double margin = risky_margin(n);
  char* w = static_cast<char*>(scratch);
  double* bpre = reinterpret_cast<double*>(w);
  w += nb * sizeof(double);
  unsigned int* cnt = reinterpret_cast<unsigned int*>(w);
  w += nb * sizeof(unsigned int);
  unsigned int* base = reinterpret_cast<unsigned int*>(w);
  w += nb * sizeof(unsigned int);
  w = reinterpret_cast<char*>(((uintptr_t)w + 255) & ~(uintptr_t)255);
  Piece* head = reinterpret_cast<Piece*>(w);
  w += nb * sizeof(Piece);
  double* bstart = reinterpret_cast<double*>(w);
  w += nb * sizeof(double);
  w = reinterpret_cast<char*>(((uintptr_t)w + 255) & ~(uintptr_t)255);
  SegP* runp = reinterpret_cast<SegP*>(w);
  w += nb * sizeof(SegP);
  const uint64_t na = (nb + kSegCta - 1) / kSegCta;
  SegP* agg = reinterpret_cast<SegP*>(w);
  w += (na + 1) * sizeof(SegP);
  w = reinterpret_cast<char*>(((uintptr_t)w + 255) & ~(uintptr_t)255);
  double* rstart = reinterpret_cast<double*>(w);

  // A: approximate block sums and their exclusive scan (only used to classify)
  if (block_sums) {  // computed with the probabilities (qsb_probabilities_block_sums)
    cudaError_t e = cudaMemcpyAsync(bpre, block_sums, nb * sizeof(double), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_status(e, "block sums");
  } else {
    k_block_sums2<<<(int)nb, kMT, 0, st>>>(probs, n, bpre);
  }
  k_scan_chunked<double><<<1, 1024, 0, st>>>(bpre, nb, bpre, nullptr);
  // B+C: pieces, serial counts and block-local serial lists in one classifying pass; the counts'
  // exclusive scan and total (read back to size the lists, with the overflow flag)
  static unsigned int* h_total = nullptr;
  if (!h_total) {
    cudaError_t e = cudaMallocHost(&h_total, sizeof(unsigned int) * 2);
    if (e != cudaSuccess) return cuda_status(e, "pinned total");
  }
  static unsigned int* d_tot = nullptr;
  if (!d_tot) {
    cudaError_t e = cudaMalloc(&d_tot, sizeof(double) * 2);
    if (e != cudaSuccess) return cuda_status(e, "device total");
  }
  const size_t loc_need = nb * kSerCap * (sizeof(Piece) + sizeof(unsigned long long));
  if (loc_need > g_loc_cap) {
    if (g_loc_buf) cudaFree(g_loc_buf);
    cudaError_t e = cudaMalloc(&g_loc_buf, loc_need);
    if (e != cudaSuccess) {
      g_loc_buf = nullptr;
      g_loc_cap = 0;
      return cuda_status(e, "block serial lists");
    }
    g_loc_cap = loc_need;
  }
  Piece* loc_after = static_cast<Piece*>(g_loc_buf);
  unsigned long long* loc_idx = reinterpret_cast<unsigned long long*>(loc_after + nb * kSerCap);
  {
    cudaError_t e = cudaMemsetAsync(d_tot, 0, sizeof(unsigned int) * 2, st);
    if (e != cudaSuccess) return cuda_status(e, "serial flags");
  }
  k_pieces2<true><<<(int)nb, kMT, 0, st>>>(probs, n, margin, bpre, nullptr, head, loc_after, loc_idx, cnt,
                                           d_tot + 1);
  k_scan_chunked<unsigned int><<<1, 1024, 0, st>>>(cnt, nb, base, d_tot);
  cudaError_t e = cudaMemcpyAsync(h_total, d_tot, sizeof(unsigned int) * 2, cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return cuda_status(e, "serial count copy");
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e, "serial count sync");
  const uint64_t ns = *h_total;
  const size_t need = (ns + 1) * (sizeof(Piece) + sizeof(unsigned long long) + sizeof(double)) + 1024;
  if (need > g_ser_cap) {
    if (g_ser_buf) cudaFree(g_ser_buf);
    g_ser_cap = need * 2;
    e = cudaMalloc(&g_ser_buf, g_ser_cap);
    if (e != cudaSuccess) {
      g_ser_buf = nullptr;
      g_ser_cap = 0;
      return cuda_status(e, "serial buffers");
    }
  }
  char* sb = static_cast<char*>(g_ser_buf);
  Piece* after = reinterpret_cast<Piece*>(sb);
  sb += (ns + 1) * sizeof(Piece);
  unsigned long long* sidx = reinterpret_cast<unsigned long long*>(sb);
  sb += (ns + 1) * sizeof(unsigned long long);
  double* sval = reinterpret_cast<double*>(sb);
  double* d_total = reinterpret_cast<double*>(d_tot) + 1;

  // C: the serial indices and after-pieces into the global lists: compacted from the block
  // lists, and for the blocks with more than kSerCap serial points (e.g. the first elements of a
  // binade under a flat distribution) a second pieces pass over just those blocks writing them
  // at the scanned bases
  k_compact_serials<<<(int)nb, 32, 0, st>>>(cnt, base, loc_after, loc_idx, after, sidx);
  if (h_total[1])
    k_pieces2<false><<<(int)nb, kMT, 0, st>>>(probs, n, margin, bpre, base, head, after, sidx, cnt, nullptr);
  // D: stitch (segmented scan of heads, serial walk, block starts, total)
  k_seg_local<<<(int)na, kMT, 0, st>>>(head, cnt, nb, runp, agg);
  k_seg_top<<<1, kMT, 0, st>>>(agg, na);
  k_seg_fix<<<(int)((nb + kMT - 1) / kMT), kMT, 0, st>>>(runp, nb, agg);
  k_stitch_serial<<<1, 1, 0, st>>>(probs, ns, sidx, after, runp, sval, rstart);
  k_block_starts<<<(int)((nb + kMT - 1) / kMT), kMT, 0, st>>>(runp, nb, rstart, bstart);
  k_total2<<<1, 1, 0, st>>>(head, cnt, nb, bstart, after, sval, ns, d_total);
  QSB_CHECK_LAUNCH("qsb_cumsum");
  ctx->n = n;
  ctx->nb = nb;
  ctx->margin = margin;
  ctx->bpre = bpre;
  ctx->base = base;
  ctx->bstart = bstart;
  ctx->sval = sval;
  ctx->d_total = d_total;
  return QSB_OK;
}

// Reference-semantics sequential version (one device thread); kept for cross-checking the
// parallel scan in the GPU tests.
extern "C" int qsb_cumsum_serial(const double* probs, uint64_t n, double* cum, void* stream) {
  cudaStream_t st = as_stream(stream);
  k_cumsum_serial<<<1, 1, 0, st>>>(probs, n, cum);
  QSB_CHECK_LAUNCH("qsb_cumsum_serial");
  return QSB_OK;
}

// ---- sampling without materialising the whole CDF ---------------------------------------------
// A draw u lands in block b when the normalised value of block b-1's last element is <= u and
// block b's is > u; those values are the (exact) block starts of the stitch divided by the total,
// the same division k_materialize2 applies, so only the blocks that hold a draw are materialised
// and searched.  Samples are bit-identical to qsb_cumsum_normalized + qsb_sample.
namespace qsb {
__global__ void k_block_ends(const double* __restrict__ bstart, uint64_t nb, const double* __restrict__ total,
                             double* __restrict__ ends) {
  const uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  ends[b] = (b + 1 < nb) ? __ddiv_rn(bstart[b + 1], *total) : 2.0;  // every u < 1
}

__global__ void __launch_bounds__(kMT) k_draw_blocks(const double* __restrict__ ends, uint64_t nb, uint64_t s_hi,
                                                     uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, uint64_t n_shots,
                                                     unsigned int* __restrict__ shot_block,
                                                     unsigned char* __restrict__ flags) {
  const uint64_t t = (uint64_t)blockIdx.x * kMT + threadIdx.x;
  const uint64_t first = t * kShotsPerThread;
  if (first >= n_shots) return;
  const u128 inc = ((u128)i_hi << 64) | i_lo;
  u128 s = pcg_advance(((u128)s_hi << 64) | s_lo, inc, first);
  const u128 mult = pcg_mult();
  for (int k = 0; k < kShotsPerThread; ++k) {
    const uint64_t shot = first + k;
    if (shot >= n_shots) break;
    s = s * mult + inc;
    const double u = (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
    uint64_t lo = 0, hi = nb;  // first block whose last value exceeds u
    while (lo < hi) {
      const uint64_t mid = lo + ((hi - lo) >> 1);
      if (ends[mid] <= u)
        lo = mid + 1;
      else
        hi = mid;
    }
    shot_block[shot] = (unsigned int)lo;
    flags[lo] = 1;
  }
}

// Sparse sampling, last pass: each draw searches its block's row ends (normalised like the CDF:
// fl(c / c_{n-1})) for the first row ending above u, then walks that row with fl(c + p_i) from
// its exact start -- the first element whose normalised value exceeds u, as searchsorted on the
// full normalised cumsum gives.
__global__ void __launch_bounds__(kMT) k_draw_rows(const double* __restrict__ p, uint64_t n,
                                                   const double* __restrict__ rs, const double* __restrict__ bstart,
                                                   uint64_t nb, const double* __restrict__ total, uint64_t s_hi,
                                                   uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, uint64_t n_shots,
                                                   const unsigned int* __restrict__ shot_block,
                                                   long long* __restrict__ out) {
  const uint64_t t = (uint64_t)blockIdx.x * kMT + threadIdx.x;
  const uint64_t first = t * kShotsPerThread;
  if (first >= n_shots) return;
  const u128 inc = ((u128)i_hi << 64) | i_lo;
  u128 s = pcg_advance(((u128)s_hi << 64) | s_lo, inc, first);
  const u128 mult = pcg_mult();
  const double tot = *total;
  for (int k = 0; k < kShotsPerThread; ++k) {
    const uint64_t shot = first + k;
    if (shot >= n_shots) break;
    s = s * mult + inc;
    const double u = (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
    const uint64_t b = shot_block[shot];
    const uint64_t b0 = b * kScanBlock;
    const uint64_t rows = min((uint64_t)kMT, (n - b0 + kScanItems - 1) / kScanItems);
    const double* r_b = rs + b * kMT;
    uint64_t lo = 0, hi = rows;  // first row whose end (the next row's start) exceeds u
    while (lo < hi) {
      const uint64_t mid = lo + ((hi - lo) >> 1);
      const double end = (mid + 1 < rows) ? r_b[mid + 1] : (b + 1 < nb ? bstart[b + 1] : tot);
      if (__ddiv_rn(end, tot) <= u)
        lo = mid + 1;
      else
        hi = mid;
    }
    const uint64_t r = lo < rows ? lo : rows - 1;
    double c = r_b[r];
    uint64_t res = n - 1;
    const uint64_t i_first = b0 + r * kScanItems;
    for (int q = 0; q < kScanItems; ++q) {
      const uint64_t i = i_first + q;
      if (i >= n) break;
      c = __dadd_rn(c, p[i]);
      if (__ddiv_rn(c, tot) > u) {
        res = i;
        break;
      }
    }
    out[shot] = (long long)res;
  }
}
}  // namespace qsb

extern "C" size_t qsb_sample_exact_scratch_bytes(uint64_t n, uint64_t n_shots) {
  const uint64_t nb = (n + kScanBlock - 1) / kScanBlock;
  size_t b = (qsb_cumsum_scratch_bytes(n) + 255) & ~(size_t)255;
  b += ((nb * sizeof(double) + 255) & ~(size_t)255);        // block ends
  b += ((nb + 255) & ~(size_t)255);                          // block flags
  b += ((n_shots * sizeof(unsigned int) + 255) & ~(size_t)255);  // block of every shot
  return b;
}

extern "C" int qsb_probabilities_block_sums(const void* amps, uint64_t n, int dtype, double* probs,
                                            double* block_sums, void* stream) {
  cudaStream_t st = as_stream(stream);
  const uint64_t nb = (n + kScanBlock - 1) / kScanBlock;
  if (n == 0) return QSB_OK;
  if (dtype == QSB_C128)
    k_probs_bsums<double><<<(int)nb, kMT, 0, st>>>(static_cast<const double2*>(amps), n, probs, block_sums);
  else if (dtype == QSB_C64)
    k_probs_bsums<float><<<(int)nb, kMT, 0, st>>>(static_cast<const float2*>(amps), n, probs, block_sums);
  else {
    set_error("unknown dtype %d", dtype);
    return QSB_ERR_ARG;
  }
  QSB_CHECK_LAUNCH("qsb_probabilities_block_sums");
  return QSB_OK;
}

static int sample_exact_impl(const double* probs, const double* block_sums, uint64_t n, double* cum, void* scratch,
                             size_t scratch_bytes, uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo,
                             uint64_t n_shots, int64_t* samples, void* stream);

extern "C" int qsb_sample_exact(const double* probs, uint64_t n, double* cum, void* scratch, size_t scratch_bytes,
                                uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, uint64_t n_shots,
                                int64_t* samples, void* stream) {
  return sample_exact_impl(probs, nullptr, n, cum, scratch, scratch_bytes, s_hi, s_lo, i_hi, i_lo, n_shots, samples,
                           stream);
}

extern "C" int qsb_sample_exact_bsums(const double* probs, const double* block_sums, uint64_t n, double* cum,
                                      void* scratch, size_t scratch_bytes, uint64_t s_hi, uint64_t s_lo,
                                      uint64_t i_hi, uint64_t i_lo, uint64_t n_shots, int64_t* samples,
                                      void* stream) {
  return sample_exact_impl(probs, block_sums, n, cum, scratch, scratch_bytes, s_hi, s_lo, i_hi, i_lo, n_shots,
                           samples, stream);
}

static int sample_exact_impl(const double* probs, const double* block_sums, uint64_t n, double* cum, void* scratch,
                             size_t scratch_bytes, uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo,
                             uint64_t n_shots, int64_t* samples, void* stream) {
  cudaStream_t st = as_stream(stream);
  if (n == 0 || n_shots == 0) {
    set_error("qsb_sample_exact: empty distribution or no shots");
    return QSB_ERR_ARG;
  }
  if (n_shots > 0xffffffffull || scratch_bytes < qsb_sample_exact_scratch_bytes(n, n_shots)) {
    set_error("qsb_sample_exact: scratch too small or too many shots");
    return QSB_ERR_ARG;
  }
  const size_t cs = (qsb_cumsum_scratch_bytes(n) + 255) & ~(size_t)255;
  CumsumCtx c;
  if (int rc = cumsum_phases(probs, n, scratch, cs, st, &c, block_sums)) return rc;
  char* w = static_cast<char*>(scratch) + cs;
  double* ends = reinterpret_cast<double*>(w);
  w += (c.nb * sizeof(double) + 255) & ~(size_t)255;
  unsigned char* flags = reinterpret_cast<unsigned char*>(w);
  w += (c.nb + 255) & ~(size_t)255;
  unsigned int* shot_block = reinterpret_cast<unsigned int*>(w);
  cudaError_t e = cudaMemsetAsync(flags, 0, c.nb, st);
  if (e != cudaSuccess) return cuda_status(e, "block flags");
  k_block_ends<<<(int)((c.nb + kMT - 1) / kMT), kMT, 0, st>>>(c.bstart, c.nb, c.d_total, ends);
  const uint64_t threads = (n_shots + kShotsPerThread - 1) / kShotsPerThread;
  const int grid = (int)((threads + kMT - 1) / kMT);
  k_draw_blocks<<<grid, kMT, 0, st>>>(ends, c.nb, s_hi, s_lo, i_hi, i_lo, n_shots, shot_block, flags);
  // row starts of the flagged blocks in `cum` (nb x 256 doubles), then the row walks
  k_row_starts<<<(int)c.nb, kMT, 0, st>>>(probs, n, c.margin, c.bpre, c.base, c.bstart, c.sval, cum, flags);
  k_draw_rows<<<grid, kMT, 0, st>>>(probs, n, cum, c.bstart, c.nb, c.d_total, s_hi, s_lo, i_hi, i_lo, n_shots,
                                    shot_block, reinterpret_cast<long long*>(samples));
  QSB_CHECK_LAUNCH("qsb_sample_exact");
  return QSB_OK;
}

extern "C" int qsb_sample(const double* cum, uint64_t n, uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo,
                          uint64_t n_shots, int64_t* samples, void* stream) {
  cudaStream_t st = as_stream(stream);
  if (n == 0 || n_shots == 0) {
    set_error("qsb_sample: empty distribution or no shots");
    return QSB_ERR_ARG;
  }
  const uint64_t threads = (n_shots + kShotsPerThread - 1) / kShotsPerThread;
  k_sample<<<(int)((threads + kMT - 1) / kMT), kMT, 0, st>>>(cum, n, s_hi, s_lo, i_hi, i_lo, n_shots,
                                                            reinterpret_cast<long long*>(samples), n - 1);
  QSB_CHECK_LAUNCH("qsb_sample");
  return QSB_OK;
}

extern "C" int qsb_sample_counts(const double* cum, uint64_t n, uint64_t s_hi, uint64_t s_lo, uint64_t i_hi,
                                 uint64_t i_lo, uint64_t n_shots, int64_t* counts, void* stream) {
  cudaStream_t st = as_stream(stream);
  if (n == 0 || n_shots == 0) {
    set_error("qsb_sample_counts: empty distribution or no shots");
    return QSB_ERR_ARG;
  }
  const uint64_t threads = (n_shots + kShotsPerThread - 1) / kShotsPerThread;
  k_sample<<<(int)((threads + kMT - 1) / kMT), kMT, 0, st>>>(cum, n, s_hi, s_lo, i_hi, i_lo, n_shots,
                                                            reinterpret_cast<long long*>(counts), ~0ull);
  QSB_CHECK_LAUNCH("qsb_sample_counts");
  return QSB_OK;
}
