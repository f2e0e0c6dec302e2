// Reduced density matrix of a qubit subset, straight from the amplitudes (no permuted copy of
// the state, no library GEMM) -- the device half of entanglement_entropy
// (/root/reference/pkg/src/qsim/evolution.py:154-173).
//
// The reference moves the partition's axes to the front, reshapes to M (2^k x 2^(n-k)) and
// takes numpy's singular values of M; their squares are the eigenvalues of rho = M M^dagger:
//   rho[i][j] = sum_b psi(i, b) * conj(psi(j, b)),
// with i the k partition bits (partition[0] = MSB of i) and b the other n-k bits.  rho is
// accumulated here in complex128 (the reference casts to complex128 first), its eigenvalues
// are taken on the host (a 2^k x 2^k Hermitian matrix, k <= 12).
//
// Kernel: one CTA per (row tile, column tile, split) with row tile <= column tile (rho is
// Hermitian; the reduction fills the lower triangle).  A tile is T x T entries (T = min(32,
// 2^k)); each split owns a fixed contiguous range of b, walked in chunks of 32: the chunk's
// amplitudes of the tile's rows and columns are staged in shared memory (b fastest across a
// warp: coalesced when the low state bits are not partition bits), and every thread
// accumulates 4 entries.  Partial tiles go to a scratch [split][2^k][2^k] and are summed in a
// fixed order by k_rdm_reduce, so the result does not depend on scheduling.
#include "qsb_common.cuh"

namespace qsb {

constexpr int kRdmThreads = 256;
constexpr int kRdmChunk = 32;
constexpr int kRdmMaxK = 12;

struct RdmArgs {
  int n, k, T, n_tiles;  // tiles per matrix side
  uint64_t split_len;    // b values per split (multiple of kRdmChunk)
  uint64_t row_dep[1 << 5];  // deposit of row offset r (< T) into state bits (low 5 row bits)
  uint8_t row_pos[kRdmMaxK];  // state bit of row bit m (m = 0 is the LSB of the row index)
  uint8_t rest_pos[64];       // state bits of b, ascending
};

__device__ __forceinline__ uint64_t deposit_rest(uint64_t b, const RdmArgs& a) {
  uint64_t x = 0;
  for (int m = 0; b; ++m, b >>= 1) x |= (b & 1ull) << a.rest_pos[m];
  return x;
}

__device__ __forceinline__ uint64_t deposit_row(uint64_t i, const RdmArgs& a) {
  uint64_t x = 0;
  for (int m = 0; m < a.k; ++m) x |= ((i >> m) & 1ull) << a.row_pos[m];
  return x;
}

template <typename R>
__global__ void __launch_bounds__(kRdmThreads) k_rdm(const cplx<R>* __restrict__ psi, const RdmArgs a,
                                                    double2* __restrict__ partials) {
  __shared__ double2 si[32][kRdmChunk + 1];
  __shared__ double2 sj[32][kRdmChunk + 1];
  __shared__ uint64_t rest_lo[kRdmChunk];
  // upper-triangle tile pair of this CTA
  int p = blockIdx.x, ti = 0;
  while (p >= a.n_tiles - ti) {
    p -= a.n_tiles - ti;
    ++ti;
  }
  const int tj = ti + p;
  const int split = blockIdx.y;
  const int T = a.T;
  const int tid = threadIdx.x;
  if (tid < kRdmChunk) rest_lo[tid] = deposit_rest((uint64_t)tid, a);
  const uint64_t rbase_i = deposit_row((uint64_t)ti * T, a);
  const uint64_t rbase_j = deposit_row((uint64_t)tj * T, a);
  __syncthreads();
  // thread -> (row r, 4 columns c0..c0+3) of the T x T tile (T = 32: 256 threads x 4 = 1024)
  const int per_row = T / 4 > 0 ? T / 4 : 1;
  const int r = tid / per_row;
  const int c0 = (tid % per_row) * 4;
  const bool active = r < T && c0 < T;
  double2 acc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = make_double2(0.0, 0.0);
  const uint64_t b_begin = (uint64_t)split * a.split_len;
  for (uint64_t b0 = b_begin; b0 < b_begin + a.split_len; b0 += kRdmChunk) {
    const uint64_t hi = deposit_rest(b0, a);
    for (int e = tid; e < T * kRdmChunk; e += kRdmThreads) {
      const int bl = e % kRdmChunk, rl = e / kRdmChunk;
      const uint64_t xo = hi | rest_lo[bl];
      const cplx<R> vi = psi[xo | rbase_i | a.row_dep[rl]];
      const cplx<R> vj = psi[xo | rbase_j | a.row_dep[rl]];
      si[rl][bl] = make_double2((double)vi.x, (double)vi.y);
      sj[rl][bl] = make_double2((double)vj.x, (double)vj.y);
    }
    __syncthreads();
    if (active) {
#pragma unroll 4
      for (int b = 0; b < kRdmChunk; ++b) {
        const double2 x = si[r][b];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 y = sj[c0 + q][b];  // x * conj(y)
          acc[q].x = fma(x.x, y.x, acc[q].x);
          acc[q].x = fma(x.y, y.y, acc[q].x);
          acc[q].y = fma(x.y, y.x, acc[q].y);
          acc[q].y = fma(-x.x, y.y, acc[q].y);
        }
      }
    }
    __syncthreads();
  }
  if (active) {
    const uint64_t dim = 1ull << a.k;
    double2* out = partials + (uint64_t)split * dim * dim;
    const uint64_t row = (uint64_t)ti * T + r;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (c0 + q < T) out[row * dim + (uint64_t)tj * T + c0 + q] = acc[q];
  }
}

// rho[i][j] = sum over splits in order (i <= j from the tiles, i > j = conjugate of rho[j][i])
__global__ void k_rdm_reduce(const double2* __restrict__ partials, int n_split, int k,
                             double2* __restrict__ rho) {
  const uint64_t dim = 1ull << k;
  const uint64_t total = dim * dim;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = e / dim, j = e % dim;
    const bool upper = i <= j;  // (j, i) lies in a computed tile whenever i > j
    const uint64_t src = upper ? e : j * dim + i;
    double2 s = make_double2(0.0, 0.0);
    for (int q = 0; q < n_split; ++q) {
      const double2 v = partials[(uint64_t)q * total + src];
      s.x += v.x;
      s.y += v.y;
    }
    if (!upper) s.y = -s.y;
    if (i == j) s.y = 0.0;  // rho_ii = sum |psi|^2 is real; drop the rounding of x * conj(x)
    rho[e] = s;
  }
}

}  // namespace qsb

using namespace qsb;

extern "C" {

int qsb_reduced_density(const void* amps, int n, int dtype, int k, const int* partition_bits, int n_split,
                        void* partials, void* rho, void* stream) {
  if (dtype != QSB_C64 && dtype != QSB_C128) {
    set_error("qsb_reduced_density: unknown dtype %d", dtype);
    return QSB_ERR_ARG;
  }
  if (n < 2 || n > 40 || k < 1 || k > kRdmMaxK || k >= n) {
    set_error("qsb_reduced_density: need 1 <= k <= %d and k < n (n=%d, k=%d)", kRdmMaxK, n, k);
    return QSB_ERR_SHAPE;
  }
  RdmArgs a;
  a.n = n;
  a.k = k;
  a.T = k >= 5 ? 32 : (1 << k);
  a.n_tiles = (1 << k) / a.T;
  uint64_t used = 0;
  for (int r = 0; r < k; ++r) {  // partition_bits[0] is the MSB of the row index
    const int b = partition_bits[r];
    if (b < 0 || b >= n || ((used >> b) & 1ull)) {
      set_error("qsb_reduced_density: bad or duplicate bit %d", b);
      return QSB_ERR_SHAPE;
    }
    used |= 1ull << b;
    a.row_pos[k - 1 - r] = (uint8_t)b;
  }
  int m = 0;
  for (int b = 0; b < n; ++b)
    if (!((used >> b) & 1ull)) a.rest_pos[m++] = (uint8_t)b;
  for (int r = 0; r < 32; ++r) {
    uint64_t x = 0;
    for (int q = 0; q < k && q < 5; ++q) x |= (uint64_t)((r >> q) & 1) << a.row_pos[q];
    a.row_dep[r] = x;
  }
  const uint64_t n_rest = 1ull << (n - k);
  if (n_split < 1 || (n_split & (n_split - 1)) || (uint64_t)n_split * kRdmChunk > n_rest) {
    set_error("qsb_reduced_density: n_split %d must be a power of two with n_split * 32 <= 2^(n-k)", n_split);
    return QSB_ERR_SHAPE;
  }
  a.split_len = n_rest / (uint64_t)n_split;
  cudaStream_t st = as_stream(stream);
  const int pairs = a.n_tiles * (a.n_tiles + 1) / 2;
  dim3 grid(pairs, n_split);
  if (dtype == QSB_C128)
    k_rdm<double><<<grid, kRdmThreads, 0, st>>>(static_cast<const double2*>(amps), a,
                                                static_cast<double2*>(partials));
  else
    k_rdm<float><<<grid, kRdmThreads, 0, st>>>(static_cast<const float2*>(amps), a,
                                               static_cast<double2*>(partials));
  const uint64_t total = 1ull << (2 * k);
  const int rblocks = (int)((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
  k_rdm_reduce<<<rblocks, 256, 0, st>>>(static_cast<const double2*>(partials), n_split, k,
                                        static_cast<double2*>(rho));
  QSB_CHECK_LAUNCH("qsb_reduced_density");
  return QSB_OK;
}

}  // extern "C"
