// Fused multi-gate pass: one HBM read + one HBM write of the state for a whole run of gates.
//
// Replaces the per-gate loop of Circuit.execute (/root/reference/pkg/src/qsim/circuit.py:121-124)
// for every gate the host planner (paper_2009_01845_b200/fusion.py) assigns to the pass.
//
// Execution model (B200, sm_100a):
//   * the state is cut into 2^(n-K) tiles of 2^K amplitudes; a tile is the set of indices whose
//     "external" bits are fixed.  Tile bit b sits at global bit tile_pos[b]; the low tile bits
//     are the low global bits, so a tile is 2^(K-L) contiguous runs of >= 256 bytes;
//   * persistent CTAs (1 per SM): one producer warp streams tiles into a 2-stage shared-memory
//     ring with cp.async.bulk (TMA bulk copies) completing on mbarriers; eight consumer warps
//     hold the current tile in REGISTERS (2^(K-8) amplitudes per thread);
//   * a register layout assigns NREG tile bits to register slots and 8 tile bits to the thread
//     id.  Gates whose targets are register bits are pure register arithmetic; a layout change is
//     one shared-memory transpose (XOR-swizzled, conflict-free for the chosen lane bits);
//   * diagonal gates never need locality: they are compiled by the host into
//       - pivot ops   (controlled-phase families, e.g. the QFT's CZPow fans): per-thread
//                     products of partner phases from small tables + one complex multiply,
//       - parity ops  (all -1 phases: Z, CZ, CZ-ladders): popcount parity -> sign flip,
//       - term ops    (anything else): predicated multiply of matching amplitudes;
//   * the result is written straight from registers to HBM (coalesced: the store layout puts
//     lane bits on the low output bits), optionally to permuted positions (SWAP gates folded
//     into the pass as relabels, tile-external swaps as an output tile permutation).
#include <mutex>
#include <cuda.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "qsb_common.cuh"
#include "pass_host.h"

namespace qsb {
namespace pass {

enum : int64_t {
  kMagic = 0x51534250,  // 'QSBP'
  kVersion = 3,
};

enum Op : int64_t {
  OP_END = 0,
  OP_LAYOUT = 1,
  OP_G1 = 2,
  OP_G2 = 3,
  OP_PIVOT = 4,
  OP_PARITY = 5,
  OP_TERM = 6,
  OP_SCALE = 7,
};

enum GKind : int64_t { G_COMPLEX = 0, G_REAL = 1, G_SWAPX = 2 };

constexpr int kConsumers = 512;
constexpr int kThrBits = 9;  // 5 lane bits + 4 warp bits
constexpr int kThreads = kConsumers + 32;
constexpr int kStages = 2;
constexpr int kMaxProgWords = 6144;  // 48 KB of program in shared memory
constexpr int kMaxPivots = 64;

template <typename R> struct Tile;
template <> struct Tile<double> { static constexpr int K = 12; static constexpr int G = 3; };
template <> struct Tile<float> { static constexpr int K = 13; static constexpr int G = 4; };

__device__ __forceinline__ double w2d(int64_t w) { return __longlong_as_double(w); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// one multi-dimensional TMA tensor load (always rank 5; unused dims have extent 1)
__device__ __forceinline__ void tma_load_5d(void* dst_smem, const CUtensorMap* map, const int32_t* c, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], "
      "[%7];" ::"r"(smem_u32(dst_smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// XOR swizzle of a tile slot: tile bit t lands on slot bit (t mod G) for the low G slot bits,
// so 2^G lanes whose lane bits have distinct residues mod G hit distinct 16/8-byte bank groups.
template <int K, int G>
__device__ __forceinline__ uint32_t swz(uint32_t j) {
  uint32_t f = 0;
#pragma unroll
  for (int s = G; s < K; s += G) f ^= (j >> s);
  return j ^ (f & ((1u << G) - 1u));
}

// --- per-layout thread state ---------------------------------------------------------------
struct Layout {
  uint32_t jt;       // tile-index contribution of this thread's bits
  uint64_t gthr;     // global-input-index contribution of this thread's bits
  uint64_t othr;     // global-output-index contribution of this thread's bits
  const int64_t* w;  // program words of the layout op (reg_tb, thr_tb, reg_goff, thr_gpos, reg_ooff, thr_opos)
};

// program layout-op word offsets (after the opcode word)
//   [0, NREG)                reg_tb
//   [NREG, NREG+8)           thr_tb
//   [NREG+8, NREG+8+A)       reg_goff[s]
//   [.., +8)                 thr_gpos
//   [.., +A)                 reg_ooff[s]
//   [.., +8)                 thr_opos
//   [.., +A)                 reg_jt[s]  (tile index of slot s)
template <int NREG>
struct LW {
  static constexpr int A = 1 << NREG;
  static constexpr int T = kThrBits;
  static constexpr int REG_TB = 0, THR_TB = NREG, REG_GOFF = NREG + T, THR_GPOS = REG_GOFF + A, REG_OOFF = THR_GPOS + T,
                       THR_OPOS = REG_OOFF + A, REG_JT = THR_OPOS + T, SIZE = REG_JT + A;
};

template <int NREG>
__device__ __forceinline__ Layout make_layout(const int64_t* w, int tid) {
  using L = LW<NREG>;
  Layout l;
  l.w = w;
  l.jt = 0;
  l.gthr = 0;
  l.othr = 0;
#pragma unroll
  for (int b = 0; b < kThrBits; ++b) {
    if ((tid >> b) & 1) {
      l.jt |= 1u << (int)w[L::THR_TB + b];
      l.gthr |= 1ull << (int)w[L::THR_GPOS + b];
      l.othr |= 1ull << (int)w[L::THR_OPOS + b];
    }
  }
  return l;
}

// --- gate bodies (register bit indices are template parameters -> fully static indexing) -----
template <typename C, int A, int IB, bool CT>
__device__ __forceinline__ void g1_complex(C (&v)[A], const int64_t* m, uint32_t rmask, uint32_t rval) {
  C a00, a01, a10, a11;
  a00.x = w2d(m[0]); a00.y = w2d(m[1]);
  a01.x = w2d(m[2]); a01.y = w2d(m[3]);
  a10.x = w2d(m[4]); a10.y = w2d(m[5]);
  a11.x = w2d(m[6]); a11.y = w2d(m[7]);
#pragma unroll
  for (int s = 0; s < A; ++s) {
    if (s & (1 << IB)) continue;
    if (CT && (s & rmask) != rval) continue;
    const int s1 = s | (1 << IB);
    const C x0 = v[s], x1 = v[s1];
    v[s] = cmad(a01, x1, cmul(a00, x0));
    v[s1] = cmad(a11, x1, cmul(a10, x0));
  }
}

template <typename C, int A, int IB, bool CT>
__device__ __forceinline__ void g1_real(C (&v)[A], const int64_t* m, uint32_t rmask, uint32_t rval) {
  using R = decltype(C().x);
  const R a00 = (R)w2d(m[0]), a01 = (R)w2d(m[2]), a10 = (R)w2d(m[4]), a11 = (R)w2d(m[6]);
#pragma unroll
  for (int s = 0; s < A; ++s) {
    if (s & (1 << IB)) continue;
    if (CT && (s & rmask) != rval) continue;
    const int s1 = s | (1 << IB);
    const C x0 = v[s], x1 = v[s1];
    C y0, y1;
    y0.x = fma(a01, x1.x, a00 * x0.x);
    y0.y = fma(a01, x1.y, a00 * x0.y);
    y1.x = fma(a11, x1.x, a10 * x0.x);
    y1.y = fma(a11, x1.y, a10 * x0.y);
    v[s] = y0;
    v[s1] = y1;
  }
}

template <typename C, int A, int IB, bool CT>
__device__ __forceinline__ void g1_swap(C (&v)[A], uint32_t rmask, uint32_t rval) {
#pragma unroll
  for (int s = 0; s < A; ++s) {
    if (s & (1 << IB)) continue;
    if (CT && (s & rmask) != rval) continue;
    const int s1 = s | (1 << IB);
    const C t = v[s];
    v[s] = v[s1];
    v[s1] = t;
  }
}

template <typename C, int A, int IB>
__device__ __forceinline__ void g1_dispatch(C (&v)[A], int64_t kind, const int64_t* m, uint32_t rmask, uint32_t rval) {
  if (rmask) {
    if (kind == G_REAL)
      g1_real<C, A, IB, true>(v, m, rmask, rval);
    else if (kind == G_SWAPX)
      g1_swap<C, A, IB, true>(v, rmask, rval);
    else
      g1_complex<C, A, IB, true>(v, m, rmask, rval);
  } else {
    if (kind == G_REAL)
      g1_real<C, A, IB, false>(v, m, 0, 0);
    else if (kind == G_SWAPX)
      g1_swap<C, A, IB, false>(v, 0, 0);
    else
      g1_complex<C, A, IB, false>(v, m, 0, 0);
  }
}

template <typename C, int A, int NREG>
__device__ __forceinline__ void apply_g1(C (&v)[A], int ib, int64_t kind, const int64_t* m, uint32_t rmask,
                                         uint32_t rval) {
  switch (ib) {
    case 0: g1_dispatch<C, A, 0>(v, kind, m, rmask, rval); break;
    case 1: g1_dispatch<C, A, 1>(v, kind, m, rmask, rval); break;
    case 2: g1_dispatch<C, A, 2>(v, kind, m, rmask, rval); break;
    case 3: g1_dispatch<C, A, 3>(v, kind, m, rmask, rval); break;
    case 4: if (NREG > 4) g1_dispatch<C, A, (NREG > 4 ? 4 : 0)>(v, kind, m, rmask, rval); break;
    default: break;
  }
}

// two-target gate on register bits IH (row bit 1 = targets[0]) and IL (row bit 0); IH > IL is
// canonicalised by the host (it transposes the matrix when needed).
template <typename C, int A, int IH, int IL, bool CT>
__device__ __forceinline__ void g2_body(C (&v)[A], int64_t kind, const int64_t* m, uint32_t rmask, uint32_t rval) {
  using R = decltype(C().x);
#pragma unroll
  for (int s = 0; s < A; ++s) {
    if (s & ((1 << IH) | (1 << IL))) continue;
    if (CT && (s & rmask) != rval) continue;
    const int sidx[4] = {s, s | (1 << IL), s | (1 << IH), s | (1 << IH) | (1 << IL)};
    C x[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) x[c] = v[sidx[c]];
    if (kind == G_REAL) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        C y;
        const R m0 = (R)w2d(m[8 * r + 0]), m1 = (R)w2d(m[8 * r + 2]), m2 = (R)w2d(m[8 * r + 4]),
                m3 = (R)w2d(m[8 * r + 6]);
        y.x = m0 * x[0].x;
        y.y = m0 * x[0].y;
        y.x = fma(m1, x[1].x, y.x);
        y.y = fma(m1, x[1].y, y.y);
        y.x = fma(m2, x[2].x, y.x);
        y.y = fma(m2, x[2].y, y.y);
        y.x = fma(m3, x[3].x, y.x);
        y.y = fma(m3, x[3].y, y.y);
        v[sidx[r]] = y;
      }
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        C y = czero<C>();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          C mc;
          mc.x = (R)w2d(m[8 * r + 2 * c]);
          mc.y = (R)w2d(m[8 * r + 2 * c + 1]);
          y = cmad(mc, x[c], y);
        }
        v[sidx[r]] = y;
      }
    }
  }
}

template <typename C, int A, int NREG>
__device__ __forceinline__ void apply_g2(C (&v)[A], int ih, int il, int64_t kind, const int64_t* m, uint32_t rmask,
                                         uint32_t rval) {
  // ih > il
#define QSB_G2(H, L)                                                                  \
  if (ih == H && il == L) {                                                           \
    if (H < NREG) {                                                                   \
      if (rmask)                                                                      \
        g2_body<C, A, (H < NREG ? H : 1), L, true>(v, kind, m, rmask, rval);          \
      else                                                                            \
        g2_body<C, A, (H < NREG ? H : 1), L, false>(v, kind, m, 0, 0);                \
    }                                                                                 \
    return;                                                                           \
  }
  QSB_G2(1, 0)
  QSB_G2(2, 0)
  QSB_G2(2, 1)
  QSB_G2(3, 0)
  QSB_G2(3, 1)
  QSB_G2(3, 2)
  QSB_G2(4, 0)
  QSB_G2(4, 1)
  QSB_G2(4, 2)
  QSB_G2(4, 3)
#undef QSB_G2
}

// pivot: amplitudes whose pivot bit is 1 are multiplied by
//   EP[p] (external partners, per tile) * TA[t & 15] * TB[t >> 4] (thread partners) * RT[s]
template <typename C, int A, int IB>
__device__ __forceinline__ void pivot_reg(C (&v)[A], C f, const int64_t* rt, bool use_rt) {
  using R = decltype(C().x);
#pragma unroll
  for (int s = 0; s < A; ++s) {
    if (!(s & (1 << IB))) continue;
    C g = f;
    if (use_rt) {
      C r;
      r.x = (R)w2d(rt[2 * s]);
      r.y = (R)w2d(rt[2 * s + 1]);
      g = cmul(f, r);
    }
    v[s] = cmul(v[s], g);
  }
}

template <typename C, int A>
__device__ __forceinline__ void pivot_all(C (&v)[A], C f, const int64_t* rt, bool use_rt) {
  using R = decltype(C().x);
#pragma unroll
  for (int s = 0; s < A; ++s) {
    C g = f;
    if (use_rt) {
      C r;
      r.x = (R)w2d(rt[2 * s]);
      r.y = (R)w2d(rt[2 * s + 1]);
      g = cmul(f, r);
    }
    v[s] = cmul(v[s], g);
  }
}

template <typename R>
struct Smem {
  static constexpr int K = Tile<R>::K;
  cplx<R> stage[kStages][1 << K];
  int64_t prog[kMaxProgWords];
  cplx<double> ep[2][kMaxPivots];  // per-tile external pivot factors, double-buffered by tile parity
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t base[kStages][2];  // input / output tile base of the tile in each stage (producer-written)
};

// Program header word offsets
enum : int {
  H_MAGIC = 0, H_VER, H_K, H_NREG, H_N, H_DTYPE, H_NTILES, H_FLAGS, H_L, H_NPIV, H_WORDS, H_TILEPOS = 16,
};

template <typename R>
__global__ void __launch_bounds__(kThreads, 1)
    k_pass(const cplx<R>* __restrict__ src, cplx<R>* __restrict__ dst, const int64_t* __restrict__ gprog,
           int n_words, const __grid_constant__ CUtensorMap tmap, const TmaPlan tp) {
  using C = cplx<R>;
  constexpr int K = Tile<R>::K;
  constexpr int G = Tile<R>::G;
  constexpr int NREG = K - kThrBits;
  constexpr int A = 1 << NREG;
  using LWN = LW<NREG>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem<R>& sm = *reinterpret_cast<Smem<R>*>(smem_raw);

  const int tid = threadIdx.x;
  for (int i = tid; i < n_words; i += kThreads) sm.prog[i] = gprog[i];
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t* P = sm.prog;
  const int n = (int)P[H_N];
  const uint64_t n_tiles = (uint64_t)P[H_NTILES];
  const int L = (int)P[H_L];  // low contiguous tile bits
  const int64_t flags = P[H_FLAGS];
  const int64_t* tile_pos = P + H_TILEPOS;
  const int64_t* ext_pos = tile_pos + K;          // n-K ascending external input bits
  const int64_t* ext_out = ext_pos + (n - K);     // n-K output positions of those bits
  const int64_t* ops = ext_out + (n - K);
  const int n_ext = n - K;

  auto tile_base = [&](uint64_t c) -> uint64_t {
    uint64_t b = 0;
    for (int m = 0; m < n_ext; ++m)
      if ((c >> m) & 1ull) b |= 1ull << (int)ext_pos[m];
    return b;
  };
  auto tile_out = [&](uint64_t c) -> uint64_t {
    uint64_t b = 0;
    for (int m = 0; m < n_ext; ++m)
      if ((c >> m) & 1ull) b |= 1ull << (int)ext_out[m];
    return b;
  };

  if (tid >= kConsumers) {
    // ===================== producer warp: TMA bulk loads =====================
    const int lane = tid - kConsumers;
    const int run_len = 1 << L;                    // amplitudes per contiguous run
    const int n_runs = 1 << (K - L);
    const uint32_t run_bytes = run_len * sizeof(C);
    int it = 0;
    for (uint64_t c = blockIdx.x; c < n_tiles; c += gridDim.x, ++it) {
      const int s = it % kStages;
      const uint32_t ph = (it / kStages) & 1;
      if (it >= kStages) mbar_wait(&sm.empty[s], ph ^ 1);
      const uint64_t base = tile_base(c);
      if (lane == 0) {
        sm.base[s][0] = base;
        sm.base[s][1] = (flags & 1) ? tile_out(c) : base;
      }
      if (tp.mode == 1) {
        if (lane == 0) {
          mbar_expect_tx(&sm.full[s], (uint32_t)((1u << K) * sizeof(C)));
          int32_t co[5] = {0, 0, 0, 0, 0};
          for (int g = 0; g < tp.n_gap; ++g)
            co[tp.gap_dim[g]] = (int32_t)((base >> tp.gap_lo[g]) & ((1ull << tp.gap_nb[g]) - 1ull));
          const int32_t top0 = tp.top_dim >= 0 ? (int32_t)(base >> tp.top_lo) : 0;
          char* dstb = reinterpret_cast<char*>(&sm.stage[s][0]);
          for (int k = 0; k < tp.n_calls; ++k) {
            if (tp.top_dim >= 0) co[tp.top_dim] = top0 + (int32_t)tp.call_coord[k];
            tma_load_5d(dstb + (size_t)k * tp.call_bytes, &tmap, co, &sm.full[s]);
          }
        }
        __syncwarp();
        continue;
      }
      if (lane == 0) mbar_expect_tx(&sm.full[s], (uint32_t)((1u << K) * sizeof(C)));
      __syncwarp();
      for (int r = lane; r < n_runs; r += 32) {
        uint64_t off = base;
        for (int b = 0; b < K - L; ++b)
          if ((r >> b) & 1) off |= 1ull << (int)tile_pos[L + b];
        bulk_g2s(&sm.stage[s][r * run_len], src + off, run_bytes, &sm.full[s]);
      }
    }
    return;
  }

  // ===================== consumer warps =====================
  C v[A];
  int it = 0;
  for (uint64_t c = blockIdx.x; c < n_tiles; c += gridDim.x, ++it) {
    const int s = it % kStages;
    const uint32_t ph = (it / kStages) & 1;
    mbar_wait(&sm.full[s], ph);
    const uint64_t base = sm.base[s][0];
    const uint64_t obase = sm.base[s][1];

    // external pivot factors for this tile: one thread per pivot op
    {
      const int npiv = (int)P[H_NPIV];
      if (tid < npiv) {
        // locate the tid-th pivot op by walking the op list (short)
        const int64_t* w = ops;
        int seen = 0;
        while (w[0] != OP_END) {
          const int64_t op = w[0];
          const int64_t len = w[1];
          if (op == OP_PIVOT) {
            if (seen == tid) {
              // w[2]=slot w[3]=pivot type w[4]=pivot value w[5]=use_rt w[6]=n_ext_partners, then pairs
              const int ne = (int)w[6];
              double2 f = make_double2(1.0, 0.0);
              for (int q = 0; q < ne; ++q) {
                const int bit = (int)w[7 + 3 * q];
                if ((base >> bit) & 1ull) {
                  const double2 ph2 = make_double2(w2d(w[8 + 3 * q]), w2d(w[9 + 3 * q]));
                  f = make_double2(f.x * ph2.x - f.y * ph2.y, f.x * ph2.y + f.y * ph2.x);
                }
              }
              sm.ep[it & 1][w[2]] = f;
              break;
            }
            ++seen;
          }
          w += len;
        }
      }
    }

    cplx<R>* buf = sm.stage[s];

    // initial layout: read registers from the natural-order stage
    const int64_t* w = ops;
    // first op is always OP_LAYOUT
    Layout lay = make_layout<NREG>(w + 2, tid);
#pragma unroll
    for (int sl = 0; sl < A; ++sl) v[sl] = buf[lay.jt | (uint32_t)w[2 + LWN::REG_JT + sl]];
    w += w[1];
    bool swizzled = false;  // stage content: natural (TMA) order until the first transpose

    consumer_sync();  // stage fully read (reused as transpose scratch) and ep[] of this tile visible

    while (true) {
      const int64_t op = w[0];
      if (op == OP_END) break;
      const int64_t len = w[1];
      const int64_t* a = w + 2;
      switch (op) {
        case OP_LAYOUT: {
          // transpose through shared memory: write current layout, read the new one
          if (swizzled) consumer_sync();  // previous reads of the scratch are complete
#pragma unroll
          for (int sl = 0; sl < A; ++sl) buf[swz<K, G>(lay.jt | (uint32_t)lay.w[LWN::REG_JT + sl])] = v[sl];
          consumer_sync();
          lay = make_layout<NREG>(a, tid);
#pragma unroll
          for (int sl = 0; sl < A; ++sl) v[sl] = buf[swz<K, G>(lay.jt | (uint32_t)a[LWN::REG_JT + sl])];
          swizzled = true;
          break;
        }
        case OP_G1: {
          // a: [ib, kind, gmask, gval, rmask, rval, m(8)]
          const uint64_t gmask = (uint64_t)a[2], gval = (uint64_t)a[3];
          if (((base | lay.gthr) & gmask) == gval)
            apply_g1<C, A, NREG>(v, (int)a[0], a[1], a + 6, (uint32_t)a[4], (uint32_t)a[5]);
          break;
        }
        case OP_G2: {
          // a: [ih, il, kind, gmask, gval, rmask, rval, m(32)]
          const uint64_t gmask = (uint64_t)a[3], gval = (uint64_t)a[4];
          if (((base | lay.gthr) & gmask) == gval)
            apply_g2<C, A, NREG>(v, (int)a[0], (int)a[1], a[2], a + 7, (uint32_t)a[5], (uint32_t)a[6]);
          break;
        }
        case OP_PIVOT: {
          // a: [slot, ptype, pval, use_rt, n_ext, ext(3*n_ext), TA(2*16), TB(2*32), RT(2A)]
          const int ne = (int)a[4];
          const int64_t* ta = a + 5 + 3 * ne;
          const int64_t* tb = ta + 32;
          const int64_t* rt = tb + 64;
          const bool use_rt = a[3] != 0;
          const int ptype = (int)a[1];
          bool active = true;
          if (ptype == 1) active = ((base | lay.gthr) & (uint64_t)a[2]) != 0;  // thread/external pivot
          if (!active) break;
          const double2 e = sm.ep[it & 1][a[0]];
          const int tl = tid & 15, th = tid >> 4;
          double2 t1 = make_double2(w2d(ta[2 * tl]), w2d(ta[2 * tl + 1]));
          double2 t2 = make_double2(w2d(tb[2 * th]), w2d(tb[2 * th + 1]));
          double2 f12 = make_double2(t1.x * t2.x - t1.y * t2.y, t1.x * t2.y + t1.y * t2.x);
          double2 fd = make_double2(e.x * f12.x - e.y * f12.y, e.x * f12.y + e.y * f12.x);
          C f;
          f.x = (R)fd.x;
          f.y = (R)fd.y;
          if (ptype == 0) {
            switch ((int)a[2]) {
              case 0: pivot_reg<C, A, 0>(v, f, rt, use_rt); break;
              case 1: pivot_reg<C, A, 1>(v, f, rt, use_rt); break;
              case 2: pivot_reg<C, A, 2>(v, f, rt, use_rt); break;
              case 3: pivot_reg<C, A, 3>(v, f, rt, use_rt); break;
              case 4: if (NREG > 4) pivot_reg<C, A, (NREG > 4 ? 4 : 0)>(v, f, rt, use_rt); break;
              default: break;
            }
          } else {
            pivot_all<C, A>(v, f, rt, use_rt);
          }
          break;
        }
        case OP_PARITY: {
          // a: [single_mask, n_d, (d, M_d) * n_d]  -> negate amplitudes with odd parity
          const uint64_t sm1 = (uint64_t)a[0];
          const int nd = (int)a[1];
#pragma unroll
          for (int sl = 0; sl < A; ++sl) {
            const uint64_t gi = base | lay.gthr | (uint64_t)lay.w[LWN::REG_GOFF + sl];
            int par = __popcll(gi & sm1);
            for (int q = 0; q < nd; ++q) par += __popcll(gi & (gi >> (int)a[2 + 2 * q]) & (uint64_t)a[3 + 2 * q]);
            if (par & 1) {
              v[sl].x = -v[sl].x;
              v[sl].y = -v[sl].y;
            }
          }
          break;
        }
        case OP_TERM: {
          // a: [mask, val, re, im]: amplitudes with (index & mask) == val are multiplied
          const uint64_t mask = (uint64_t)a[0], val = (uint64_t)a[1];
          C ph;
          ph.x = (R)w2d(a[2]);
          ph.y = (R)w2d(a[3]);
#pragma unroll
          for (int sl = 0; sl < A; ++sl) {
            const uint64_t gi = base | lay.gthr | (uint64_t)lay.w[LWN::REG_GOFF + sl];
            if ((gi & mask) == val) v[sl] = cmul(v[sl], ph);
          }
          break;
        }
        case OP_SCALE: {
          C ph;
          ph.x = (R)w2d(a[0]);
          ph.y = (R)w2d(a[1]);
#pragma unroll
          for (int sl = 0; sl < A; ++sl) v[sl] = cmul(v[sl], ph);
          break;
        }
        default:
          break;
      }
      w += len;
    }
    // the stage (or its reuse as transpose scratch) is no longer read: hand it back
    fence_proxy_async();
    mbar_arrive(&sm.empty[s]);
    // store from registers to the output positions of the final layout
#pragma unroll
    for (int sl = 0; sl < A; ++sl) dst[obase | lay.othr | (uint64_t)lay.w[LWN::REG_OOFF + sl]] = v[sl];
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

int encode_tensor_map(CUtensorMap* map, void* base, const cuuint64_t* gdim, const cuuint64_t* gstride,
                      const cuuint32_t* box, const cuuint32_t* estride) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return QSB_ERR_CUDA;
  }
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, base, gdim, gstride, box, estride,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return QSB_ERR_ARG;
  }
  return QSB_OK;
}

// Describe the state as a rank-5 tensor of 8-byte elements whose box is one tile.
void plan_tma(const void* src, int n, int K, const int64_t* tile_pos, int amp_bytes, CUtensorMap* map,
              TmaPlan* tp) {
  memset(tp, 0, sizeof *tp);
  tp->mode = 0;
  tp->top_dim = -1;
  EncodeTiledFn enc = encode_fn();
  if (!enc) return;
  const int epa = amp_bytes / 8;  // 8-byte elements per amplitude
  uint64_t tmask = 0;
  for (int b = 0; b < K; ++b) tmask |= 1ull << tile_pos[b];
  struct D { int lo, nb; bool tile; };
  D dims[64];
  int nd = 0;
  int b = 0;
  while (b < n) {
    const bool t = (tmask >> b) & 1ull;
    int e = b;
    while (e < n && (((tmask >> e) & 1ull) != 0) == t) ++e;
    if (t) {
      int p = b;
      while (p < e) {
        const int lim = (nd == 0 && epa == 2) ? 7 : 8;  // box extent <= 256 elements
        const int w = (e - p) < lim ? (e - p) : lim;
        dims[nd++] = {p, w, true};
        p += w;
      }
    } else {
      dims[nd++] = {b, e - b, false};
    }
    b = e;
  }
  int use = nd;
  uint64_t iter_mask = 0;
  int top_lo = n;
  if (nd > 5) {
    use = 5;
    top_lo = dims[4].lo;
    iter_mask = (tmask >> top_lo);  // tile bits inside the merged top dim are iterated
    dims[4] = {top_lo, n - top_lo, false};
  }
  const int iter_bits = __builtin_popcountll(iter_mask);
  if (iter_bits > 5) return;  // > 32 calls: bulk-copy fallback
  for (int d = 0; d < use; ++d)
    if (!dims[d].tile && dims[d].nb > 31) return;
  cuuint64_t gdim[5], gstride[4];
  cuuint32_t box[5], estride[5];
  uint64_t extent_bytes = 8;
  for (int d = 0; d < 5; ++d) {
    if (d < use) {
      gdim[d] = (1ull << dims[d].nb) * (d == 0 ? epa : 1);
      box[d] = dims[d].tile ? (cuuint32_t)gdim[d] : 1u;
      if (d > 0) gstride[d - 1] = (1ull << dims[d].lo) * amp_bytes;
    } else {
      gdim[d] = 1;
      box[d] = 1;
      if (d > 0) gstride[d - 1] = (1ull << n) * amp_bytes;
    }
    estride[d] = 1;
  }
  (void)extent_bytes;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<void*>(src), gdim, gstride, box, estride,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return;
  tp->n_gap = 0;
  for (int d = 0; d < use; ++d) {
    if (dims[d].tile) continue;
    if (nd > 5 && d == 4) continue;
    tp->gap_dim[tp->n_gap] = d;
    tp->gap_lo[tp->n_gap] = dims[d].lo;
    tp->gap_nb[tp->n_gap] = dims[d].nb;
    ++tp->n_gap;
  }
  uint64_t box_elems = 1;
  for (int d = 0; d < 5; ++d) box_elems *= box[d];
  tp->call_bytes = (uint32_t)(box_elems * 8);
  if (nd > 5) {
    tp->top_dim = 4;
    tp->top_lo = top_lo;
    tp->n_calls = 1 << iter_bits;
    for (int k = 0; k < tp->n_calls; ++k) {
      // deposit the bits of k onto the tile bits of the top dim (ascending)
      uint32_t off = 0;
      int j = 0;
      for (int q = 0; q < 64 && (iter_mask >> q); ++q)
        if ((iter_mask >> q) & 1ull) {
          if ((k >> j) & 1) off |= 1u << q;
          ++j;
        }
      tp->call_coord[k] = off;
    }
  } else {
    tp->n_calls = 1;
    tp->call_coord[0] = 0;
  }
  tp->mode = 1;
}

// Device ring for per-launch program / coefficient words, one per CUDA device.  Copies are
// stream-ordered; when a ring wraps, the whole device is synchronised once, so no launch queued
// on ANY stream (other host threads' streams, side streams, user streams) can still be reading
// the slots that are about to be overwritten.  Staging is refused while `st` is being captured
// into a CUDA graph: a replay would re-read a ring slot that later launches overwrite (callers
// that capture own their words in device buffers, see qsb_jit_run_pass_dev).
int stage_words(const void* host, size_t bytes, void** device_out, cudaStream_t st) {
  // The words go through a pinned host mirror of the device ring, so the upload is a real
  // asynchronous DMA (a pageable source would make the driver synchronise with the stream,
  // stalling the host behind the GPU at every pass).
  constexpr int kMaxDevices = 64;
  static char* ring[kMaxDevices] = {};
  static char* hring[kMaxDevices] = {};
  static size_t cursor[kMaxDevices] = {};
  static std::mutex mu;  // ctypes drops the GIL: host threads may stage concurrently
  std::lock_guard<std::mutex> lock(mu);
  constexpr size_t kRing = 16u << 20;
  if (bytes > kRing / 4) {
    set_error("stage_words: %zu bytes too large", bytes);
    return QSB_ERR_ARG;
  }
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone) {
    set_error("stage_words: host-staged words cannot be captured into a CUDA graph (own them on the device)");
    return QSB_ERR_ARG;
  }
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "program ring device");
  if (dev < 0 || dev >= kMaxDevices) {
    set_error("stage_words: device %d out of range", dev);
    return QSB_ERR_ARG;
  }
  if (!ring[dev]) {
    e = cudaMalloc(&ring[dev], kRing);
    if (e != cudaSuccess) {
      ring[dev] = nullptr;
      return cuda_status(e, "program ring");
    }
    e = cudaMallocHost(&hring[dev], kRing);
    if (e != cudaSuccess) {
      cudaFree(ring[dev]);
      ring[dev] = nullptr;
      hring[dev] = nullptr;
      return cuda_status(e, "pinned program ring");
    }
  }
  size_t off = (cursor[dev] + 255) & ~(size_t)255;
  if (off + bytes > kRing) {
    // every earlier upload out of the pinned mirror and every launch reading the device ring,
    // on whichever stream, has finished after this: both rings can be reused from the start
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_status(e, "program ring wrap");
    off = 0;
  }
  cursor[dev] = off + bytes;
  memcpy(hring[dev] + off, host, bytes);
  e = cudaMemcpyAsync(ring[dev] + off, hring[dev] + off, bytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_status(e, "program upload");
  *device_out = ring[dev] + off;
  return QSB_OK;
}

template <typename R>
static int launch(const void* src, void* dst, const int64_t* hprog, int64_t n_words, cudaStream_t st) {
  constexpr int K = Tile<R>::K;
  if (n_words > kMaxProgWords) {
    set_error("qsb_run_pass: program of %lld words exceeds %d", (long long)n_words, kMaxProgWords);
    return QSB_ERR_ARG;
  }
  if (hprog[H_MAGIC] != kMagic || hprog[H_VER] != kVersion || hprog[H_K] != K || hprog[H_NREG] != K - kThrBits) {
    set_error("qsb_run_pass: program header mismatch (magic/version/K)");
    return QSB_ERR_ARG;
  }
  if (hprog[H_NPIV] > kMaxPivots) {
    set_error("qsb_run_pass: too many pivot ops");
    return QSB_ERR_ARG;
  }
  void* dprog_v = nullptr;
  if (int rc = stage_words(hprog, sizeof(int64_t) * n_words, &dprog_v, st)) return rc;
  int64_t* dprog = static_cast<int64_t*>(dprog_v);
  cudaError_t e;
  const size_t smem = sizeof(Smem<R>);
  static bool attr_set = false;
  if (!attr_set) {
    e = cudaFuncSetAttribute(k_pass<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "pass smem attribute");
    attr_set = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t n_tiles = (uint64_t)hprog[H_NTILES];
  const int grid = (int)(n_tiles < (uint64_t)sms ? n_tiles : (uint64_t)sms);
  alignas(64) CUtensorMap map;
  memset(&map, 0, sizeof map);
  TmaPlan tp;
  static const bool no_tma = getenv("QSB_NO_TMA_TENSOR") != nullptr;
  if (no_tma) {
    memset(&tp, 0, sizeof tp);
    tp.top_dim = -1;
  } else {
    plan_tma(src, (int)hprog[H_N], K, hprog + H_TILEPOS, (int)sizeof(cplx<R>), &map, &tp);
  }
  k_pass<R><<<grid, kThreads, smem, st>>>(static_cast<const cplx<R>*>(src), static_cast<cplx<R>*>(dst), dprog,
                                         (int)n_words, map, tp);
  QSB_CHECK_LAUNCH("qsb_run_pass");
  return QSB_OK;
}

}  // namespace pass
}  // namespace qsb

extern "C" int qsb_pass_max_tile_bits(int dtype) {
  return dtype == QSB_C128 ? qsb::pass::Tile<double>::K : qsb::pass::Tile<float>::K;
}

extern "C" int qsb_run_pass(const void* src, void* dst, int n_qubits, int dtype, const int64_t* program,
                            int64_t n_words, void* stream) {
  using namespace qsb;
  if (program == nullptr || n_words < pass::H_TILEPOS) {
    set_error("qsb_run_pass: empty program");
    return QSB_ERR_ARG;
  }
  if (program[pass::H_N] != n_qubits || program[pass::H_DTYPE] != dtype) {
    set_error("qsb_run_pass: program built for n=%lld dtype=%lld", (long long)program[pass::H_N],
              (long long)program[pass::H_DTYPE]);
    return QSB_ERR_ARG;
  }
  if (dtype == QSB_C128) return pass::launch<double>(src, dst, program, n_words, as_stream(stream));
  if (dtype == QSB_C64) return pass::launch<float>(src, dst, program, n_words, as_stream(stream));
  set_error("unknown dtype %d", dtype);
  return QSB_ERR_ARG;
}
