// Host/device declarations shared by the interpreted pass kernel (pass.cu) and the JIT-compiled
// pass kernels (jit.cu): the TMA tile-fetch plan and the program ring buffers.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace qsb {
namespace pass {

// How the producer fetches one tile: mode 1 = TMA tensor loads described by a rank-5 tensor map
// over the state (tile-bit runs are box dims, the bits between them are coordinate dims);
// mode 0 = one bulk copy per contiguous run (fallback for tiles with too many runs).
constexpr int kMaxTmaCalls = 32;
struct TmaPlan {
  int mode;
  int n_gap;
  int gap_dim[5];
  int gap_lo[5];
  int gap_nb[5];
  int top_dim;  // -1: none; else coordinate = tile_base >> top_lo (+ per-call offset)
  int top_lo;
  int n_calls;
  uint32_t call_bytes;
  uint32_t call_coord[kMaxTmaCalls];
};


// Fill `map`/`tp` for a pass whose tile bits are tile_pos[0..K) over an n-qubit state.
// tp->mode stays 0 (bulk-copy fallback) when no tensor map fits.
void plan_tma(const void* src, int n, int K, const int64_t* tile_pos, int amp_bytes, CUtensorMap* map, TmaPlan* tp);

// Encode a rank-5 FLOAT64 tiled tensor map (no swizzle, 256-B L2 promotion) over `base`.
int encode_tensor_map(CUtensorMap* map, void* base, const cuuint64_t* gdim, const cuuint64_t* gstride,
                      const cuuint32_t* box, const cuuint32_t* estride);

// Stage `n` int64 words / doubles in a library-owned device ring (stream-ordered copies).
int stage_words(const void* host, size_t bytes, void** device_out, cudaStream_t st);

}  // namespace pass
}  // namespace qsb
