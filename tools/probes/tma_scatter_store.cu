// Probe: can TMA tensor stores write a 64 KB tile as 16-byte pieces at 256-byte stride (the
// last QFT pass with the bit-reversal folded in) at HBM speed, with L2 merging the pieces of
// each 256-byte segment written by 16 different CTAs?  Reads are plain contiguous TMA loads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_scatter_store tma_scatter_store.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>

typedef unsigned long long u64;
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// state of 2^n c128 amplitudes; tile = 4096 amplitudes.  Input tile t = contiguous amps
// [4096 t, 4096 t + 4096).  Output: amplitude j of tile t goes to index
//   (j & 15) << (n - 4)  |  (j >> 4) << 4  |  ... (t's bits)  -- i.e. the tile's low 4 bits go
// to the top 4 output bits and the tile's low 4 *external* bits (t & 15) become output bits 0..3.
__global__ void __launch_bounds__(128, 1) k_probe(const __grid_constant__ CUtensorMap in_map,
                                                  const __grid_constant__ CUtensorMap out_map, int n, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  u64* bar = reinterpret_cast<u64*>(sm + 65536);
  const u64 n_tiles = 1ull << (n - 12);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned ph = 0;
  for (u64 t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    if (threadIdx.x == 0) {
      // previous store must have read the buffer before we overwrite it
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(65536u) : "memory");
      int c0 = 0, c1 = (int)(t * 32);  // in map: rows of 2 KB, 32 rows per tile
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(sm)), "l"(&in_map), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
      asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}"
                   ::"r"(smem_u32(bar)), "r"(ph) : "memory");
      ph ^= 1;
      if (mode == 0) {
        // contiguous store (reference speed)
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];"
                     ::"l"(&out_map), "r"(c0), "r"(c1), "r"(smem_u32(sm)) : "memory");
      } else {
        // scattered: out map dims (elem2=2, lowbits=16 [coord], mid=2^(n-8) [box 256? see host], top=16 [box])
        const int lo = (int)(t & 15), mid = (int)(t >> 4);
        asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
                     ::"l"(&out_map), "r"(0), "r"(lo), "r"(mid * 256), "r"(0), "r"(smem_u32(sm)) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int n = 28;
  const size_t bytes = (size_t(1) << n) * 16;
  void *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMemset(a, 0, bytes);
  EncFn enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap in_map, out0, out1;
  {
    // input: dims (256 elems = 2 KB, 32 rows, tiles) -> box (256, 32, 1) = 64 KB; issue as 2d with
    // inner dim 256 and rows = 32 * tiles
    cuuint64_t gd[2] = {256, (cuuint64_t)32 << (n - 12)};
    cuuint64_t gs[1] = {2048};
    cuuint32_t bx[2] = {256, 32}, es[2] = {1, 1};
    printf("enc in %d\n", (int)enc(&in_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a, gd, gs, bx, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    printf("enc out0 %d\n", (int)enc(&out0, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, b, gd, gs, bx, es,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  {
    // scattered output: element dim 2 (one c128), bits 0..3 (coord, box 1), bits 4..n-5 (box 256 of
    // them per tile: the tile's middle 8 bits), bits n-4..n-1 (box 16: the tile's low 4 bits)
    cuuint64_t gd[4] = {2, 16, (cuuint64_t)1 << (n - 8), 16};
    cuuint64_t gs[3] = {16, 256, (cuuint64_t)16 << (n - 4)};
    cuuint32_t bx[4] = {2, 1, 256, 16}, es[4] = {1, 1, 1, 1};
    printf("enc out1 %d\n", (int)enc(&out1, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, b, gd, gs, bx, es,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 0; mode < 2; ++mode) {
    for (int blocks_per_sm = 1; blocks_per_sm <= 3; ++blocks_per_sm) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int w = 0; w < 2; ++w) k_probe<<<sms * blocks_per_sm, 128, 65536 + 64>>>(in_map, mode ? out1 : out0, n, mode);
      cudaEventRecord(e0);
      const int reps = 5;
      for (int r = 0; r < reps; ++r) k_probe<<<sms * blocks_per_sm, 128, 65536 + 64>>>(in_map, mode ? out1 : out0, n, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= reps;
      printf("mode %s ctas/SM %d: %.3f ms  %.1f GB/s  (%s)\n", mode ? "scatter16B" : "contig", blocks_per_sm, ms,
             2.0 * bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
