// Memory-path probe for the fused pass (round 2): why does a TMA-staged identity pass run at
// ~6.3 TB/s when plain streaming kernels reach ~6.9?  In-place passes over 2^30 complex128
// (17.2 GB), contiguous 64 KB / 32 KB tiles, variants:
//   plain<ITEMS>           : LDG.128 x ITEMS per thread, then STG.128 (the single-gate kernels' shape)
//   tma<T,S,C,M>           : 1-D cp.async.bulk tile loads by a producer warp into S stages of T amps,
//                            C consumer threads copy the stage to registers, then
//                            M=0: release the stage, STG.128 from registers (the current pass kernel)
//                            M=1: STS back into the stage, one thread bulk-stores it (cp.async.bulk
//                                 shared->global), the stage is released once the store has read it
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

typedef unsigned long long u64;
typedef unsigned int u32;
__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* b, u32 c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(u64* b, u32 n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* b, u32 par) {
  asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n}" ::"r"(
                   smem_u32(b)),
               "r"(par)
               : "memory");
}

template <int ITEMS>
__global__ void __launch_bounds__(256) k_plain(double2* x, u64 n) {
  const u64 stride = (u64)gridDim.x * blockDim.x * ITEMS;
  for (u64 i = (u64)blockIdx.x * blockDim.x * ITEMS + threadIdx.x; i < n; i += stride) {
    double2 v[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) v[k] = x[i + (u64)k * blockDim.x];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      v[k].x *= 1.0000000001;
      x[i + (u64)k * blockDim.x] = v[k];
    }
  }
}

// one block per chunk, no loop (the single-gate kernels' launch shape)
template <int ITEMS>
__global__ void __launch_bounds__(256) k_plain_oneshot(double2* x) {
  const u64 i = (u64)blockIdx.x * blockDim.x * ITEMS + threadIdx.x;
  double2 v[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) v[k] = x[i + (u64)k * blockDim.x];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    v[k].x *= 1.0000000001;
    x[i + (u64)k * blockDim.x] = v[k];
  }
}

// ORDER 0: CTA b takes tiles b, b+G, b+2G, ... (lockstep sweep); 1: CTA b takes the contiguous
// range [b*n/G, (b+1)*n/G); 2: one-shot CTAs of TPC consecutive tiles (grid = n_tiles / TPC)
template <int T, int S, int C, int M, int CTAS, int ORDER = 0, int TPC = 1>
__global__ void __launch_bounds__(C + 32, CTAS) k_tma(double2* x, u64 n_tiles) {
  u64 t0, t1, tstep;
  if (ORDER == 0) {
    t0 = blockIdx.x; t1 = n_tiles; tstep = gridDim.x;
  } else if (ORDER == 1) {
    t0 = n_tiles * blockIdx.x / gridDim.x; t1 = n_tiles * (blockIdx.x + 1) / gridDim.x; tstep = 1;
  } else {
    t0 = (u64)blockIdx.x * TPC; t1 = t0 + TPC; tstep = 1;
  }
  extern __shared__ __align__(128) unsigned char smem[];
  double2* stage = reinterpret_cast<double2*>(smem);
  u64* full = reinterpret_cast<u64*>(smem + (size_t)S * T * 16);
  u64* empty = full + S;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], M == 0 ? C : 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid >= C) {
    if (tid != C) return;
    int it = 0;
    for (u64 c = t0; c < t1; c += tstep, ++it) {
      const int s = it % S;
      if (it >= S) mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
      mbar_expect_tx(&full[s], T * 16);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(stage + (size_t)s * T)),
          "l"(x + c * T), "r"(T * 16), "r"(smem_u32(&full[s]))
          : "memory");
    }
    return;
  }
  constexpr int A = T / C;
  int it = 0;
  for (u64 c = t0; c < t1; c += tstep, ++it) {
    const int s = it % S;
    mbar_wait(&full[s], (it / S) & 1);
    double2* buf = stage + (size_t)s * T;
    double2 v[A];
#pragma unroll
    for (int k = 0; k < A; ++k) v[k] = buf[k * C + tid];
#pragma unroll
    for (int k = 0; k < A; ++k) v[k].x *= 1.0000000001;
    if (M == 0) {
      mbar_arrive(&empty[s]);
      double2* d = x + c * T;
#pragma unroll
      for (int k = 0; k < A; ++k) d[k * C + tid] = v[k];
    } else {
#pragma unroll
      for (int k = 0; k < A; ++k) buf[k * C + tid] = v[k];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"n"(C) : "memory");
      if (tid == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(x + c * T), "r"(smem_u32(buf)),
                     "r"(T * 16)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        // the previous tile's store has read its stage: hand that stage back to the producer
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        if (it >= 1) mbar_arrive(&empty[(it - 1) % S]);
      }
    }
  }
  if (M == 1 && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static double2* g_x;
static const u64 N = 1ull << 30;

template <typename F>
static float timeit(F f, int reps = 10) {
  f();
  f();
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("  CUDA error %s\n", cudaGetErrorString(e));
  return ms / reps;
}

static void report(const char* name, float ms) {
  printf("%-40s %7.3f ms  %7.0f GB/s\n", name, ms, 2.0 * N * 16 / ms / 1e6);
  fflush(stdout);
}

template <int ITEMS>
static void run_plain(int blocks_per_sm) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  char name[64];
  snprintf(name, sizeof name, "plain items=%d bps=%d", ITEMS, blocks_per_sm);
  report(name, timeit([&] { k_plain<ITEMS><<<sms * blocks_per_sm, 256>>>(g_x, N); }));
}

template <int ITEMS>
static void run_plain_oneshot() {
  char name[64];
  snprintf(name, sizeof name, "plain one-shot items=%d", ITEMS);
  report(name, timeit([&] { k_plain_oneshot<ITEMS><<<(unsigned)(N / (256 * ITEMS)), 256>>>(g_x); }));
}

template <int T, int S, int C, int M, int CTAS, int ORDER = 0, int TPC = 1>
static void run_tma() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = (size_t)S * T * 16 + 2 * S * 8;
  auto k = k_tma<T, S, C, M, CTAS, ORDER, TPC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  char name[96];
  snprintf(name, sizeof name, "tma tile=%dKB st=%d cons=%d %s ctas=%d ord=%d tpc=%d", T * 16 / 1024, S, C,
           M ? "bulk" : "stg", CTAS, ORDER, TPC);
  const unsigned grid = ORDER == 2 ? (unsigned)(N / T / TPC) : (unsigned)(sms * CTAS);
  report(name, timeit([&] { k<<<grid, C + 32, smem>>>(g_x, N / T); }));
}

int main() {
  cudaMalloc(&g_x, N * 16);
  cudaMemset(g_x, 0, N * 16);
  run_plain_oneshot<4>();
  run_plain_oneshot<8>();
  run_plain<4>(8);
  run_plain<16>(2);
  run_tma<4096, 2, 256, 0, 1>();
  run_tma<4096, 3, 256, 1, 1>();
  run_tma<4096, 2, 256, 0, 1, 1>();
  run_tma<4096, 3, 256, 1, 1, 1>();
  run_tma<2048, 4, 256, 1, 1, 1>();
  run_tma<4096, 2, 256, 0, 1, 2, 4>();
  run_tma<4096, 3, 256, 1, 1, 2, 4>();
  run_tma<4096, 3, 256, 1, 1, 2, 16>();
  run_tma<2048, 3, 128, 1, 2, 2, 8>();
  run_tma<2048, 2, 128, 0, 2, 2, 8>();
  run_tma<2048, 3, 128, 1, 2, 1>();
  run_tma<2048, 2, 256, 0, 2, 2, 4>();
  run_tma<1024, 4, 128, 1, 3, 2, 8>();
  run_plain_oneshot<4>();
  return 0;
}
