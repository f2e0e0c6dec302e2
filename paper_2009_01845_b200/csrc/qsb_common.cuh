// Shared device/host helpers for the qsb200 state-vector library (sm_100a).
//
// Layout contract (mirrors the reference qsim, /root/reference/pkg/src/qsim/state.py:1-6,34-36):
// the state is a flat array of 2**n interleaved (re, im) complex numbers; qubit q lives at
// bit position (n - 1 - q) of the basis index.  The device code only ever sees BIT positions;
// the qubit -> bit mapping is done by the Python host layer.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/qsb200.h"

namespace qsb {

template <typename R> struct CplxOf;
template <> struct CplxOf<double> { using T = double2; };
template <> struct CplxOf<float> { using T = float2; };
template <typename R> using cplx = typename CplxOf<R>::T;

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
// a * b with the FMA pattern spelled out (no contraction left to the compiler), so every
// kernel that applies the same gate -- per-gate, batched or sharded -- rounds identically
template <typename C> __device__ __forceinline__ C cmul(C a, C b) {
  C r;
  r.x = fma(a.x, b.x, -mul_rn(a.y, b.y));
  r.y = fma(a.x, b.y, mul_rn(a.y, b.x));
  return r;
}
// acc + a * b
template <typename C> __device__ __forceinline__ C cmad(C a, C b, C acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
template <typename C> __device__ __forceinline__ C czero() {
  C r;
  r.x = 0;
  r.y = 0;
  return r;
}

// Maximum number of occupied (target + control) bit positions a single-gate kernel handles.
constexpr int kMaxOcc = 64;

// Sorted ascending list of bit positions removed from the group counter.
struct OccBits {
  int n;
  uint8_t pos[kMaxOcc];
};

// Open a zero bit at every listed position (ascending) of the group counter g:
// the device form of the reference's _insert_zero_bits (gates.py:355-360), one register chain
// per thread instead of an int64 index array.
__device__ __forceinline__ uint64_t insert_zero_bits(uint64_t g, const OccBits& occ) {
  for (int k = 0; k < occ.n; ++k) {
    const uint64_t low = g & ((1ull << occ.pos[k]) - 1ull);
    g = ((g ^ low) << 1) | low;
  }
  return g;
}

// Error plumbing for the C ABI: every entry point returns a qsb_status and leaves a readable
// message in a thread-local buffer.
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int blocks_for(uint64_t work, int per_block) {
  uint64_t b = (work + per_block - 1) / per_block;
  if (b < 1) b = 1;
  return static_cast<int>(b);
}

}  // namespace qsb

#define QSB_CHECK_LAUNCH(where)                                   \
  do {                                                           \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::qsb::cuda_status(_e, where); \
  } while (0)
