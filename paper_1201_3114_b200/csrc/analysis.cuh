// analysis.cuh — NEXT-4 analysis kernel: Fig.1 digit frequencies of Lorenz trajectories.
//
// P:239-266 §3.1: "frequency distribution of the integer part as well as the decimal part
// of the Lorenz's attractor": integer part, and digit pairs 1-2, 3-4, 5-6 of the decimal
// part. One lane integrates one trajectory (the same RK4 / Euler / RK4-FMA code as the
// cipher, so the states are bit-identical to the oracle's) and bins every coordinate of the
// state after each `stride` steps (after `skip` transient steps) into per-warp shared-memory
// histograms; the CTA then adds them to the global uint64 histogram.
#pragma once
#include <cstdint>

#include "lorenz_device.cuh"

namespace lz {

constexpr int kHistBins = 3 * 4 * 128;  // [coordinate][kind][bin]

template <int INTEG>
__device__ __forceinline__ void integrate_n(double& x, double& y, double& z, const DevConst& C, uint32_t n) {
  DevConst c2 = C;
  c2.n_it = n;
  integrate<INTEG>(x, y, z, c2);
}

__device__ __forceinline__ void bin_coordinate(uint32_t* h, int c, double v) {
  long long ip = (long long)__double2ll_rz(v);  // trunc(v)
  ip += 64;
  ip = ip < 0 ? 0 : (ip > 127 ? 127 : ip);
  atomicAdd(&h[(c * 4 + 0) * 128 + (int)ip], 1u);
  const double a = fabs(v);
  uint32_t d1, d2, d3;
  if (a < 4000.0) {  // every attractor point (|v| < 64): floor(a 10^6) < 2^32, 32-bit remainders
    d1 = __double2uint_rz(dmul(a, 100.0)) % 100u;
    d2 = __double2uint_rz(dmul(a, 10000.0)) % 100u;
    d3 = __double2uint_rz(dmul(a, 1000000.0)) % 100u;
  } else {
    d1 = (uint32_t)(__double2ull_rz(dmul(a, 100.0)) % 100);
    d2 = (uint32_t)(__double2ull_rz(dmul(a, 10000.0)) % 100);
    d3 = (uint32_t)(__double2ull_rz(dmul(a, 1000000.0)) % 100);
  }
  atomicAdd(&h[(c * 4 + 1) * 128 + (int)d1], 1u);
  atomicAdd(&h[(c * 4 + 2) * 128 + (int)d2], 1u);
  atomicAdd(&h[(c * 4 + 3) * 128 + (int)d3], 1u);
}

template <int INTEG>
__global__ void __launch_bounds__(kCta)
    digit_hist_kernel(const DevConst C, const double* __restrict__ ic, uint64_t lanes, uint32_t skip,
                      uint32_t samples, uint32_t stride, unsigned long long* __restrict__ hist) {
  __shared__ uint32_t h[kWarps][kHistBins];  // per-warp copies: fewer same-address collisions
  for (int i = threadIdx.x; i < kWarps * kHistBins; i += kCta) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint64_t g = (uint64_t)blockIdx.x * kCta + threadIdx.x;
  uint32_t* hw = h[threadIdx.x >> 5];
  if (g < lanes) {
    double x = ic[3 * g], y = ic[3 * g + 1], z = ic[3 * g + 2];
    integrate_n<INTEG>(x, y, z, C, skip);
    for (uint32_t t = 0; t < samples; ++t) {
      integrate_n<INTEG>(x, y, z, C, stride);
      bin_coordinate(hw, 0, x);
      bin_coordinate(hw, 1, y);
      bin_coordinate(hw, 2, z);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kHistBins; i += kCta) {
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += h[w][i];
    if (s) atomicAdd(&hist[i], (unsigned long long)s);
  }
}

}  // namespace lz
