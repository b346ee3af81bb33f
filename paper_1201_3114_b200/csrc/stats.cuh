// stats.cuh — integer-exact reductions for the C5 sensitivity sweep (avalanche statistics).
//
// The paper judges the cipher by byte histograms / entropy of the ciphertext (§4,
// Fig.2) and by the effect of "slightly different passwords". C5 measures, per trial,
// the bit differences between ciphertexts of one-bit-flipped passwords / messages and the
// 256-bin byte histograms; entropy and chi-square are computed on the host from the integer
// counts. These are HBM-bound streaming reductions (16-byte loads, popcount, smem atomics).
#pragma once
#include <cstdint>

#include "../../include/lorenz.h"

namespace lz {

constexpr int kStatCta = 256;
constexpr uint64_t kStatTile = 1 << 16;  // bytes of one span handled by one CTA

__device__ __forceinline__ void block_add_u64(uint64_t v, uint64_t* dst, uint64_t* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t s = 0;
    for (int i = 0; i < kStatCta / 32; ++i) s += red[i];
    if (s) atomicAdd(reinterpret_cast<unsigned long long*>(dst), (unsigned long long)s);
  }
  __syncthreads();
}

// grid.x = tiles per span (max over spans), grid.y = span index.
// out[3*i+0] += differing bits, [3*i+1] += differing bytes, [3*i+2] += bytes with equal LSB.
__global__ void __launch_bounds__(kStatCta)
    compare_spans_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                         const lorenz_span* __restrict__ spans, uint64_t* __restrict__ out) {
  __shared__ uint64_t red[kStatCta / 32];
  const lorenz_span sp = spans[blockIdx.y];
  const uint64_t t0 = (uint64_t)blockIdx.x * kStatTile;
  if (t0 >= sp.len) return;
  const uint64_t t1 = (t0 + kStatTile < sp.len) ? t0 + kStatTile : sp.len;
  const uint8_t* pa = a + sp.a_off;
  const uint8_t* pb = b + sp.b_off;
  uint64_t bits = 0, bytes = 0, lsb_eq = 0;
  // 16-byte path when both spans are 16-aligned at t0, byte tail otherwise
  const bool vec = ((reinterpret_cast<uintptr_t>(pa + t0) | reinterpret_cast<uintptr_t>(pb + t0)) & 15) == 0;
  uint64_t i = t0;
  if (vec) {
    const uint64_t v1 = t0 + ((t1 - t0) & ~15ULL);
    for (uint64_t k = t0 + 16 * threadIdx.x; k < v1; k += 16 * kStatCta) {
      const uint4 x = __ldcs(reinterpret_cast<const uint4*>(pa + k));
      const uint4 y = __ldcs(reinterpret_cast<const uint4*>(pb + k));
      const uint32_t d[4] = {x.x ^ y.x, x.y ^ y.y, x.z ^ y.z, x.w ^ y.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        bits += __popc(d[q]);
        bytes += __popc(__vcmpne4(d[q], 0u)) >> 3;
        lsb_eq += 4 - __popc(d[q] & 0x01010101u);
      }
    }
    i = v1;
  }
  for (uint64_t k = i + threadIdx.x; k < t1; k += kStatCta) {
    const uint32_t d = pa[k] ^ pb[k];
    bits += __popc(d);
    bytes += d != 0;
    lsb_eq += (d & 1) == 0;
  }
  block_add_u64(bits, out + 3 * blockIdx.y + 0, red);
  block_add_u64(bytes, out + 3 * blockIdx.y + 1, red);
  block_add_u64(lsb_eq, out + 3 * blockIdx.y + 2, red);
}

// 256-bin byte histogram per span: hist[256*i + v] += count of byte v in span i of `a`.
__global__ void __launch_bounds__(kStatCta)
    histogram_kernel(const uint8_t* __restrict__ a, const lorenz_span* __restrict__ spans,
                     uint64_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  const lorenz_span sp = spans[blockIdx.y];
  const uint64_t t0 = (uint64_t)blockIdx.x * kStatTile;
  if (t0 >= sp.len) return;
  const uint64_t t1 = (t0 + kStatTile < sp.len) ? t0 + kStatTile : sp.len;
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint8_t* pa = a + sp.a_off;
  uint64_t i = t0;
  if (((reinterpret_cast<uintptr_t>(pa + t0)) & 15) == 0) {
    const uint64_t v1 = t0 + ((t1 - t0) & ~15ULL);
    for (uint64_t k = t0 + 16 * threadIdx.x; k < v1; k += 16 * kStatCta) {
      const uint4 x = __ldcs(reinterpret_cast<const uint4*>(pa + k));
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int s = 0; s < 4; ++s) atomicAdd(&h[(w[q] >> (8 * s)) & 0xFF], 1u);
    }
    i = v1;
  }
  for (uint64_t k = i + threadIdx.x; k < t1; k += kStatCta) atomicAdd(&h[pa[k]], 1u);
  __syncthreads();
  if (h[threadIdx.x])
    atomicAdd(reinterpret_cast<unsigned long long*>(hist + 256 * blockIdx.y + threadIdx.x),
              (unsigned long long)h[threadIdx.x]);
}

}  // namespace lz
