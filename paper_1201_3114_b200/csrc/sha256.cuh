// sha256.cuh — SHA-256 compression (FIPS 180-4) for the product path (host + device).
// The paper keys Omega with "a hash function such as MD5 or SHA" (§3.1, Eq.7);
// reading Q11 fixes SHA-256. Written independently of the CPU oracle.
//
// Device use: the caller keeps the 16-word block in registers (all indices are
// compile-time after unrolling), the schedule is rolled in place.
#pragma once
#include <cstdint>

#ifndef LZ_HD
#define LZ_HD __host__ __device__ __forceinline__
#endif

namespace lz {

__host__ __device__ constexpr uint32_t kSha256K(int i) {
  constexpr uint32_t k[64] = {
      0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
      0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
      0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
      0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
      0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
      0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
      0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
      0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};
  return k[i];
}

LZ_HD uint32_t ror(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

struct Sha256State {
  uint32_t h[8];
  LZ_HD void init() {
    h[0] = 0x6a09e667u; h[1] = 0xbb67ae85u; h[2] = 0x3c6ef372u; h[3] = 0xa54ff53au;
    h[4] = 0x510e527fu; h[5] = 0x9b05688cu; h[6] = 0x1f83d9abu; h[7] = 0x5be0cd19u;
  }
  // One compression of the 16 big-endian message words w (w is clobbered).
  LZ_HD void compress(uint32_t w[16]) {
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], k = h[7];
#pragma unroll
    for (int t = 0; t < 64; ++t) {
      uint32_t wt;
      if (t < 16) {
        wt = w[t];
      } else {
        uint32_t w15 = w[(t - 15) & 15], w2 = w[(t - 2) & 15];
        uint32_t s0 = ror(w15, 7) ^ ror(w15, 18) ^ (w15 >> 3);
        uint32_t s1 = ror(w2, 17) ^ ror(w2, 19) ^ (w2 >> 10);
        wt = w[t & 15] + s0 + w[(t - 7) & 15] + s1;
        w[t & 15] = wt;
      }
      uint32_t t1 = k + (ror(e, 6) ^ ror(e, 11) ^ ror(e, 25)) + ((e & f) ^ (~e & g)) + kSha256K(t) + wt;
      uint32_t t2 = (ror(a, 2) ^ ror(a, 13) ^ ror(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
      k = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += k;
  }
};

// Host-side whole-message digest (used by keysetup; not on the device path).
inline void sha256_host(const uint8_t* msg, uint64_t len, uint8_t out[32]) {
  Sha256State s;
  s.init();
  uint64_t off = 0;
  uint32_t w[16];
  auto load = [&](const uint8_t* p) {
    for (int i = 0; i < 16; ++i)
      w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
  };
  for (; off + 64 <= len; off += 64) { load(msg + off); s.compress(w); }
  uint8_t last[128] = {0};
  uint64_t r = len - off;
  for (uint64_t i = 0; i < r; ++i) last[i] = msg[off + i];
  last[r] = 0x80;
  int nblk = (r + 9 <= 64) ? 1 : 2;
  uint64_t bits = len * 8;
  for (int i = 0; i < 8; ++i) last[64 * nblk - 1 - i] = (uint8_t)(bits >> (8 * i));
  for (int bk = 0; bk < nblk; ++bk) { load(last + 64 * bk); s.compress(w); }
  for (int i = 0; i < 8; ++i) {
    out[4 * i] = (uint8_t)(s.h[i] >> 24); out[4 * i + 1] = (uint8_t)(s.h[i] >> 16);
    out[4 * i + 2] = (uint8_t)(s.h[i] >> 8); out[4 * i + 3] = (uint8_t)s.h[i];
  }
}

}  // namespace lz
