// lorenz_device.cuh — device side of the per-block chaotic operation mode (sm_100a).
//
// One lane (thread) owns one block of the message: it derives the block's key
// (§3.1, Eqs.2-7), then runs the block's characters through Steps 1-3
// (§3.2) with the Lorenz state in registers, FP64 round-to-nearest and no
// FMA (__dadd_rn/__dmul_rn are never contracted), in the operation order of
// the same order the CPU oracle follows, so the outputs are
// bit-identical. Bytes stream through a per-warp shared-memory stage with coalesced
// 16-byte global loads/stores; warp shuffles reduce the per-block tags.
#pragma once
#include <cstdint>

#include "../../include/lorenz.h"
#include "sha256.cuh"

namespace lz {

// ------------------------------------------------------------------ launch data
struct DevKey {          // one stream password (by value for one message, array for a batch)
  uint32_t mid[8];       // FAST: SHA-256 midstate after the raw password's full 64-byte blocks
  uint32_t fin[32];      // FAST: final SHA-256 block(s) of pw || BE32(b) || padding, b slot zeroed
  uint32_t pw[6];        // STRONG: normalised password bytes as big-endian words, zero padded
  uint32_t fin_blocks;   // FAST: 1 or 2
  uint32_t b_off;        // FAST: byte offset of the BE32(b) slot inside fin
  uint32_t pw_len;       // STRONG: 3..23
  uint32_t pad_;
};

struct DevConst {
  double sigma, rho, beta, h, h2, h6;  // exact bit patterns from the key
  uint64_t n;                          // plaintext length of each message
  uint64_t B;                          // block size (STRONG: n)
  uint64_t b0;                         // first global block of this launch
  uint64_t lanes;                      // lanes (= blocks) in this launch
  uint64_t nb;                         // blocks per message (batch lane -> (message, block))
  uint64_t in_msg_stride, out_msg_stride;
  uint32_t n_it;                       // map iterations per character
  uint32_t fast;                       // 1: per-block sub-keys
  uint32_t batch;                      // 1: keys from the device array, tags per message; 2: ragged
  uint32_t variant;                    // NEXT-4 Step-3 reading (0 = Q13; see lorenz.h)
  // batch == 2 (ragged: messages of different lengths), device arrays over the `count` messages:
  const uint64_t* rag_blk;             // block prefix sums, count + 1 entries (lane -> message)
  const uint64_t* rag_len;             // plaintext lengths
  const uint64_t* rag_in;              // byte offset of each message in `in`
  const uint64_t* rag_out;             // byte offset of each message in `out`
  unsigned long long* rag_bad;         // decrypt / verify: min failing block per message
  uint32_t count;
};

enum { OP_ENC = 0, OP_DEC = 1, OP_VERIFY = 2 };
enum { ST_INTEGRITY = 1, ST_DIVERGENCE = 4 };

#ifndef LZ_CTA
#define LZ_CTA 128
#endif
constexpr int kCta = LZ_CTA;           // default 4 warps: one per SM sub-partition
constexpr int kWarps = kCta / 32;
constexpr int kWin = 64;               // characters per lane per staged window
constexpr int kRow = kWin + 16;        // smem row stride: per-lane 16-B reads are conflict-free
constexpr int kChunks = kWin / 16;

// "LORENZCHAOS-MAC1" (Q15) as two little-endian words.
constexpr uint64_t kSentLo = 0x48435A4E45524F4CULL;
constexpr uint64_t kSentHi = 0x3143414D2D534F41ULL;

__device__ __forceinline__ uint32_t sent_byte(uint32_t i) {
  return (uint32_t)(((i < 8) ? (kSentLo >> (8 * i)) : (kSentHi >> (8 * (i - 8)))) & 0xFF);
}

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// r[i] for i in {0,1,2}: two predicated selects, no branch
__device__ __forceinline__ double sel3(uint32_t i, double x, double y, double z) {
  double r = x;
  r = (i == 1) ? y : r;
  r = (i == 2) ? z : r;
  return r;
}

// big-endian byte i (0-based, i < 24) of six words; i is warp-uniform in practice
__device__ __forceinline__ uint32_t pw_byte(const uint32_t w[6], uint32_t i) {
  uint32_t q = i >> 2, word = w[0];
#pragma unroll
  for (int k = 1; k < 6; ++k) word = (q == (uint32_t)k) ? w[k] : word;
  return (word >> (24 - 8 * (i & 3))) & 0xFF;
}

// 10^e, e in [3, 8]: exact binary64 values (Theta's divisor)
__device__ __forceinline__ double pow10_theta(uint32_t e) {
  double v = 1e3;
  v = (e == 4) ? 1e4 : v;
  v = (e == 5) ? 1e5 : v;
  v = (e == 6) ? 1e6 : v;
  v = (e == 7) ? 1e7 : v;
  v = (e == 8) ? 1e8 : v;
  return v;
}

// 10^ceil(log10 2^{8(L+1)}) for L = 1..7 (g of P:209): 1e5,1e8,1e10,1e13,1e15,1e17,1e20
__device__ __forceinline__ double g_divisor(uint32_t L) {
  double v = 1e5;
  v = (L == 2) ? 1e8 : v;
  v = (L == 3) ? 1e10 : v;
  v = (L == 4) ? 1e13 : v;
  v = (L == 5) ? 1e15 : v;
  v = (L == 6) ? 1e17 : v;
  v = (L == 7) ? 1e20 : v;
  return v;
}

// floor(|alpha| * 10^13) of the rounded product (Eq.8, Q8, Q9). The product is one DMUL;
// the floor is taken from its bit pattern on the integer pipes (equal to F2I.U64.TRUNC for
// every product below 2^53; inside the guard box the product is < 2^51, Q7).
__device__ __forceinline__ uint64_t quantise(double alpha) {
  const uint64_t bits = (uint64_t)__double_as_longlong(dmul(fabs(alpha), 1e13));
  const int e = (int)(bits >> 52) - 1023;  // unbiased exponent (sign bit is clear)
  const uint64_t mant = (bits & 0xFFFFFFFFFFFFFULL) | (1ULL << 52);
  // branch-free; e < 0 shifts everything out (52 - e >= 53). Exact for every product below
  // 2^53: inside the guard box (|coordinates| <= 150) products are < 2^51; outside it the
  // chain is already flagged DIVERGENCE (Q18) and its bytes are not defined.
  return mant >> (uint32_t)min(max(52 - e, 0), 63);
}

// x mod k for x < 1024, 1 <= k <= 6, with inv = ceil(2^16 / k): one multiply instead of
// a division (floor(x/k) = (x inv) >> 16 since x (inv - 2^16/k) / 2^16 < 1/64 < 1/k).
__device__ __forceinline__ uint32_t small_mod(uint32_t x, uint32_t k, uint32_t inv) {
  return x - k * ((x * inv) >> 16);
}

// Guard box of Q18 on the integer pipes: |x| <= 100, |y| <= 100, -50 <= z <= 150, all
// finite (NaN / inf bit patterns compare above every finite bound).
__device__ __forceinline__ bool in_guard_box(double x, double y, double z) {
  constexpr uint64_t kAbs = 0x7FFFFFFFFFFFFFFFULL;
  constexpr uint64_t k100 = 0x4059000000000000ULL, k150 = 0x4062C00000000000ULL, k50 = 0x4049000000000000ULL;
  const uint64_t bx = (uint64_t)__double_as_longlong(x) & kAbs, by = (uint64_t)__double_as_longlong(y) & kAbs;
  const uint64_t rz = (uint64_t)__double_as_longlong(z), bz = rz & kAbs;
  return (bx <= k100) & (by <= k100) & (bz <= ((rz >> 63) ? k50 : k150));
}

__device__ __forceinline__ uint32_t rbyte(uint64_t m, uint32_t omega) {
  return (uint32_t)(m >> (8 * omega)) & 0xFF;
}

// ------------------------------------------------------------------ chain state
struct Chain {
  double x, y, z;          // r
  double apx, apy, apz;    // a', added after every character
  uint64_t m1, m2;         // floor(|alpha_1,2| 10^13) feeding Step 1
  uint64_t m3;             // floor(|alpha_3| 10^13) (used by the literal-order variant)
  uint32_t mu1, mu2, mu3;
  uint32_t om1, om2, om3;  // Eq.7
  uint32_t k1, k2, k3;     // k1,k2 and k3 of Step 3
  uint32_t ik1, ik2, ik3;  // ceil(2^16 / k) for small_mod
};

// Key schedule of one stream password. FAST derives the block password
// SHA-256(pw || BE32 b)[0:18] from the midstate first (Q16). All hashes run
// through one in-register compression inside a job loop (small code, no local memory).
__device__ __forceinline__ void key_schedule(const DevKey& K, bool fast, uint32_t b, uint32_t variant,
                                             Chain& ch) {
  uint32_t pw[6];
  uint32_t np;
  Sha256State s;
  if (fast) {
#pragma unroll
    for (int i = 0; i < 8; ++i) s.h[i] = K.mid[i];
    const uint32_t q = K.b_off >> 2, sh = K.b_off & 3;
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      if (blk < (int)K.fin_blocks) {
        uint32_t w[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const uint32_t wi = 16 * blk + k;
          uint32_t v = K.fin[16 * blk + k];
          if (wi == q) v |= sh ? (b >> (8 * sh)) : b;
          if (sh && wi == q + 1) v |= b << (8 * (4 - sh));
          w[k] = v;
        }
        s.compress(w);
      }
    }
    pw[0] = s.h[0]; pw[1] = s.h[1]; pw[2] = s.h[2]; pw[3] = s.h[3];
    pw[4] = s.h[4] & 0xFFFF0000u; pw[5] = 0;
    np = 18;
  } else {
#pragma unroll
    for (int i = 0; i < 6; ++i) pw[i] = K.pw[i];
    np = K.pw_len;
  }

  // Eqs.2-4: L = floor(n/3), little-endian digit groups + remainder bytes
  const uint32_t L = np / 3, rem = np - 3 * L;
  uint64_t g1 = 0, g2 = 0, g3 = 0;
#pragma unroll
  for (uint32_t j = 0; j < 7; ++j) {
    if (j < L) {
      g1 |= (uint64_t)pw_byte(pw, j) << (8 * j);
      g2 |= (uint64_t)pw_byte(pw, L + j) << (8 * j);
      g3 |= (uint64_t)pw_byte(pw, 2 * L + j) << (8 * j);
    }
  }
  const uint64_t a1 = rem == 0 ? g1 : ((g1 << 8) | pw_byte(pw, 3 * L));
  const uint64_t a2 = rem == 2 ? ((g2 << 8) | pw_byte(pw, 3 * L + 1)) : g2;
  const uint64_t a3 = g3;

  // a' = g(a)
  const double gd = g_divisor(L);
  ch.apx = __ddiv_rn(__ull2double_rn(a1), gd);
  ch.apy = __ddiv_rn(__ull2double_rn(a2), gd);
  ch.apz = __ddiv_rn(__ull2double_rn(a3), gd);

  // jobs: 0 = SHA-256(pi_b) for k (Q12); 1..3 = lambda_i (Q10); 4..6 = Omega_i (Eq.7, Q11)
  double lam1 = 0, lam2 = 0, lam3 = 0;
  uint32_t hk = 0;
  uint64_t ho1 = 0, ho2 = 0, ho3 = 0;
#pragma unroll 1
  for (uint32_t job = 0; job < 7; ++job) {
    uint32_t w[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) w[k] = 0;
    if (job == 0) {
#pragma unroll
      for (int k = 0; k < 6; ++k) w[k] = pw[k];
      const uint32_t q = np >> 2, bit = 24 - 8 * (np & 3);
#pragma unroll
      for (int k = 0; k < 6; ++k) w[k] |= (q == (uint32_t)k) ? (0x80u << bit) : 0u;
      w[15] = np * 8;
    } else if (job <= 3) {
      // 0x4C || BE64 a1 || BE64 a2 || BE64 a3 || u8 i || 0x80 ... || len=208
      const uint32_t i = job;
      w[0] = 0x4C000000u | (uint32_t)(a1 >> 40);
      w[1] = (uint32_t)(a1 >> 8);
      w[2] = ((uint32_t)a1 << 24) | (uint32_t)(a2 >> 40);
      w[3] = (uint32_t)(a2 >> 8);
      w[4] = ((uint32_t)a2 << 24) | (uint32_t)(a3 >> 40);
      w[5] = (uint32_t)(a3 >> 8);
      w[6] = ((uint32_t)a3 << 24) | (i << 16) | 0x8000u;
      w[15] = 26 * 8;
    } else {
      // BE64(i a1) || BE64(i a2) || BE64(i a3), products mod 2^64, len=192
      const uint64_t i = job - 3;
      const uint64_t p1 = i * a1, p2 = i * a2, p3 = i * a3;
      w[0] = (uint32_t)(p1 >> 32); w[1] = (uint32_t)p1;
      w[2] = (uint32_t)(p2 >> 32); w[3] = (uint32_t)p2;
      w[4] = (uint32_t)(p3 >> 32); w[5] = (uint32_t)p3;
      w[6] = 0x80000000u;
      w[15] = 24 * 8;
    }
    s.init();
    s.compress(w);
    const uint64_t h64 = ((uint64_t)s.h[0] << 32) | s.h[1];
    if (job == 0) {
      hk = s.h[0];
    } else if (job <= 3) {
      // lambda_i = lo_i + (double(h) 2^-64)(hi_i - lo_i)  (P:216 ranges; Q10)
      const double lo = job == 1 ? -15.67 : (job == 2 ? -11.28 : 0.090);
      const double hi = job == 1 ? 16.01 : (job == 2 ? 16.01 : 62.000);
      const double t = dmul(__ull2double_rn(h64), 0x1p-64);
      const double lam = dadd(lo, dmul(t, dsub(hi, lo)));
      if (job == 1) lam1 = lam; else if (job == 2) lam2 = lam; else lam3 = lam;
    } else {
      if (job == 4) ho1 = h64; else if (job == 5) ho2 = h64; else ho3 = h64;
    }
  }
  // k_i = 3 + H[i-1] mod 2; k3 of Step 3 = 1 + H[3] mod 6 (Q12)
  const uint32_t k1i = 3 + ((hk >> 24) & 1), k3i = 3 + ((hk >> 8) & 1);
  // NEXT-4 "distinct k": k2 = 7 - k1
  const uint32_t k2i = (variant & LORENZ_V_DISTINCT_K) ? 7 - k1i : 3 + ((hk >> 16) & 1);
  ch.k1 = k1i;
  ch.k2 = k2i;
  ch.k3 = 1 + (hk & 0xFF) % 6;
  ch.ik1 = (65535 + ch.k1) / ch.k1;
  ch.ik2 = (65535 + ch.k2) / ch.k2;
  ch.ik3 = (65535 + ch.k3) / ch.k3;
  ch.om1 = (uint32_t)(ho1 % k1i);
  ch.om2 = (uint32_t)(ho2 % k2i);
  ch.om3 = (uint32_t)(ho3 % k3i);
  // mu, over the integers, reduced mod 3
  const uint64_t r1 = a1 % 3, r2 = a2 % 3, r3 = a3 % 3;
  ch.mu1 = (uint32_t)((r1 + r2 + r3) % 3);
  ch.mu2 = (uint32_t)((r1 * r2 + r3) % 3);
  ch.mu3 = (uint32_t)((r1 + r2 * r3) % 3);
  // r0 = a' + lambda (Eq.5); alpha0 = r0[mu] (Eq.6, n = 0, Q14)
  ch.x = dadd(ch.apx, lam1);
  ch.y = dadd(ch.apy, lam2);
  ch.z = dadd(ch.apz, lam3);
  ch.m1 = quantise(sel3(ch.mu1, ch.x, ch.y, ch.z));
  ch.m2 = quantise(sel3(ch.mu2, ch.x, ch.y, ch.z));
  ch.m3 = quantise(sel3(ch.mu3, ch.x, ch.y, ch.z));
}

// n_it steps of the Lorenz map. RK4 in the canonical order of DESIGN.md §2
// (43 DADD + 32 DMUL per step, no FMA), or forward Euler (NEXT-1).
#ifndef LZ_EULER_UNROLL
#define LZ_EULER_UNROLL 4
#endif
// One forward-Euler step s' = s + f(s) h in the RHS order of DESIGN.md §2 (15 ops).
__device__ __forceinline__ void euler_step(double& x, double& y, double& z, double S, double R, double Bt,
                                           double h) {
  const double fx = dmul(S, dsub(y, x));
  const double fy = dsub(dsub(dmul(R, x), y), dmul(x, z));
  const double fz = dsub(dmul(x, y), dmul(Bt, z));
  x = dadd(x, dmul(fx, h));
  y = dadd(y, dmul(fy, h));
  z = dadd(z, dmul(fz, h));
}

// PIN (the balanced kernel): pass the six constants through an opaque x + 0.0 (exact: all are
// positive) once per character, so they sit in registers for the loop. Without it ptxas
// re-reads them from the constant bank inside the RK4 loop of that kernel's cut-unit paths
// (3 LDCU.128 per step, 81 instead of 78 instructions); the wave kernel keeps them in uniform
// registers by itself.
// Not for the FMA form: its three-operand DFMAs then read the constants from the general register
// file and lose issue slots to register-bank conflicts; ptxas's per-step reload of the constants
// into uniform registers (3 LDCU.128, off the FP64 pipe) costs far less (C3 in the balanced kernel:
// 85.3 % -> 94.4 % of the FP64 pipe, tools/tune.py). Bit i of LZ_PIN_MASK pins integrator i.
#ifndef LZ_PIN_MASK
#define LZ_PIN_MASK 3
#endif
#ifndef LZ_IMM_CONST
#define LZ_IMM_CONST 3  // bit i: integrator i takes sigma, rho, beta as compile-time operands
#endif
template <int INTEG, bool PIN = false>
__device__ __forceinline__ void integrate(double& x, double& y, double& z, const DevConst& C) {
  // IMM (RK4, Euler): sigma = 10, rho = 28 and beta = RN(8/3) are fixed by the cipher (every key
  // holds these bit patterns, lorenz_keysetup) and enter as compile-time operands: 10 and 28 become FP64
  // immediates, beta a uniform register, so each step's DMUL/DADDs read 3 fewer general registers
  // (C4 98.07 % -> 98.87 % of the FP64 pipe, C3 98.03 -> 98.65, Euler C3 92.1 -> 93.0; tools/tune.py,
  // profiles/tune_r02.jsonl). Not for the FMA form, whose 256 MiB launch lost 1.3 points with it.
  constexpr bool IMM = (LZ_IMM_CONST >> INTEG) & 1;
  constexpr double kSigma = 10.0, kRho = 28.0, kBeta = 0x1.5555555555555p+1;  // RN(8/3)
  double S = IMM ? kSigma : C.sigma, R = IMM ? kRho : C.rho, Bt = IMM ? kBeta : C.beta;
  // (h, h/2, h/6 as compile-time operands too — a dt-specialised loop — measured 0.45 % slower: the
  // loop then spends 8 UMOVs per step on them; profiles/tune_r02.jsonl, tag "fixdt")
  double h = C.h, h2 = C.h2, h6 = C.h6;
  if (PIN && ((LZ_PIN_MASK >> INTEG) & 1)) {
    if (!IMM) {
      asm volatile("add.rn.f64 %0, %0, 0d0000000000000000;" : "+d"(S));
      asm volatile("add.rn.f64 %0, %0, 0d0000000000000000;" : "+d"(R));
      asm volatile("add.rn.f64 %0, %0, 0d0000000000000000;" : "+d"(Bt));
    }
    asm volatile("add.rn.f64 %0, %0, 0d0000000000000000;" : "+d"(h));
    asm volatile("add.rn.f64 %0, %0, 0d0000000000000000;" : "+d"(h2));
    asm volatile("add.rn.f64 %0, %0, 0d0000000000000000;" : "+d"(h6));
  }
  if constexpr (INTEG == LORENZ_EULER) {
    // forward Euler (NEXT-1): 15 ops per step, so the loop's own 3 instructions are worth
    // unrolling away (C3 88 % -> 92 %, C4 93.8 % -> 94.5 % of the FP64 pipe)
    uint32_t it = 0;
#pragma unroll 1
    for (; it + LZ_EULER_UNROLL <= C.n_it; it += LZ_EULER_UNROLL) {
#pragma unroll
      for (int u = 0; u < LZ_EULER_UNROLL; ++u) euler_step(x, y, z, S, R, Bt, h);
    }
#pragma unroll 1
    for (; it < C.n_it; ++it) euler_step(x, y, z, S, R, Bt, h);
  } else {
#pragma unroll 1
    for (uint32_t it = 0; it < C.n_it; ++it) {
      if constexpr (INTEG == LORENZ_RK4) {
        const double k1x = dmul(S, dsub(y, x));
        const double k1y = dsub(dsub(dmul(R, x), y), dmul(x, z));
        const double k1z = dsub(dmul(x, y), dmul(Bt, z));
        const double ax = dadd(x, dmul(h2, k1x)), ay = dadd(y, dmul(h2, k1y)), az = dadd(z, dmul(h2, k1z));
        const double k2x = dmul(S, dsub(ay, ax));
        const double k2y = dsub(dsub(dmul(R, ax), ay), dmul(ax, az));
        const double k2z = dsub(dmul(ax, ay), dmul(Bt, az));
        const double bx = dadd(x, dmul(h2, k2x)), by = dadd(y, dmul(h2, k2y)), bz = dadd(z, dmul(h2, k2z));
        const double k3x = dmul(S, dsub(by, bx));
        const double k3y = dsub(dsub(dmul(R, bx), by), dmul(bx, bz));
        const double k3z = dsub(dmul(bx, by), dmul(Bt, bz));
        const double cx = dadd(x, dmul(h, k3x)), cy = dadd(y, dmul(h, k3y)), cz = dadd(z, dmul(h, k3z));
        const double k4x = dmul(S, dsub(cy, cx));
        const double k4y = dsub(dsub(dmul(R, cx), cy), dmul(cx, cz));
        const double k4z = dsub(dmul(cx, cy), dmul(Bt, cz));
        double sx = dadd(k1x, k2x), sy = dadd(k1y, k2y), sz = dadd(k1z, k2z);
        sx = dadd(sx, k2x); sy = dadd(sy, k2y); sz = dadd(sz, k2z);
        sx = dadd(sx, k3x); sy = dadd(sy, k3y); sz = dadd(sz, k3z);
        sx = dadd(sx, k3x); sy = dadd(sy, k3y); sz = dadd(sz, k3z);
        sx = dadd(sx, k4x); sy = dadd(sy, k4y); sz = dadd(sz, k4z);
        x = dadd(x, dmul(h6, sx));
        y = dadd(y, dmul(h6, sy));
        z = dadd(z, dmul(h6, sz));
      } else {
        // NEXT-3: same RK4, fused multiply-adds at fixed sites; 45 pipe ops
        const double k1x = dmul(S, dsub(y, x));
        const double k1y = __fma_rn(-x, z, __fma_rn(R, x, -y));
        const double k1z = __fma_rn(x, y, -dmul(Bt, z));
        const double ax = __fma_rn(h2, k1x, x), ay = __fma_rn(h2, k1y, y), az = __fma_rn(h2, k1z, z);
        const double k2x = dmul(S, dsub(ay, ax));
        const double k2y = __fma_rn(-ax, az, __fma_rn(R, ax, -ay));
        const double k2z = __fma_rn(ax, ay, -dmul(Bt, az));
        const double bx = __fma_rn(h2, k2x, x), by = __fma_rn(h2, k2y, y), bz = __fma_rn(h2, k2z, z);
        const double k3x = dmul(S, dsub(by, bx));
        const double k3y = __fma_rn(-bx, bz, __fma_rn(R, bx, -by));
        const double k3z = __fma_rn(bx, by, -dmul(Bt, bz));
        const double cx = __fma_rn(h, k3x, x), cy = __fma_rn(h, k3y, y), cz = __fma_rn(h, k3z, z);
        const double k4x = dmul(S, dsub(cy, cx));
        const double k4y = __fma_rn(-cx, cz, __fma_rn(R, cx, -cy));
        const double k4z = __fma_rn(cx, cy, -dmul(Bt, cz));
        const double sx = dadd(__fma_rn(2.0, k3x, __fma_rn(2.0, k2x, k1x)), k4x);
        const double sy = dadd(__fma_rn(2.0, k3y, __fma_rn(2.0, k2y, k1y)), k4y);
        const double sz = dadd(__fma_rn(2.0, k3z, __fma_rn(2.0, k2z, k1z)), k4z);
        x = __fma_rn(h6, sx, x);
        y = __fma_rn(h6, sy, y);
        z = __fma_rn(h6, sz, z);
      }
    }
  }
}

// Steps 2-3 after the character's plaintext byte p is known (Q13).
// Returns false if the guard of Q18 fails.
template <int INTEG, bool PIN = false>
__device__ __forceinline__ bool advance(Chain& ch, uint32_t p, const DevConst& C, const double* theta_tab) {
  // Step 2: Theta = P_i / 10^{3+Omega_3} (correctly rounded, Q19; from the per-CTA table of
  // __ddiv_rn quotients) added to r[mu_3]
  const double theta = theta_tab[ch.om3 * 256 + p];
  const double t = dadd(sel3(ch.mu3, ch.x, ch.y, ch.z), theta);
  ch.x = ch.mu3 == 0 ? t : ch.x;
  ch.y = ch.mu3 == 1 ? t : ch.y;
  ch.z = ch.mu3 == 2 ? t : ch.z;
  integrate<INTEG, PIN>(ch.x, ch.y, ch.z, C);
  const bool ok = in_guard_box(ch.x, ch.y, ch.z);
  const uint32_t order = C.variant & 3;  // warp-uniform
  if (order == LORENZ_V_LITERAL) {
    // NEXT-4 literal order: mu from the previous alpha, alpha from the new mu, then Omega
    ch.mu1 = (ch.mu1 + rbyte(ch.m1, ch.om1)) % 3;
    ch.mu2 = (ch.mu2 + rbyte(ch.m2, ch.om2)) % 3;
    ch.mu3 = (ch.mu3 + rbyte(ch.m3, ch.om3)) % 3;
    ch.m1 = quantise(sel3(ch.mu1, ch.x, ch.y, ch.z));
    ch.m2 = quantise(sel3(ch.mu2, ch.x, ch.y, ch.z));
    ch.m3 = quantise(sel3(ch.mu3, ch.x, ch.y, ch.z));
    ch.om1 = small_mod(ch.om1 + rbyte(ch.m1, ch.om1), ch.k1, ch.ik1);
    ch.om2 = small_mod(ch.om2 + rbyte(ch.m2, ch.om2), ch.k2, ch.ik2);
    ch.om3 = small_mod(ch.om3 + rbyte(ch.m3, ch.om3), ch.k3, ch.ik3);
  } else {
    // Step 3 (Q13): alpha_i = r[mu_i]; R_i = R(alpha_i, Omega_i); mu, Omega += R_i
    const uint64_t m1 = quantise(sel3(ch.mu1, ch.x, ch.y, ch.z));
    const uint64_t m2 = quantise(sel3(ch.mu2, ch.x, ch.y, ch.z));
    const uint64_t m3 = quantise(sel3(ch.mu3, ch.x, ch.y, ch.z));
    const uint32_t R1 = rbyte(m1, ch.om1), R2 = rbyte(m2, ch.om2), R3 = rbyte(m3, ch.om3);
    ch.mu1 = (ch.mu1 + R1) % 3;
    ch.mu2 = (ch.mu2 + R2) % 3;
    ch.mu3 = (ch.mu3 + R3) % 3;
    if (order == LORENZ_V_CYCLIC) {  // NEXT-4: Omega_i takes its byte from alpha_{i+1}
      ch.om1 = small_mod(ch.om1 + rbyte(m2, ch.om1), ch.k1, ch.ik1);
      ch.om2 = small_mod(ch.om2 + rbyte(m3, ch.om2), ch.k2, ch.ik2);
      ch.om3 = small_mod(ch.om3 + rbyte(m1, ch.om3), ch.k3, ch.ik3);
    } else {
      ch.om1 = small_mod(ch.om1 + R1, ch.k1, ch.ik1);
      ch.om2 = small_mod(ch.om2 + R2, ch.k2, ch.ik2);
      ch.om3 = small_mod(ch.om3 + R3, ch.k3, ch.ik3);
    }
    ch.m1 = m1;
    ch.m2 = m2;
    ch.m3 = m3;
  }
  // r_n = r_n + a'
  ch.x = dadd(ch.x, ch.apx);
  ch.y = dadd(ch.y, ch.apy);
  ch.z = dadd(ch.z, ch.apz);
  return ok;
}

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  return v;
}

__device__ __forceinline__ uint4 ld_stream(const uint8_t* p) {
  return __ldcs(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ void st_stream(uint8_t* p, uint4 v) {
  __stcs(reinterpret_cast<uint4*>(p), v);
}

#ifndef LZ_MIN_CTAS
#define LZ_MIN_CTAS 1
#endif
// Resident CTAs per SM (tools/tune.py sweeps). RK4 and Euler: 16 warps per SM (<= 128
// registers) as 4 CTAs of 128 threads or 2 of 256 — the host picks the CTA size per launch
// (lorenz.cu: chain_cta). The FMA form gains 2 points (92.7 % -> 94.8 % of the FP64 pipe
// on C4) from a fifth 128-thread CTA (<= 102 registers).
template <int INTEG, int CTA>
constexpr int min_ctas() {
  return INTEG == LORENZ_RK4_FMA ? 5 : (LZ_MIN_CTAS > 1 ? LZ_MIN_CTAS : 512 / CTA);
}

// ------------------------------------------------------------------ per-lane pieces
// Where lane g of a launch reads and writes: message s, global block bl, block rb inside
// the slice, the lane's input/output rows, and its character count (block + sentinel).
struct LaneIO {
  const uint8_t* irow;
  uint8_t* orow;
  uint64_t s, bl, rb, len, total;  // total = len + 16 characters; 0 for an inactive lane
  bool active;
};

template <int OP>
__device__ __forceinline__ LaneIO lane_io(const DevConst& C, const uint8_t* in, uint8_t* out, uint64_t g) {
  LaneIO io;
  io.active = g < C.lanes;
  uint64_t s = 0, bl = C.b0 + g, msg_n = C.n;
  if (C.batch == 1) { s = g / C.nb; bl = g - s * C.nb; }
  if (C.batch == 2 && io.active) {  // ragged: the message whose block range holds g (binary search)
    uint32_t lo = 0, hi = C.count;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (C.rag_blk[mid] <= g) lo = mid; else hi = mid;
    }
    s = lo;
    bl = g - C.rag_blk[lo];
    msg_n = C.rag_len[lo];
  }
  uint64_t len = 0;
  if (io.active) {
    const uint64_t start = C.fast ? bl * C.B : 0;
    len = C.fast ? ((msg_n - start) < C.B ? (msg_n - start) : C.B) : msg_n;
  }
  io.s = s;
  io.bl = bl;
  io.len = len;
  io.total = io.active ? len + 16 : 0;
  io.rb = bl - C.b0;
  io.irow = in + s * C.in_msg_stride + io.rb * (OP == OP_ENC ? C.B : C.B + 16);
  io.orow = out + s * C.out_msg_stride + io.rb * (OP == OP_ENC ? C.B + 16 : C.B);
  if (C.batch == 2) {
    io.irow = in + (io.active ? C.rag_in[s] : 0) + bl * (OP == OP_ENC ? C.B : C.B + 16);
    io.orow = out + (io.active ? C.rag_out[s] : 0) + bl * (OP == OP_ENC ? C.B + 16 : C.B);
  }
  if (!io.active) { io.irow = in; io.orow = out; }
  return io;
}

// What a lane accumulates over its characters besides the chain itself.
struct LaneAcc {
  uint64_t tlo, thi;  // last 16 ciphertext bytes = the block tag
  bool guard_ok, bad;
};

// Stage-in of one window: chunk c of row `row` (16 bytes at w0 + 16 c), zero past the lane's
// characters and (SEG) past the window limit wlim; the sentinel bytes are synthesised on encrypt.
template <int OP, int WIN, bool SEG>
__device__ __forceinline__ void stage_load(const LaneIO& io, uint64_t w0, uint64_t wlim, uint32_t lane,
                                           uint4 (&v)[WIN / 16]) {
  constexpr int CHUNKS = WIN / 16;
#pragma unroll
  for (int it = 0; it < CHUNKS; ++it) {
    const uint32_t q = it * 32 + lane, row = q / CHUNKS, c = q % CHUNKS;
    const uint8_t* r_in = (const uint8_t*)__shfl_sync(0xffffffffu, (unsigned long long)io.irow, row);
    const uint64_t r_len = __shfl_sync(0xffffffffu, io.len, row);
    const uint64_t r_tot = __shfl_sync(0xffffffffu, io.total, row);
    const uint64_t pos = w0 + 16 * c;
    v[it] = make_uint4(0, 0, 0, 0);
    if (pos < r_tot && (!SEG || pos < wlim)) {
      const uint64_t r_src = (OP == OP_ENC) ? r_len : r_tot;  // bytes readable from memory
      if (pos + 16 <= r_src) {
        v[it] = ld_stream(r_in + pos);
      } else if (OP == OP_ENC && pos >= r_len && ((r_len & 15) == 0)) {
        v[it] = make_uint4((uint32_t)kSentLo, (uint32_t)(kSentLo >> 32), (uint32_t)kSentHi,
                           (uint32_t)(kSentHi >> 32));
      } else {
        uint32_t wv[4] = {0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint64_t j = pos + i;
          uint32_t bv = 0;
          if (j < r_src) bv = r_in[j];
          else if (OP == OP_ENC && j < r_tot) bv = sent_byte((uint32_t)(j - r_len));
          wv[i >> 2] |= bv << (8 * (i & 3));
        }
        v[it] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      }
    }
  }
}

// Characters [c0, c1) of every lane of the warp: stage in, run the chain, stage out, one
// WIN-character window at a time. c0 is a multiple of 16; c1 is a multiple of 16 (SEG: the
// balanced kernel, which also keeps its constants in registers, see integrate) or at least
// every lane's total (the wave kernel). Lanes stop at their own total. Warp-uniform control flow.
// (Issuing the next window's loads before this window's characters — a register prefetch — measured
// no faster, even with the buffers in mapped host memory: other warps cover the wait.)
template <int OP, int INTEG, int WIN, bool SEG = false>
__device__ __forceinline__ void run_chars(const DevConst& C, const LaneIO& io, Chain& ch, LaneAcc& acc,
                                          uint8_t* wst, const double* theta_tab, uint64_t c0, uint64_t c1,
                                          uint32_t lane) {
  constexpr int ROW = WIN + 16, CHUNKS = WIN / 16;
  for (uint64_t w0 = c0; w0 < c1; w0 += WIN) {
    // this window's end inside [c0, c1). SEG (the balanced kernel) cuts units inside windows;
    // the wave kernel's c1 covers every lane's total, so the lane bounds alone suffice there
    // (and leaving the checks out keeps its register allocation: RK4-FMA 92.8 % -> 95.0 %)
    const uint64_t wlim = (!SEG || w0 + WIN < c1) ? w0 + WIN : c1;
    // ---- stage in: 32 rows x WIN bytes, coalesced 16-B chunks ----
    uint4 v[CHUNKS];
    stage_load<OP, WIN, SEG>(io, w0, wlim, lane, v);
#pragma unroll
    for (int it = 0; it < CHUNKS; ++it) {
      const uint32_t q = it * 32 + lane, row = q / CHUNKS, c = q % CHUNKS;
      *reinterpret_cast<uint4*>(wst + row * ROW + 16 * c) = v[it];
    }
    __syncwarp();

    // ---- the chain over this lane's characters [w0, min(wlim, total)) ----
    if (w0 < io.total) {
      const uint64_t wend = (wlim < io.total) ? wlim : io.total;
      for (uint64_t j0 = w0; j0 < wend; j0 += 16) {
        uint4* cell = reinterpret_cast<uint4*>(wst + lane * ROW + (j0 - w0));
        const uint4 v = *cell;
        uint64_t ilo = (uint64_t)v.x | ((uint64_t)v.y << 32), ihi = (uint64_t)v.z | ((uint64_t)v.w << 32);
        uint64_t olo = 0, ohi = 0;
        const uint32_t cnt = (uint32_t)((wend - j0) < 16 ? (wend - j0) : 16);
        for (uint32_t i = 0; i < cnt; ++i) {
          const uint64_t j = j0 + i;
          const uint32_t xin = (uint32_t)ilo & 0xFF;
          ilo = (ilo >> 8) | (ihi << 56);
          ihi >>= 8;
          // Step 1 (Eqs.8-10): keystream sum_{i=1,2} R(alpha_i, Omega_i)
          const uint32_t ks = rbyte(ch.m1, ch.om1) + rbyte(ch.m2, ch.om2);
          uint32_t yout, p, cbyte;
          if (OP == OP_ENC) {
            yout = (xin + ks) & 0xFF; p = xin; cbyte = yout;
          } else {
            yout = (xin - ks) & 0xFF; p = yout; cbyte = xin;
            if (j >= io.len) acc.bad |= (yout != sent_byte((uint32_t)(j - io.len)));
          }
          olo = (olo >> 8) | (ohi << 56);
          ohi = (ohi >> 8) | ((uint64_t)yout << 56);
          acc.tlo = (acc.tlo >> 8) | (acc.thi << 56);
          acc.thi = (acc.thi >> 8) | ((uint64_t)cbyte << 56);
          if (j + 1 == io.total) break;  // the last character is not advanced (Q20)
          acc.guard_ok &= advance<INTEG, SEG>(ch, p, C, theta_tab);
        }
        if (cnt < 16) {  // left-align a partial chunk
          const uint32_t sh = 8 * (16 - cnt);
          if (sh >= 64) { olo = ohi >> (sh - 64); ohi = 0; }
          else { olo = (olo >> sh) | (ohi << (64 - sh)); ohi >>= sh; }
        }
        *cell = make_uint4((uint32_t)olo, (uint32_t)(olo >> 32), (uint32_t)ohi, (uint32_t)(ohi >> 32));
      }
    }
    __syncwarp();

    // ---- stage out ----
    if (OP != OP_VERIFY) {
#pragma unroll
      for (int it = 0; it < CHUNKS; ++it) {
        const uint32_t q = it * 32 + lane, row = q / CHUNKS, c = q % CHUNKS;
        uint8_t* r_out = (uint8_t*)__shfl_sync(0xffffffffu, (unsigned long long)io.orow, row);
        const uint64_t r_len = __shfl_sync(0xffffffffu, io.len, row);
        const uint64_t r_tot = __shfl_sync(0xffffffffu, io.total, row);
        const uint64_t r_dst = (OP == OP_ENC) ? r_tot : r_len;
        const uint64_t pos = w0 + 16 * c;
        if (r_tot && pos < r_dst && (!SEG || pos < wlim)) {
          const uint4 v = *reinterpret_cast<const uint4*>(wst + row * ROW + 16 * c);
          if (pos + 16 <= r_dst) {
            st_stream(r_out + pos, v);
          } else {
            const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (pos + i < r_dst) r_out[pos + i] = (uint8_t)(wv[i >> 2] >> (8 * (i & 3)));
          }
        }
      }
    }
    __syncwarp();
  }
}

// Per-block verdicts and the tag combine once a warp's lanes have run their last character.
template <int OP>
__device__ __forceinline__ void finish_lanes(const DevConst& C, const LaneIO& io, LaneAcc acc,
                                             lorenz_result* __restrict__ res, uint8_t* __restrict__ tags_batch,
                                             uint8_t* __restrict__ block_ok, uint32_t lane) {
  if (io.active) {
    if (!acc.guard_ok) atomicOr(&res->status, (uint32_t)ST_DIVERGENCE);
    if (OP != OP_ENC) {
      if (acc.bad) {
        atomicMin((unsigned long long*)&res->first_bad, (unsigned long long)io.bl);
        if (C.batch == 2) atomicMin(C.rag_bad + io.s, (unsigned long long)io.bl);
        atomicOr(&res->status, (uint32_t)ST_INTEGRITY);
        if (OP == OP_DEC)  // never release unauthenticated plaintext
          for (uint64_t j = 0; j < io.len; ++j) io.orow[j] = 0;
      }
      if (block_ok) block_ok[io.rb] = acc.bad ? 0 : 1;
    }
  }
  if (C.batch) {
    if (io.active) {
      unsigned long long* t = reinterpret_cast<unsigned long long*>(tags_batch + 16 * io.s);
      atomicXor(t, (unsigned long long)acc.tlo);
      atomicXor(t + 1, (unsigned long long)acc.thi);
    }
  } else {
    uint64_t tlo = acc.tlo, thi = acc.thi;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tlo ^= __shfl_xor_sync(0xffffffffu, tlo, o);
      thi ^= __shfl_xor_sync(0xffffffffu, thi, o);
    }
    if (lane == 0 && (tlo | thi)) {
      unsigned long long* t = reinterpret_cast<unsigned long long*>(res->tag_xor);
      atomicXor(t, (unsigned long long)tlo);
      atomicXor(t + 1, (unsigned long long)thi);
    }
  }
}

// RN(p / 10^{3+e}) for e = Omega_3 in [0,6) and p a byte, once per CTA (Step 2, Q19)
template <int CTA>
__device__ __forceinline__ void fill_theta(double* theta_tab) {
  for (uint32_t i = threadIdx.x; i < 6 * 256; i += CTA)
    theta_tab[i] = __ddiv_rn(__uint2double_rn(i & 255), pow10_theta(3 + (i >> 8)));
}

// ------------------------------------------------------------------ the wave kernel
// OP: OP_ENC / OP_DEC / OP_VERIFY; CTA: 128, 256 or 512 threads. One lane per block, one
// warp per 32 consecutive blocks; warps are independent (only __syncwarp), so the CTA never
// waits on its slowest warp.
template <int OP, int INTEG, int CTA>
__global__ void __launch_bounds__(CTA, (min_ctas<INTEG, CTA>()))
    lorenz_chain_kernel(const DevConst C, const DevKey K1, const DevKey* __restrict__ Kb,
                        const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                        lorenz_result* __restrict__ res, uint8_t* __restrict__ tags_batch,
                        uint8_t* __restrict__ block_ok) {
  constexpr int WIN = CTA >= 512 ? 32 : kWin;  // 512-thread CTAs: shorter windows keep smem < 48 KB
  __shared__ __align__(16) uint8_t stage[(CTA / 32) * 32 * (WIN + 16)];
  __shared__ double theta_tab[6 * 256];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  fill_theta<CTA>(theta_tab);
  __syncthreads();  // the only CTA-wide barrier; warps run independently afterwards

  const LaneIO io = lane_io<OP>(C, in, out, (uint64_t)blockIdx.x * CTA + threadIdx.x);
  Chain ch;
  if (io.active) key_schedule(C.batch ? Kb[io.s] : K1, C.fast != 0, (uint32_t)io.bl, C.variant, ch);
  LaneAcc acc{0, 0, true, false};
  run_chars<OP, INTEG, WIN>(C, io, ch, acc, stage + warp * 32 * (WIN + 16), theta_tab, 0,
                            warp_max_u64(io.total), lane);
  finish_lanes<OP>(C, io, acc, res, tags_batch, block_ok, lane);
}

// ------------------------------------------------------------------ the balanced kernel
// The wave kernel gives every SM sub-partition whole warps of 32 chains; when the warp count
// is not a multiple of the resident slots (C3: 2,048 warps over 592 sub-partitions = 3.46)
// the sub-partitions holding one warp more finish last and the FP64 pipe idles in the tail
// (C3: 84.9 % of peak). Here the same work is cut into equal slices instead (McNaughton's
// wrap-around rule for preemptive scheduling): unit u = 32 consecutive chains of Q 16-char
// chunks occupies chunk positions [uQ, (u+1)Q) of a line of U*Q, and resident warp slot k
// takes positions [k Cq, (k+1) Cq), Cq = ceil(U Q / S) >= Q. A unit cut by a slot boundary
// runs its FIRST chunks at the start of slot k+1, hands its 32 chain states over through
// global memory, and slot k finishes it at its end; since Q <= Cq the two pieces never
// overlap in time. Slots are numbered by start order (a ticket), later starters taking
// earlier positions, so a warp only ever waits on a piece that a warp which started before
// it runs first thing: no deadlock even when not every CTA is resident.
struct SegPlan {
  uint64_t units;  // U = ceil(lanes / 32)
  uint64_t cq;     // chunks per slot (warp group 0 when skewed)
  uint32_t q;      // chunks per unit = ceil((B + 16) / 16)
  uint32_t slots;  // S (<= U)
  uint32_t wpc;    // warps per CTA when skewed (S = CTAs x wpc), else 0
  uint32_t dq;     // skew: slots of warp index w get cq + (w / 4) dq chunks
};

// Chunk line position [x0, x1) of slot k. Unskewed: [k Cq, (k+1) Cq). Skewed: position k holds
// the slot of warp index wpc - 1 - (k mod wpc) (later starters take earlier positions), whose
// capacity grows by dq per warp group of four.
__device__ __forceinline__ void seg_slot_range(const SegPlan& P, uint64_t k, uint64_t& x0, uint64_t& x1) {
  if (P.wpc == 0) {
    x0 = k * P.cq;
    x1 = x0 + P.cq;
    return;
  }
  const uint32_t ng = P.wpc / 4, r = (uint32_t)(k % P.wpc);
  const uint64_t block = (uint64_t)P.wpc * P.cq + 2ull * P.dq * ng * (ng - 1);  // one CTA's slots
  uint64_t off = 0;
  for (uint32_t j = 0; j < r; ++j) off += P.cq + (uint64_t)((P.wpc - 1 - j) >> 2) * P.dq;
  x0 = (k / P.wpc) * block + off;
  x1 = x0 + P.cq + (uint64_t)((P.wpc - 1 - r) >> 2) * P.dq;
}
constexpr int kSegWords = 18;  // u64 words of one lane's handed-over state
#ifndef LZ_SEG_UNIFIED
#define LZ_SEG_UNIFIED 0
#endif

__device__ __forceinline__ void seg_save(uint64_t* dst, uint32_t lane, const Chain& c, const LaneAcc& a) {
  const uint64_t w[kSegWords] = {
      (uint64_t)__double_as_longlong(c.x),   (uint64_t)__double_as_longlong(c.y),
      (uint64_t)__double_as_longlong(c.z),   (uint64_t)__double_as_longlong(c.apx),
      (uint64_t)__double_as_longlong(c.apy), (uint64_t)__double_as_longlong(c.apz),
      c.m1, c.m2, c.m3,
      c.mu1 | ((uint64_t)c.mu2 << 32), c.mu3 | ((uint64_t)c.om1 << 32), c.om2 | ((uint64_t)c.om3 << 32),
      c.k1 | ((uint64_t)c.k2 << 32),   c.k3 | ((uint64_t)c.ik1 << 32),  c.ik2 | ((uint64_t)c.ik3 << 32),
      a.tlo, a.thi, (uint64_t)a.guard_ok | ((uint64_t)a.bad << 32)};
#pragma unroll
  for (int f = 0; f < kSegWords; ++f) __stcg(dst + f * 32 + lane, w[f]);
}

__device__ __forceinline__ void seg_load(const uint64_t* src, uint32_t lane, Chain& c, LaneAcc& a) {
  uint64_t w[kSegWords];
#pragma unroll
  for (int f = 0; f < kSegWords; ++f) w[f] = __ldcg(src + f * 32 + lane);
  c.x = __longlong_as_double((long long)w[0]);
  c.y = __longlong_as_double((long long)w[1]);
  c.z = __longlong_as_double((long long)w[2]);
  c.apx = __longlong_as_double((long long)w[3]);
  c.apy = __longlong_as_double((long long)w[4]);
  c.apz = __longlong_as_double((long long)w[5]);
  c.m1 = w[6]; c.m2 = w[7]; c.m3 = w[8];
  c.mu1 = (uint32_t)w[9];  c.mu2 = (uint32_t)(w[9] >> 32);
  c.mu3 = (uint32_t)w[10]; c.om1 = (uint32_t)(w[10] >> 32);
  c.om2 = (uint32_t)w[11]; c.om3 = (uint32_t)(w[11] >> 32);
  c.k1 = (uint32_t)w[12];  c.k2 = (uint32_t)(w[12] >> 32);
  c.k3 = (uint32_t)w[13];  c.ik1 = (uint32_t)(w[13] >> 32);
  c.ik2 = (uint32_t)w[14]; c.ik3 = (uint32_t)(w[14] >> 32);
  a.tlo = w[15]; a.thi = w[16];
  a.guard_ok = (uint32_t)w[17] != 0;
  a.bad = (uint32_t)(w[17] >> 32) != 0;
}

__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

#ifdef LZ_SEG_TRACE  // tuning builds only (tools/seg_trace.py): per-slot timeline
static __device__ unsigned long long g_seg_trace[4096 * 8];  // per translation unit
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SEG_TRACE(k, f, v) \
  do { if (lane == 0 && (k) < 4096) g_seg_trace[(k) * 8 + (f)] = (v); } while (0)
#else
#define SEG_TRACE(k, f, v) do {} while (0)
#endif

// Scratch (zeroed by the host before the launch): seg_ticket[0] = start-order counter,
// seg_flag[S + 1] = "the first piece of the unit cut at boundary k is done",
// seg_state[(S + 1) * kSegWords * 32] = the handed-over lane states.
template <int OP, int INTEG, int CTA>
__global__ void __launch_bounds__(CTA, 1)
    lorenz_chain_seg_kernel(const DevConst C, const DevKey K1, const DevKey* __restrict__ Kb,
                            const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                            lorenz_result* __restrict__ res, uint8_t* __restrict__ tags_batch,
                            uint8_t* __restrict__ block_ok, const SegPlan P, uint32_t* __restrict__ seg_ticket,
                            uint32_t* __restrict__ seg_flag, uint64_t* __restrict__ seg_state) {
  constexpr int WIN = CTA >= 512 ? 32 : kWin;  // 512-thread CTAs: shorter windows keep smem < 48 KB
  __shared__ __align__(16) uint8_t stage[(CTA / 32) * 32 * (WIN + 16)];
  __shared__ double theta_tab[6 * 256];
  __shared__ uint32_t s_ticket;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  fill_theta<CTA>(theta_tab);
  if (threadIdx.x == 0) s_ticket = atomicAdd(seg_ticket, 1u);
  __syncthreads();
  const uint64_t t = (uint64_t)s_ticket * (CTA / 32) + warp;  // start order
  if (t >= P.slots) return;
  const uint64_t k = P.slots - 1 - t;  // later starters take earlier positions
  const uint64_t Q = P.q, UQ = P.units * Q;
  uint64_t X0, X1;
  seg_slot_range(P, k, X0, X1);
  if (X0 >= UQ) return;
  if (X1 > UQ) X1 = UQ;
  uint8_t* wst = stage + warp * 32 * (WIN + 16);
  uint64_t u = X0 / Q;
#ifdef LZ_SEG_TRACE
  {
    uint32_t smid, wid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    asm volatile("mov.u32 %0, %warpid;" : "=r"(wid));
    SEG_TRACE(k, 0, gtimer());
    SEG_TRACE(k, 6, ((unsigned long long)smid << 32) | wid);
    SEG_TRACE(k, 7, t);
  }
#endif

#if LZ_SEG_UNIFIED
  // One loop over the slot's pieces with a single inlined copy of the character loop (so ptxas can
  // keep the integrator's constants in uniform registers): piece 0 may be the FIRST chunks [0, a) of
  // the unit cut at X0 (hands its state to slot k-1), then whole units, then possibly the LAST chunks
  // [a', Q) of the unit cut at X1 (takes its state from slot k+1).
  const uint64_t u_end = (X1 + Q - 1) / Q;  // one past the last unit the slot touches
  for (; u < u_end; ++u) {
    const bool first_piece = u * Q < X0;                       // starts before X0: chunks [0, (u+1)Q - X0)
    const bool last_piece = !first_piece && (u + 1) * Q > X1;  // ends after X1: chunks [(u+1)Q - X1, Q)
    const uint64_t c0 = last_piece ? (u + 1) * Q - X1 : 0;
    const uint64_t c1 = first_piece ? (u + 1) * Q - X0 : Q;
    const LaneIO io = lane_io<OP>(C, in, out, u * 32 + lane);
    Chain ch;
    LaneAcc acc{0, 0, true, false};
    if (last_piece) {
      SEG_TRACE(k, 2, gtimer());
      if (lane == 0)
        while (ld_acquire_u32(seg_flag + k + 1) == 0) __nanosleep(256);
      __syncwarp();
      SEG_TRACE(k, 3, gtimer());
      (void)ld_acquire_u32(seg_flag + k + 1);
      seg_load(seg_state + (k + 1) * (kSegWords * 32), lane, ch, acc);
    } else if (io.active) {
      key_schedule(C.batch ? Kb[io.s] : K1, C.fast != 0, (uint32_t)io.bl, C.variant, ch);
    }
    run_chars<OP, INTEG, WIN, true>(C, io, ch, acc, wst, theta_tab, 16 * c0, 16 * c1, lane);
    if (first_piece) {
      seg_save(seg_state + k * (kSegWords * 32), lane, ch, acc);
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release_u32(seg_flag + k, 1u);
      SEG_TRACE(k, 1, gtimer());
    } else {
      finish_lanes<OP>(C, io, acc, res, tags_batch, block_ok, lane);
    }
  }
#else
  if (X0 % Q) {  // first piece: chunks [0, a) of unit u, which slot k-1 finishes
    const uint64_t a = (u + 1) * Q - X0;
    const LaneIO io = lane_io<OP>(C, in, out, u * 32 + lane);
    Chain ch;
    if (io.active) key_schedule(C.batch ? Kb[io.s] : K1, C.fast != 0, (uint32_t)io.bl, C.variant, ch);
    LaneAcc acc{0, 0, true, false};
    run_chars<OP, INTEG, WIN, true>(C, io, ch, acc, wst, theta_tab, 0, 16 * a, lane);
    seg_save(seg_state + k * (kSegWords * 32), lane, ch, acc);
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release_u32(seg_flag + k, 1u);
    SEG_TRACE(k, 1, gtimer());
    ++u;
  }
  for (; (u + 1) * Q <= X1; ++u) {  // whole units
    const LaneIO io = lane_io<OP>(C, in, out, u * 32 + lane);
    Chain ch;
    if (io.active) key_schedule(C.batch ? Kb[io.s] : K1, C.fast != 0, (uint32_t)io.bl, C.variant, ch);
    LaneAcc acc{0, 0, true, false};
    run_chars<OP, INTEG, WIN, true>(C, io, ch, acc, wst, theta_tab, 0, 16 * Q, lane);
    finish_lanes<OP>(C, io, acc, res, tags_batch, block_ok, lane);
  }
  if (u * Q < X1) {  // last piece: chunks [a, Q) of unit u, whose first a chunks open slot k+1
    const uint64_t a = (u + 1) * Q - X1;
    const LaneIO io = lane_io<OP>(C, in, out, u * 32 + lane);
    SEG_TRACE(k, 2, gtimer());
    if (lane == 0)
      while (ld_acquire_u32(seg_flag + k + 1) == 0) __nanosleep(256);
    __syncwarp();
    SEG_TRACE(k, 3, gtimer());
    (void)ld_acquire_u32(seg_flag + k + 1);
    Chain ch;
    LaneAcc acc;
    seg_load(seg_state + (k + 1) * (kSegWords * 32), lane, ch, acc);
    run_chars<OP, INTEG, WIN, true>(C, io, ch, acc, wst, theta_tab, 16 * a, 16 * Q, lane);
    finish_lanes<OP>(C, io, acc, res, tags_batch, block_ok, lane);
  }
#endif
  SEG_TRACE(k, 4, gtimer());
}

// Zero the plaintext slice if the launch found an integrity failure (async decrypt
// without per-block verdicts: unauthenticated plaintext is never released).
static __global__ void zero_if_failed_kernel(const lorenz_result* __restrict__ res, uint8_t* __restrict__ pt,
                                      uint64_t nbytes) {
  if (!(res->status & ST_INTEGRITY)) return;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nbytes;
       i += (uint64_t)gridDim.x * blockDim.x)
    pt[i] = 0;
}

static __global__ void result_init_kernel(lorenz_result* res) {
  if (threadIdx.x == 0) {
    *reinterpret_cast<unsigned long long*>(res->tag_xor) = 0;
    *reinterpret_cast<unsigned long long*>(res->tag_xor + 8) = 0;
    res->first_bad = ~0ULL;
    res->status = 0;
    res->reserved = 0;
  }
}

}  // namespace lz
