/* lorenz_ref.c — CPU ORACLE (test infrastructure only; see lorenz_ref.h).
 *
 * Plain definition of the per-block chaotic operation mode of arXiv 1201.3114,
 * written from PAPER.md and the readings listed in DESIGN.md §3. Every
 * function cites the passage it follows. Nothing here is blocked, fused or
 * reordered: one character at a time, one RK4 step at a time, scalar doubles.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread
 * (x86-64 SSE2 doubles; -ffp-contract=off forbids FMA contraction, which would
 * change the rounding of the canonical operation order — SURVEY.md F6).
 */
#include "lorenz_ref.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ======================================================================== */
/* SHA-256, FIPS 180-4 (the paper's "hash function such as MD5 or SHA", P:235;
 * SHA-256 per S:159/S:181, reading Q11).                                    */
/* ======================================================================== */
static const uint32_t SHA_K[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u,
    0xab1c5ed5u, 0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu,
    0x9bdc06a7u, 0xc19bf174u, 0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu,
    0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau, 0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u,
    0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u, 0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu,
    0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u, 0xa2bfe8a1u, 0xa81a664bu,
    0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u, 0x19a4c116u,
    0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
    0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u,
    0xc67178f2u};

static uint32_t rotr32(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

static void sha256_block(uint32_t h[8], const uint8_t blk[64]) {
  uint32_t w[64];
  for (int t = 0; t < 16; ++t)
    w[t] = ((uint32_t)blk[4 * t] << 24) | ((uint32_t)blk[4 * t + 1] << 16) |
           ((uint32_t)blk[4 * t + 2] << 8) | (uint32_t)blk[4 * t + 3];
  for (int t = 16; t < 64; ++t) {
    uint32_t s0 = rotr32(w[t - 15], 7) ^ rotr32(w[t - 15], 18) ^ (w[t - 15] >> 3);
    uint32_t s1 = rotr32(w[t - 2], 17) ^ rotr32(w[t - 2], 19) ^ (w[t - 2] >> 10);
    w[t] = w[t - 16] + s0 + w[t - 7] + s1;
  }
  uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
  for (int t = 0; t < 64; ++t) {
    uint32_t S1 = rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25);
    uint32_t ch = (e & f) ^ (~e & g);
    uint32_t T1 = hh + S1 + ch + SHA_K[t] + w[t];
    uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);
    uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
    uint32_t T2 = S0 + mj;
    hh = g; g = f; f = e; e = d + T1; d = c; c = b; b = a; a = T1 + T2;
  }
  h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

void lorenz_ref_sha256(const uint8_t* msg, size_t len, uint8_t out[32]) {
  uint32_t h[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                   0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
  size_t full = len / 64;
  for (size_t i = 0; i < full; ++i) sha256_block(h, msg + 64 * i);
  uint8_t tail[128];
  size_t rem = len - 64 * full;
  memset(tail, 0, sizeof tail);
  if (rem) memcpy(tail, msg + 64 * full, rem);
  tail[rem] = 0x80;
  size_t tl = (rem + 1 + 8 <= 64) ? 64 : 128;
  uint64_t bits = (uint64_t)len * 8u;
  for (int i = 0; i < 8; ++i) tail[tl - 1 - i] = (uint8_t)(bits >> (8 * i));
  sha256_block(h, tail);
  if (tl == 128) sha256_block(h, tail + 64);
  for (int i = 0; i < 8; ++i) {
    out[4 * i] = (uint8_t)(h[i] >> 24);
    out[4 * i + 1] = (uint8_t)(h[i] >> 16);
    out[4 * i + 2] = (uint8_t)(h[i] >> 8);
    out[4 * i + 3] = (uint8_t)h[i];
  }
}

static uint64_t be64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v = (v << 8) | p[i];
  return v;
}
static void put_be64(uint8_t* p, uint64_t v) {
  for (int i = 7; i >= 0; --i) { p[i] = (uint8_t)v; v >>= 8; }
}

/* ======================================================================== */
/* Key schedule (§3.1)                                            */
/* ======================================================================== */

/* Eqs.2-4: pack pi_1..pi_n (1-based) into a1,a2,a3; L=floor(n/3). */
int lorenz_ref_pack(const uint8_t* pw, size_t n, uint64_t a[3]) {
  if (n < 3 || n > 23) return LREF_E_PASSWORD; /* Q17: 3 <= n_pi <= 23 */
  size_t L = n / 3;
  const uint8_t* pi = pw - 1; /* pi[i] == pi_i, 1-based as in the paper */
  uint64_t a1 = 0, a2 = 0, a3 = 0;
  /* Eq.2 */
  if (n % 3 == 0) {
    for (size_t i = 1; i <= L; ++i) a1 += (uint64_t)pi[i] << (8 * (i - 1));
  } else {
    for (size_t i = 1; i <= L; ++i) a1 += (uint64_t)pi[i] << (8 * i);
    a1 += pi[3 * L + 1];
  }
  /* Eq.3 */
  if (n % 3 != 2) {
    for (size_t i = L + 1; i <= 2 * L; ++i) a2 += (uint64_t)pi[i] << (8 * (i - L - 1));
  } else {
    for (size_t i = L + 1; i <= 2 * L; ++i) a2 += (uint64_t)pi[i] << (8 * (i - L));
    a2 += pi[3 * L + 2];
  }
  /* Eq.4 */
  for (size_t i = 2 * L + 1; i <= 3 * L; ++i) a3 += (uint64_t)pi[i] << (8 * (i - 2 * L - 1));
  a[0] = a1; a[1] = a2; a[2] = a3;
  return LREF_OK;
}

/* g(x) = x / 10^ceil(log10 2^{8(L+1)}) (log base 10 per Q6). */
int lorenz_ref_norm_exponent(int L) {
  return (int)ceil((double)(8 * (L + 1)) * log10(2.0));
}

static double pow10_exact(int e) { /* 10^e, exact in binary64 for e <= 22 */
  double v = 1.0;
  for (int i = 0; i < e; ++i) v = v * 10.0;
  return v;
}

void lorenz_ref_normalize(const uint64_t a[3], int L, double ap[3]) {
  double div = pow10_exact(lorenz_ref_norm_exponent(L));
  for (int i = 0; i < 3; ++i) ap[i] = (double)a[i] / div;
}

/* lambda: the paper gives only the ranges; selection rule of S:132,
 * reading Q10: h_i = BE64(SHA-256(0x4C ‖ BE64 a1 ‖ BE64 a2 ‖ BE64 a3 ‖ u8 i)),
 * lambda_i = lo_i + (double(h_i) * 2^-64) * (hi_i - lo_i), i = 1..3.        */
void lorenz_ref_lambda(const uint64_t a[3], double lam[3]) {
  const double lo[3] = {-15.67, -11.28, 0.090};
  const double hi[3] = {16.01, 16.01, 62.000};
  for (int i = 1; i <= 3; ++i) {
    uint8_t msg[26], dig[32];
    msg[0] = 0x4C;
    put_be64(msg + 1, a[0]);
    put_be64(msg + 9, a[1]);
    put_be64(msg + 17, a[2]);
    msg[25] = (uint8_t)i;
    lorenz_ref_sha256(msg, sizeof msg, dig);
    double t = (double)be64(dig);
    t = t * ldexp(1.0, -64);
    double w = hi[i - 1] - lo[i - 1];
    lam[i - 1] = lo[i - 1] + t * w;
  }
}

/* mu: mu1=(a1+a2+a3) mod 3, mu2=(a1*a2+a3) mod 3, mu3=(a1+a2*a3) mod 3,
 * over the integers (reduced mod 3 first so nothing overflows).            */
void lorenz_ref_mu(const uint64_t a[3], int mu[3]) {
  uint64_t r1 = a[0] % 3, r2 = a[1] % 3, r3 = a[2] % 3;
  mu[0] = (int)((r1 + r2 + r3) % 3);
  mu[1] = (int)((r1 * r2 + r3) % 3);
  mu[2] = (int)((r1 + r2 * r3) % 3);
}

/* k (P:230, 2 < k_i <= floor((52-14)/8) = 4) and k3 of Step 3 (P:322,
 * 0 < k3 < nu-2) from H = SHA-256(pi): k_i = 3 + H[i-1] mod 2,
 * k3chain = 1 + H[3] mod 6 (reading Q12).
 * Omega_i = hash(i a) mod k_i (Eq.7): BE64 prefix of
 * SHA-256(BE64(i a1) ‖ BE64(i a2) ‖ BE64(i a3)), products mod 2^64 (Q11).   */
static void k_omega_hashes(const uint8_t* pw, size_t n, const uint64_t a[3], int k[3],
                           int* k3chain, int omega[3], uint64_t hom[3]) {
  uint8_t H[32];
  lorenz_ref_sha256(pw, n, H);
  for (int i = 0; i < 3; ++i) k[i] = 3 + (H[i] % 2);
  *k3chain = 1 + (H[3] % 6);
  for (int i = 1; i <= 3; ++i) {
    uint8_t msg[24], dig[32];
    for (int j = 0; j < 3; ++j) put_be64(msg + 8 * j, (uint64_t)i * a[j]);
    lorenz_ref_sha256(msg, sizeof msg, dig);
    hom[i - 1] = be64(dig);
    omega[i - 1] = (int)(hom[i - 1] % (uint64_t)k[i - 1]);
  }
}

void lorenz_ref_k_omega(const uint8_t* pw, size_t n, const uint64_t a[3], int k[3],
                        int* k3chain, int omega[3]) {
  uint64_t hom[3];
  k_omega_hashes(pw, n, a, k, k3chain, omega, hom);
}

/* Passwords longer than 23 bytes are replaced by SHA-256(pi)[0:18]; shorter
 * than 3 is an error (reading Q17).                          */
int lorenz_ref_normalize_password(const uint8_t* pw, size_t n, uint8_t out[23], size_t* n_out) {
  if (n < 3) return LREF_E_PASSWORD;
  if (n > 23) {
    uint8_t H[32];
    lorenz_ref_sha256(pw, n, H);
    memcpy(out, H, 18);
    *n_out = 18;
  } else {
    memcpy(out, pw, n);
    *n_out = n;
  }
  return LREF_OK;
}

/* Per-block password of the parallel version: "for each process a particular
 * initial condition is selected"; pi_b = SHA-256(pi ‖ BE32 b)[0:18]
 * (reading Q16/Q17: the raw password is hashed).                    */
void lorenz_ref_subpassword(const uint8_t* pw, size_t n, uint32_t b, uint8_t out[18]) {
  uint8_t* msg = (uint8_t*)malloc(n + 4);
  memcpy(msg, pw, n);
  msg[n] = (uint8_t)(b >> 24);
  msg[n + 1] = (uint8_t)(b >> 16);
  msg[n + 2] = (uint8_t)(b >> 8);
  msg[n + 3] = (uint8_t)b;
  uint8_t H[32];
  lorenz_ref_sha256(msg, n + 4, H);
  free(msg);
  memcpy(out, H, 18);
}

/* Composite §3.1: a, a', lambda, r0 = a' + lambda (Eq.5), mu, k, Omega,
 * alpha_i = r0[mu_i] (Eq.6 with n = 0).                                     */
int lorenz_ref_keymaterial(const uint8_t* pw_norm, size_t n, lref_km* km) {
  memset(km, 0, sizeof *km);
  int st = lorenz_ref_pack(pw_norm, n, km->a);
  if (st) return st;
  km->L = (int)(n / 3);
  km->d = lorenz_ref_norm_exponent(km->L);
  lorenz_ref_normalize(km->a, km->L, km->ap);
  lorenz_ref_lambda(km->a, km->lam);
  for (int i = 0; i < 3; ++i) km->r0[i] = km->ap[i] + km->lam[i];
  lorenz_ref_mu(km->a, km->mu);
  k_omega_hashes(pw_norm, n, km->a, km->k, &km->k3chain, km->omega, km->hom);
  for (int i = 0; i < 3; ++i) km->alpha[i] = km->r0[km->mu[i]];
  return LREF_OK;
}

/* NEXT-4 variant "distinct k": k2 = 7 - k1, so k1 != k2 (both stay in
 * the paper's range 2 < k <= 4) and Omega0_2 = hash(2a) mod the new k2.       */
void lorenz_ref_apply_variant(lref_km* km, uint32_t variant) {
  if (variant & LREF_V_DISTINCT_K) {
    km->k[1] = 7 - km->k[0];
    km->omega[1] = (int)(km->hom[1] % (uint64_t)km->k[1]);
  }
}

/* ======================================================================== */
/* Quantiser and encode/decode (Eqs.8-10)                        */
/* ======================================================================== */

/* R_nu(alpha, Omega) = (floor(alpha 10^nu) AND 255*2^{8 Omega}) / 2^{8 Omega},
 * nu = floor(log10 2^{52-6}) = 13. |alpha| (Q8); floor of the rounded
 * product (Q9); the integer fits 53 bits (Q7).                              */
int lorenz_ref_R(double alpha, int omega) {
  double prod = fabs(alpha) * 1e13;
  uint64_t m = (uint64_t)prod; /* truncation == floor for prod >= 0 */
  uint64_t mask = (uint64_t)255 << (8 * omega);
  return (int)((m & mask) >> (8 * omega));
}

/* Eq.9: y = [x + sum R] mod 2^8 ;  Eq.10: x = [y - sum R] mod 2^8 */
int lorenz_ref_encode(int p, int ksum) { return ((p + ksum) % 256 + 256) % 256; }
int lorenz_ref_decode(int c, int ksum) { return ((c - ksum) % 256 + 256) % 256; }

/* ======================================================================== */
/* Dynamics (§3.1 Eq.1; RK4 per the north star, reading Q1-Q3)    */
/* ======================================================================== */
static const double SIGMA = 10.0, RHO = 28.0;
#define BETA (8.0 / 3.0)

double lorenz_ref_dt(uint32_t dt_code) {
  switch (dt_code) {
    case 0: return 0.01;
    case 1: return 0.005;
    case 2: return 0.02;
    case 3: return 0.027;
    default: return NAN;
  }
}

/* Lorenz right-hand side, standard form (Q2), term order of S:40:
 * fx = sigma*(y-x); fy = (rho*x - y) - x*z; fz = x*y - beta*z.             */
void lorenz_ref_rhs(const double s[3], double f[3]) {
  double x = s[0], y = s[1], z = s[2];
  double beta = BETA;
  f[0] = SIGMA * (y - x);
  f[1] = (RHO * x - y) - x * z;
  f[2] = x * y - beta * z;
}

/* Classical RK4, canonical order (Q3): k1=f(s), a=s+h2*k1, k2=f(a),
 * b=s+h2*k2, k3=f(b), c=s+h*k3, k4=f(c),
 * s' = s + h6*(((((k1+k2)+k2)+k3)+k3)+k4), h2=h*0.5, h6=h/6.0.             */
void lorenz_ref_rk4_step(double s[3], double h) {
  double h2 = h * 0.5, h6 = h / 6.0;
  double k1[3], k2[3], k3[3], k4[3], t[3];
  lorenz_ref_rhs(s, k1);
  for (int c = 0; c < 3; ++c) t[c] = s[c] + h2 * k1[c];
  lorenz_ref_rhs(t, k2);
  for (int c = 0; c < 3; ++c) t[c] = s[c] + h2 * k2[c];
  lorenz_ref_rhs(t, k3);
  for (int c = 0; c < 3; ++c) t[c] = s[c] + h * k3[c];
  lorenz_ref_rhs(t, k4);
  for (int c = 0; c < 3; ++c) {
    double sum = k1[c] + k2[c];
    sum = sum + k2[c];
    sum = sum + k3[c];
    sum = sum + k3[c];
    sum = sum + k4[c];
    s[c] = s[c] + h6 * sum;
  }
}

/* Forward Euler, the paper's own discretisation in the standard
 * (non-garbled) form of S:40: s' = s + f(s)*h.                              */
void lorenz_ref_euler_step(double s[3], double h) {
  double f[3];
  lorenz_ref_rhs(s, f);
  for (int c = 0; c < 3; ++c) s[c] = s[c] + f[c] * h;
}

/* NEXT-3: the same classical RK4 with fused multiply-adds at fixed sites.
 * fma() is correctly rounded (C99 7.12.13.1), so this is as deterministic as the
 * unfused form; it is a different cipher definition (fewer roundings, 45 operations).
 * RHS: fx = sigma*(y-x); fy = fma(-x, z, fma(rho, x, -y)); fz = fma(x, y, -(beta*z)).  */
static void rhs_fma(const double s[3], double f[3]) {
  double x = s[0], y = s[1], z = s[2];
  double beta = BETA;
  f[0] = SIGMA * (y - x);
  f[1] = fma(-x, z, fma(RHO, x, -y));
  f[2] = fma(x, y, -(beta * z));
}

/* stages a = fma(h2, k1, s), b = fma(h2, k2, s), c = fma(h, k3, s);
 * s' = fma(h6, (fma(2, k3, fma(2, k2, k1)) + k4), s).                                    */
void lorenz_ref_rk4fma_step(double s[3], double h) {
  double h2 = h * 0.5, h6 = h / 6.0;
  double k1[3], k2[3], k3[3], k4[3], t[3];
  rhs_fma(s, k1);
  for (int c = 0; c < 3; ++c) t[c] = fma(h2, k1[c], s[c]);
  rhs_fma(t, k2);
  for (int c = 0; c < 3; ++c) t[c] = fma(h2, k2[c], s[c]);
  rhs_fma(t, k3);
  for (int c = 0; c < 3; ++c) t[c] = fma(h, k3[c], s[c]);
  rhs_fma(t, k4);
  for (int c = 0; c < 3; ++c) {
    double sum = fma(2.0, k2[c], k1[c]);
    sum = fma(2.0, k3[c], sum);
    sum = sum + k4[c];
    s[c] = fma(h6, sum, s[c]);
  }
}

void lorenz_ref_iterate(double s[3], uint32_t dt_code, uint32_t integrator, uint64_t n) {
  double h = lorenz_ref_dt(dt_code);
  for (uint64_t i = 0; i < n; ++i) {
    if (integrator == LREF_EULER) lorenz_ref_euler_step(s, h);
    else if (integrator == LREF_RK4_FMA) lorenz_ref_rk4fma_step(s, h);
    else lorenz_ref_rk4_step(s, h);
  }
}

/* ======================================================================== */
/* The chain, Steps 1-3 (§3.2)                                     */
/* ======================================================================== */
static const uint8_t SENT[16] = {'L', 'O', 'R', 'E', 'N', 'Z', 'C', 'H',
                                 'A', 'O', 'S', '-', 'M', 'A', 'C', '1'}; /* S:248, Q15 */

typedef struct {
  double r[3];
  int mu[3], omega[3], k[3];
  double alpha[3], ap[3];
} chain_t;

static void chain_init(chain_t* ch, const lref_km* km) {
  for (int i = 0; i < 3; ++i) {
    ch->r[i] = km->r0[i];
    ch->mu[i] = km->mu[i];
    ch->omega[i] = km->omega[i];
    ch->alpha[i] = km->alpha[i]; /* Eq.6 with n = 0 (Q14) */
    ch->ap[i] = km->ap[i];
  }
  ch->k[0] = km->k[0];
  ch->k[1] = km->k[1];
  ch->k[2] = km->k3chain; /* Step 3 uses k3 in (0, nu-2) */
}

/* Step 1 keystream: sum_{i=1,2} R_nu(alpha_i, Omega_i) (Eq.9). */
static int chain_keysum(const chain_t* ch) {
  return lorenz_ref_R(ch->alpha[0], ch->omega[0]) + lorenz_ref_R(ch->alpha[1], ch->omega[1]);
}

static int guard_ok(const double r[3]) { /* reading Q18 */
  if (!isfinite(r[0]) || !isfinite(r[1]) || !isfinite(r[2])) return 0;
  if (fabs(r[0]) > 100.0 || fabs(r[1]) > 100.0) return 0;
  if (r[2] < -50.0 || r[2] > 150.0) return 0;
  return 1;
}

/* Steps 2-3 after the plaintext byte p of this character is known. */
/* Step 2: Theta = P_i / 10^{3+Omega_3}, one correctly rounded division (Q19). */
double lorenz_ref_theta(int p, int omega3) { return (double)p / pow10_exact(3 + omega3); }

static int chain_advance(chain_t* ch, int p, const lref_params* prm) {
  /* Step 2: Theta added to the coordinate selected by mu_3. */
  double theta = lorenz_ref_theta(p, ch->omega[2]);
  ch->r[ch->mu[2]] = ch->r[ch->mu[2]] + theta;
  /* the trajectory: n_it iterations of the map */
  lorenz_ref_iterate(ch->r, prm->dt_code, prm->integrator, prm->n_it);
  if (!guard_ok(ch->r)) return LREF_E_DIVERGENCE;
  int R[3];
  if ((prm->variant & LREF_V_ORDER_MASK) == LREF_V_LITERAL) {
    /* NEXT-4 literal textual order of P:320-322: mu_i' = [mu_i + R(alpha_i, Omega_i)] mod 3
     * with the alpha of the previous character; then "alpha given by Eq.6" from the new mu;
     * then Omega_i = [Omega_i' + R(alpha_{[(i+2) mod 3]+1}, Omega_i')] mod k_i, where the
     * printed permutation is the identity for 1-based i.                        */
    for (int i = 0; i < 3; ++i) R[i] = lorenz_ref_R(ch->alpha[i], ch->omega[i]);
    for (int i = 0; i < 3; ++i) ch->mu[i] = (ch->mu[i] + R[i]) % 3;
    for (int i = 0; i < 3; ++i) ch->alpha[i] = ch->r[ch->mu[i]];
    for (int i = 0; i < 3; ++i)
      ch->omega[i] = (ch->omega[i] + lorenz_ref_R(ch->alpha[i], ch->omega[i])) % ch->k[i];
  } else {
    /* Step 3, order of reading Q13: alpha_i = r[mu_i] (Eq.6 with the
     * old mu); R_i = R(alpha_i, Omega_i) with the old Omega; mu_i = (mu_i + R_i)
     * mod 3; Omega_i = (Omega_i + R_i) mod k_i.                                */
    for (int i = 0; i < 3; ++i) ch->alpha[i] = ch->r[ch->mu[i]];
    for (int i = 0; i < 3; ++i) R[i] = lorenz_ref_R(ch->alpha[i], ch->omega[i]);
    for (int i = 0; i < 3; ++i) ch->mu[i] = (ch->mu[i] + R[i]) % 3;
    if ((prm->variant & LREF_V_ORDER_MASK) == LREF_V_CYCLIC) {
      /* NEXT-4 cyclic reading of the index [(i+2) mod 3]+1: Omega_i takes its byte from
       * alpha_{i+1} (alpha_1 for i = 3) instead of alpha_i.                         */
      for (int i = 0; i < 3; ++i)
        ch->omega[i] = (ch->omega[i] + lorenz_ref_R(ch->alpha[(i + 1) % 3], ch->omega[i])) % ch->k[i];
    } else {
      for (int i = 0; i < 3; ++i) ch->omega[i] = (ch->omega[i] + R[i]) % ch->k[i];
    }
  }
  /* r_n = r_n + a' */
  for (int i = 0; i < 3; ++i) ch->r[i] = ch->r[i] + ch->ap[i];
  return LREF_OK;
}

static void fill_defaults(const lref_params* in, lref_params* out) {
  *out = *in;
  if (out->n_it == 0) out->n_it = (out->mode == LREF_FAST) ? 100u : 3000u;
  if (out->block_size == 0) out->block_size = 1024u;
}

/* encrypt_stream: P ‖ SENT, per character Step 1 then Steps 2-3
 * with the plaintext byte; the last character is not advanced (Q20).       */
int lorenz_ref_encrypt_stream(const lref_km* km, const lref_params* prm_in, const uint8_t* p,
                              size_t len, uint8_t* c, double* trace) {
  lref_params prm;
  fill_defaults(prm_in, &prm);
  chain_t ch;
  chain_init(&ch, km);
  size_t total = len + 16;
  for (size_t j = 0; j < total; ++j) {
    int pj = (j < len) ? p[j] : SENT[j - len];
    c[j] = (uint8_t)lorenz_ref_encode(pj, chain_keysum(&ch));
    if (j + 1 == total) break;
    int st = chain_advance(&ch, pj, &prm);
    if (st) return st;
    if (trace) memcpy(trace + 3 * j, ch.r, sizeof ch.r);
  }
  return LREF_OK;
}

/* decrypt_stream: Step 1 inverted; the chain advances with the
 * RECOVERED plaintext byte; the trailing 16 bytes must equal SENT.  */
int lorenz_ref_decrypt_stream(const lref_km* km, const lref_params* prm_in, const uint8_t* c,
                              size_t clen, uint8_t* p, int* ok, double* trace) {
  if (clen < 16) return LREF_E_LENGTH;
  lref_params prm;
  fill_defaults(prm_in, &prm);
  chain_t ch;
  chain_init(&ch, km);
  size_t len = clen - 16;
  int good = 1;
  for (size_t j = 0; j < clen; ++j) {
    int pj = lorenz_ref_decode(c[j], chain_keysum(&ch));
    if (j < len) p[j] = (uint8_t)pj;
    else if (pj != SENT[j - len]) good = 0;
    if (j + 1 == clen) break;
    int st = chain_advance(&ch, pj, &prm);
    if (st) return st;
    if (trace) memcpy(trace + 3 * j, ch.r, sizeof ch.r);
  }
  *ok = good;
  return LREF_OK;
}

/* ======================================================================== */
/* Message framing (§5; reading Q16, Q21)       */
/* ======================================================================== */
uint64_t lorenz_ref_num_blocks(const lref_params* prm_in, uint64_t n) {
  lref_params prm;
  fill_defaults(prm_in, &prm);
  if (prm.mode == LREF_STRONG) return 1;
  uint64_t B = prm.block_size;
  uint64_t nb = (n + B - 1) / B;
  return nb == 0 ? 1 : nb;
}

uint64_t lorenz_ref_ct_len(const lref_params* prm, uint64_t n) {
  return n + 16 * lorenz_ref_num_blocks(prm, n);
}

int lorenz_ref_pt_len(const lref_params* prm_in, uint64_t ct_len, uint64_t* n_out) {
  lref_params prm;
  fill_defaults(prm_in, &prm);
  if (ct_len < 16) return LREF_E_LENGTH;
  if (prm.mode == LREF_STRONG) { *n_out = ct_len - 16; return LREF_OK; }
  uint64_t per = (uint64_t)prm.block_size + 16;
  uint64_t nb = (ct_len + per - 1) / per;
  if (ct_len < 16 * nb) return LREF_E_LENGTH;
  uint64_t n = ct_len - 16 * nb;
  if (lorenz_ref_num_blocks(&prm, n) != nb) return LREF_E_LENGTH;
  *n_out = n;
  return LREF_OK;
}

static int check_params(const lref_params* prm) {
  if (prm->mode > 1 || prm->integrator > 2 || prm->dt_code > 3) return LREF_E_ARG;
  if ((prm->variant & LREF_V_ORDER_MASK) == 3 || prm->variant > 7) return LREF_E_ARG;
  if (prm->mode == LREF_FAST && (prm->block_size < 1024 || prm->block_size % 16)) return LREF_E_ARG;
  return LREF_OK;
}

/* key material of global block b */
static int block_km(const uint8_t* pw, size_t pw_len, const lref_params* prm, uint64_t b,
                    lref_km* km) {
  int st;
  if (prm->mode == LREF_FAST) {
    uint8_t sub[18];
    lorenz_ref_subpassword(pw, pw_len, (uint32_t)b, sub);
    st = lorenz_ref_keymaterial(sub, 18, km);
  } else {
    uint8_t norm[23];
    size_t nn;
    st = lorenz_ref_normalize_password(pw, pw_len, norm, &nn);
    if (st) return st;
    st = lorenz_ref_keymaterial(norm, nn, km);
  }
  if (!st) lorenz_ref_apply_variant(km, prm->variant);
  return st;
}

typedef struct {
  const uint8_t* pw;
  size_t pw_len;
  lref_params prm;
  uint64_t n, b_lo, b_hi;
  const uint8_t* in;
  uint8_t* out;
  int decrypt;
  uint8_t* ok; /* per block, indexed b - b_base */
  uint64_t b_base;
  int status;
} job_t;

static void* run_job(void* arg) {
  job_t* jb = (job_t*)arg;
  uint64_t B = jb->prm.mode == LREF_FAST ? jb->prm.block_size : jb->n;
  jb->status = LREF_OK;
  for (uint64_t b = jb->b_lo; b < jb->b_hi; ++b) {
    uint64_t start = b * B;
    uint64_t len = jb->n - start < B ? jb->n - start : B;
    if (jb->prm.mode == LREF_STRONG) { start = 0; len = jb->n; }
    lref_km km;
    int st = block_km(jb->pw, jb->pw_len, &jb->prm, b, &km);
    if (!st) {
      if (!jb->decrypt) {
        st = lorenz_ref_encrypt_stream(&km, &jb->prm, jb->in + start, len,
                                       jb->out + start + 16 * b, NULL);
      } else {
        int good = 0;
        st = lorenz_ref_decrypt_stream(&km, &jb->prm, jb->in + start + 16 * b, len + 16,
                                       jb->out + start, &good, NULL);
        jb->ok[b - jb->b_base] = (uint8_t)good;
      }
    }
    if (st && !jb->status) jb->status = st;
  }
  return NULL;
}

static int run_blocks(const uint8_t* pw, size_t pw_len, const lref_params* prm, uint64_t n,
                      uint64_t b0, uint64_t b1, const uint8_t* in, uint8_t* out, int decrypt,
                      uint8_t* ok, int threads) {
  if (threads <= 0) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  uint64_t nbk = b1 - b0;
  if ((uint64_t)threads > nbk) threads = (int)nbk;
  if (threads < 1) threads = 1;
  job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) { /* static contiguous partition */
    job_t* jb = &jobs[t];
    jb->pw = pw; jb->pw_len = pw_len; jb->prm = *prm; jb->n = n;
    jb->b_lo = b0 + nbk * (uint64_t)t / (uint64_t)threads;
    jb->b_hi = b0 + nbk * (uint64_t)(t + 1) / (uint64_t)threads;
    jb->in = in; jb->out = out; jb->decrypt = decrypt; jb->ok = ok; jb->b_base = b0;
  }
  for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, run_job, &jobs[t]);
  run_job(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
  int st = LREF_OK;
  for (int t = 0; t < threads; ++t) if (jobs[t].status && !st) st = jobs[t].status;
  free(jobs);
  free(tid);
  return st;
}

int lorenz_ref_encrypt(const uint8_t* pw, size_t pw_len, const lref_params* prm_in, uint64_t n,
                       uint64_t b0, uint64_t b1, const uint8_t* pt, uint8_t* ct,
                       uint8_t tag_xor[16], int threads) {
  lref_params prm;
  fill_defaults(prm_in, &prm);
  if (check_params(&prm)) return LREF_E_ARG;
  if (pw_len < 3) return LREF_E_PASSWORD;
  uint64_t nb = lorenz_ref_num_blocks(&prm, n);
  if (b0 > b1 || b1 > nb) return LREF_E_ARG;
  memset(tag_xor, 0, 16);
  if (b0 == b1) return LREF_OK;
  int st = run_blocks(pw, pw_len, &prm, n, b0, b1, pt, ct, 0, NULL, threads);
  if (st) return st;
  uint64_t B = prm.mode == LREF_FAST ? prm.block_size : n;
  for (uint64_t b = b0; b < b1; ++b) { /* T = XOR of block tags (Q15) */
    uint64_t end = (b + 1) * B < n ? (b + 1) * B : n;
    if (prm.mode == LREF_STRONG) end = n;
    const uint8_t* tag = ct + end + 16 * b;
    for (int i = 0; i < 16; ++i) tag_xor[i] ^= tag[i];
  }
  return LREF_OK;
}

/* ======================================================================== */
/* NEXT-4 analysis: Fig.1 digit frequencies (§3.1)                 */
/* ======================================================================== */
/* "frequency distribution of the integer part as well as the decimal part of the Lorenz's
 * attractor": (a) integer part, (b) 1st-2nd, (c) 3rd-4th, (d) 5th-6th decimal digits.
 * Reading: every coordinate v of the state after each `stride` steps,
 * following `skip` transient steps, of each trajectory; a = |v|;
 *   kind 0: bin = trunc(v) + 64 (clamped to [0,127]);
 *   kind k = 1,2,3: bin = floor(RN(a * 10^{2k})) mod 100.
 * hist[(c*4 + kind)*128 + bin], c = x,y,z; accumulated (not cleared).                  */
void lorenz_ref_digit_hist(const double* ic, uint64_t lanes, uint32_t skip, uint32_t samples,
                           uint32_t stride, uint32_t dt_code, uint32_t integrator, uint64_t* hist) {
  const double scale[4] = {0.0, 100.0, 10000.0, 1000000.0};
  for (uint64_t l = 0; l < lanes; ++l) {
    double s[3] = {ic[3 * l], ic[3 * l + 1], ic[3 * l + 2]};
    lorenz_ref_iterate(s, dt_code, integrator, skip);
    for (uint32_t t = 0; t < samples; ++t) {
      lorenz_ref_iterate(s, dt_code, integrator, stride);
      for (int c = 0; c < 3; ++c) {
        double v = s[c];
        long long ip = (long long)v; /* truncation toward zero */
        long long b0 = ip + 64;
        if (b0 < 0) b0 = 0;
        if (b0 > 127) b0 = 127;
        hist[(c * 4 + 0) * 128 + b0] += 1;
        double a = fabs(v);
        for (int k = 1; k <= 3; ++k) {
          uint64_t m = (uint64_t)(a * scale[k]);
          hist[(c * 4 + k) * 128 + (m % 100)] += 1;
        }
      }
    }
  }
}

/* One global block b of a message of length n, from that block's own bytes:
 * blk_pt = the block's plaintext (len_b bytes), blk_ct receives len_b + 16 bytes. */
int lorenz_ref_encrypt_block(const uint8_t* pw, size_t pw_len, const lref_params* prm_in, uint64_t n,
                             uint64_t b, const uint8_t* blk_pt, uint8_t* blk_ct) {
  lref_params prm;
  fill_defaults(prm_in, &prm);
  if (check_params(&prm)) return LREF_E_ARG;
  if (pw_len < 3) return LREF_E_PASSWORD;
  if (b >= lorenz_ref_num_blocks(&prm, n)) return LREF_E_ARG;
  uint64_t B = prm.mode == LREF_FAST ? prm.block_size : n;
  uint64_t start = prm.mode == LREF_FAST ? b * B : 0;
  uint64_t len = n - start < B ? n - start : B;
  lref_km km;
  int st = block_km(pw, pw_len, &prm, b, &km);
  if (st) return st;
  return lorenz_ref_encrypt_stream(&km, &prm, blk_pt, (size_t)len, blk_ct, NULL);
}

int lorenz_ref_decrypt(const uint8_t* pw, size_t pw_len, const lref_params* prm_in, uint64_t n,
                       uint64_t b0, uint64_t b1, const uint8_t* ct, uint8_t* pt,
                       int64_t* first_bad, uint8_t* block_ok, int threads) {
  lref_params prm;
  fill_defaults(prm_in, &prm);
  if (check_params(&prm)) return LREF_E_ARG;
  if (pw_len < 3) return LREF_E_PASSWORD;
  uint64_t nb = lorenz_ref_num_blocks(&prm, n);
  if (b0 > b1 || b1 > nb) return LREF_E_ARG;
  *first_bad = -1;
  if (b0 == b1) return LREF_OK;
  uint8_t* ok = (uint8_t*)calloc((size_t)(b1 - b0), 1);
  int st = run_blocks(pw, pw_len, &prm, n, b0, b1, ct, pt, 1, ok, threads);
  if (st) { free(ok); return st; }
  uint64_t B = prm.mode == LREF_FAST ? prm.block_size : n;
  for (uint64_t b = b0; b < b1; ++b)
    if (!ok[b - b0]) { *first_bad = (int64_t)b; break; }
  if (*first_bad >= 0) {
    for (uint64_t b = b0; b < b1; ++b) {
      if (block_ok && ok[b - b0]) continue;
      uint64_t start = prm.mode == LREF_FAST ? b * B : 0;
      uint64_t end = prm.mode == LREF_FAST ? ((b + 1) * B < n ? (b + 1) * B : n) : n;
      memset(pt + start, 0, (size_t)(end - start));
    }
  }
  if (block_ok) memcpy(block_ok, ok, (size_t)(b1 - b0));
  free(ok);
  return *first_bad >= 0 ? LREF_E_INTEGRITY : LREF_OK;
}

/* ======================================================================== */
/* NEXT-4 analysis suite: the §4 statistics of the paper's Figs. 3 and 4.    */
/* Plain definitions, O(N) per output, O(N^2) per matrix (N = H*W).          */
/* ======================================================================== */

/* mean-centred samples d = x - mean(x) ("auto-correlation matrices"; S:434 mean-center) */
static double* centred(const uint8_t* x, uint64_t N) {
  double* d = (double*)malloc((size_t)N * sizeof(double));
  double sum = 0.0;
  for (uint64_t i = 0; i < N; ++i) sum += (double)x[i];
  const double mean = sum / (double)N;
  for (uint64_t i = 0; i < N; ++i) d[i] = (double)x[i] - mean;
  return d;
}

static double autocorr_lag(const double* d, uint32_t H, uint32_t W, uint32_t u, uint32_t v, double var) {
  if (var == 0.0) return (u == 0 && v == 0) ? 1.0 : 0.0; /* constant input: S:436 convention (Q25) */
  double c = 0.0;
  for (uint32_t i = 0; i < H; ++i)
    for (uint32_t j = 0; j < W; ++j)
      c += d[(uint64_t)i * W + j] * d[(uint64_t)((i + u) % H) * W + (j + v) % W];
  return c / var;
}

static double centred_var(const double* d, uint64_t N) {
  double var = 0.0;
  for (uint64_t i = 0; i < N; ++i) var += d[i] * d[i];
  return var;
}

/* Normalised circular 2-D autocorrelation of the H x W byte matrix x (row-major), Fig.3 / Q25:
 * r(u,v) = sum_{i,j} d[i][j] d[(i+u) mod H][(j+v) mod W] / sum_{i,j} d[i][j]^2,  d = x - mean(x).
 * r[u*W + v]; lag (0,0) at index 0.                                                         */
void lorenz_ref_autocorr(const uint8_t* x, uint32_t H, uint32_t W, double* r) {
  const uint64_t N = (uint64_t)H * W;
  double* d = centred(x, N);
  const double var = centred_var(d, N);
  for (uint32_t u = 0; u < H; ++u)
    for (uint32_t v = 0; v < W; ++v) r[(uint64_t)u * W + v] = autocorr_lag(d, H, W, u, v, var);
  free(d);
}

/* one lag of the same matrix (for sampled checks at sizes where the full matrix is too slow) */
double lorenz_ref_autocorr_at(const uint8_t* x, uint32_t H, uint32_t W, uint32_t u, uint32_t v) {
  const uint64_t N = (uint64_t)H * W;
  double* d = centred(x, N);
  const double r = autocorr_lag(d, H, W, u, v, centred_var(d, N));
  free(d);
  return r;
}

#define LREF_TWO_PI 6.283185307179586476925286766559
/* Power of the 2-D DFT at frequency (k,l), Fig.4 (g)-(i) / Q26:
 * F(k,l) = sum_{m,n} x[m][n] exp(-2 pi i (k m / H + l n / W)) = sum x exp(-2 pi i t / N),
 * t = (k m W + l n H) mod N;  P = |F|^2 / N^2 (so sum P = mean(x^2), Parseval).
 * cs: optional table cos/sin(2 pi t / N) for t < N (interleaved), else computed per term.   */
static double power_bin(const uint8_t* x, uint32_t H, uint32_t W, uint32_t k, uint32_t l, const double* cs) {
  const uint64_t N = (uint64_t)H * W;
  double re = 0.0, im = 0.0;
  for (uint32_t m = 0; m < H; ++m)
    for (uint32_t n = 0; n < W; ++n) {
      const uint64_t t = ((uint64_t)k * m % H * W + (uint64_t)l * n % W * H) % N;
      double c, s;
      if (cs) {
        c = cs[2 * t];
        s = cs[2 * t + 1];
      } else {
        const double a = LREF_TWO_PI * (double)t / (double)N;
        c = cos(a);
        s = sin(a);
      }
      const double v = (double)x[(uint64_t)m * W + n];
      re += v * c;
      im -= v * s;
    }
  const double N2 = (double)N * (double)N;
  return (re * re + im * im) / N2;
}

/* Full power spectrum, DC-centred: P(k,l) stored at ((k + H/2) mod H, (l + W/2) mod W). */
void lorenz_ref_power_spectrum(const uint8_t* x, uint32_t H, uint32_t W, double* P) {
  const uint64_t N = (uint64_t)H * W;
  double* cs = (double*)malloc((size_t)(2 * N) * sizeof(double));
  for (uint64_t t = 0; t < N; ++t) {
    const double a = LREF_TWO_PI * (double)t / (double)N;
    cs[2 * t] = cos(a);
    cs[2 * t + 1] = sin(a);
  }
  for (uint32_t k = 0; k < H; ++k)
    for (uint32_t l = 0; l < W; ++l)
      P[(uint64_t)((k + H / 2) % H) * W + (l + W / 2) % W] = power_bin(x, H, W, k, l, cs);
  free(cs);
}

/* one frequency (k,l) (unshifted indices) of the same spectrum */
double lorenz_ref_power_at(const uint8_t* x, uint32_t H, uint32_t W, uint32_t k, uint32_t l) {
  return power_bin(x, H, W, k, l, NULL);
}

/* Spectral flatness of a DC-centred spectrum: geometric mean / arithmetic mean of the
 * non-DC bins. No non-DC power at all -> 0 (Q26). A zero bin makes the geometric mean 0.     */
double lorenz_ref_spectral_flatness(const double* P, uint32_t H, uint32_t W) {
  const uint64_t N = (uint64_t)H * W, dc = (uint64_t)(H / 2) * W + W / 2;
  double slog = 0.0, sum = 0.0;
  for (uint64_t i = 0; i < N; ++i) {
    if (i == dc) continue;
    slog += log(P[i]);
    sum += P[i];
  }
  const double M = (double)(N - 1);
  if (sum == 0.0) return 0.0;
  return exp(slog / M) / (sum / M);
}
