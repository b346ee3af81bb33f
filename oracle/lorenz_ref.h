/* lorenz_ref.h — CPU ORACLE for the per-block chaotic operation mode of
 * Marco, Martinez & Bruno, "Fast, parallel and secure cryptography algorithm
 * using Lorenz's attractor" (arXiv 1201.3114).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1201_3114_b200/) never links, imports or calls it,
 * and shares no code, header, table or constant generator with it.
 *
 * Plain, slow, obviously-correct C: scalar IEEE binary64, round-to-nearest,
 * no fused multiply-add (built with -O2 -ffp-contract=off -fno-fast-math),
 * operations in the order of the paper and of the readings in DESIGN.md §3.
 * Citations: "P:n" = PAPER.md line n (section / equation); "S:n" = SPEC.md
 * line n; "Q*" = reading number in DESIGN.md §3 (= SURVEY.md §8c.2).
 */
#ifndef LORENZ_REF_H
#define LORENZ_REF_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (values mirror the SPEC CLI exit-code meanings) */
#define LREF_OK 0
#define LREF_E_INTEGRITY 1
#define LREF_E_ARG 2
#define LREF_E_PASSWORD 3
#define LREF_E_LENGTH 4
#define LREF_E_DIVERGENCE 5

#define LREF_STRONG 0
#define LREF_FAST 1
#define LREF_RK4 0
#define LREF_EULER 1
#define LREF_RK4_FMA 2 /* NEXT-3 */

typedef struct {
  uint32_t mode;       /* LREF_STRONG / LREF_FAST                                   */
  uint32_t n_it;       /* iterations per character; 0 -> 3000 / 100      */
  uint32_t dt_code;    /* 0:0.01 1:0.005 2:0.02 3:0.027 (P:187 range)        */
  uint32_t block_size; /* FAST block size B (bytes); 0 -> 1024                       */
  uint32_t integrator; /* LREF_RK4 (north star) / LREF_EULER (NEXT-1) / LREF_RK4_FMA (NEXT-3) */
  uint32_t variant;    /* NEXT-4 Step-3 reading variants; 0 = the adopted reading (Q13)          */
} lref_params;

/* NEXT-4 variant bits */
#define LREF_V_ORDER_MASK 3u
#define LREF_V_LITERAL 1u    /* literal textual order of P:320-322 */
#define LREF_V_CYCLIC 2u     /* cyclic reading of the index [(i+2) mod 3]+1 */
#define LREF_V_DISTINCT_K 4u /* k2 = 7 - k1 */

/* Everything derived from one stream password (§3.1). */
typedef struct {
  uint64_t a[3];     /* Eqs.2-4 */
  int L;             /* floor(n_pi/3) */
  int d;             /* exponent of g's divisor */
  double ap[3];      /* a' = g(a) */
  double lam[3];     /* lambda (Eq.5 ranges) */
  double r0[3];      /* r0 = a' + lambda (Eq.5) */
  int mu[3];         /* mu0 */
  int k[3];          /* k_i in {3,4} */
  int k3chain;       /* k3 of Step 3, in [1,6] */
  int omega[3];      /* Omega0 (Eq.7) */
  double alpha[3];   /* alpha0 (Eq.6, n=0) */
  uint64_t hom[3];   /* BE64 prefixes of hash(i a) (Eq.7) before the mod */
} lref_km;

/* ---- components (each pinned separately in tests/) ---- */
void lorenz_ref_sha256(const uint8_t* msg, size_t len, uint8_t out[32]);
int lorenz_ref_pack(const uint8_t* pw, size_t n, uint64_t a[3]);
int lorenz_ref_norm_exponent(int L);
void lorenz_ref_normalize(const uint64_t a[3], int L, double ap[3]);
void lorenz_ref_lambda(const uint64_t a[3], double lam[3]);
void lorenz_ref_mu(const uint64_t a[3], int mu[3]);
void lorenz_ref_k_omega(const uint8_t* pw, size_t n, const uint64_t a[3], int k[3],
                        int* k3chain, int omega[3]);
int lorenz_ref_R(double alpha, int omega);
double lorenz_ref_theta(int p, int omega3);
int lorenz_ref_encode(int p, int ksum);
int lorenz_ref_decode(int c, int ksum);
void lorenz_ref_rhs(const double s[3], double f[3]);
void lorenz_ref_rk4_step(double s[3], double h);
void lorenz_ref_euler_step(double s[3], double h);
void lorenz_ref_rk4fma_step(double s[3], double h);
void lorenz_ref_iterate(double s[3], uint32_t dt_code, uint32_t integrator, uint64_t n);
double lorenz_ref_dt(uint32_t dt_code);
int lorenz_ref_normalize_password(const uint8_t* pw, size_t n, uint8_t out[23], size_t* n_out);
void lorenz_ref_subpassword(const uint8_t* pw, size_t n, uint32_t b, uint8_t out[18]);
int lorenz_ref_keymaterial(const uint8_t* pw_norm, size_t n, lref_km* km);
void lorenz_ref_apply_variant(lref_km* km, uint32_t variant);

/* ---- one stream (§3.2 Steps 1-3) ----
 * encrypt: c must hold len+16 bytes (body ‖ encrypted sentinel).
 * decrypt: clen >= 16; p receives clen-16 bytes; *ok = sentinel matched.
 * trace (nullable): r after each advanced character, 3 doubles per char.     */
int lorenz_ref_encrypt_stream(const lref_km* km, const lref_params* prm, const uint8_t* p,
                              size_t len, uint8_t* c, double* trace);
int lorenz_ref_decrypt_stream(const lref_km* km, const lref_params* prm, const uint8_t* c,
                              size_t clen, uint8_t* p, int* ok, double* trace);

/* ---- message framing (FAST blocks / STRONG single stream) ---- */
uint64_t lorenz_ref_num_blocks(const lref_params* prm, uint64_t n);
uint64_t lorenz_ref_ct_len(const lref_params* prm, uint64_t n);
int lorenz_ref_pt_len(const lref_params* prm, uint64_t ct_len, uint64_t* n_out);
/* Global blocks [b0,b1) of a message of plaintext length n. pt/ct point at the
 * start of the FULL message buffers. tag_xor = XOR of the blocks' tags.
 * threads: 0 -> all online cores.                                             */
int lorenz_ref_encrypt(const uint8_t* pw, size_t pw_len, const lref_params* prm, uint64_t n,
                       uint64_t b0, uint64_t b1, const uint8_t* pt, uint8_t* ct,
                       uint8_t tag_xor[16], int threads);
/* NEXT-4 analysis: Fig.1 digit histograms; hist: uint64[3*4*128], accumulated. */
void lorenz_ref_digit_hist(const double* ic, uint64_t lanes, uint32_t skip, uint32_t samples,
                           uint32_t stride, uint32_t dt_code, uint32_t integrator, uint64_t* hist);
/* NEXT-4 analysis, §4 Figs. 3-4 (readings Q25-Q27). x: H x W bytes, row-major.
 * autocorr: r[u*W+v] = normalised circular 2-D autocorrelation at lag (u,v), r[0] = 1.
 * power_spectrum: P = |DFT|^2 / (HW)^2, DC-centred (bin (k,l) at ((k+H/2)%H, (l+W/2)%W)).
 * *_at: one lag / one (unshifted) frequency. flatness: non-DC geometric / arithmetic mean. */
void lorenz_ref_autocorr(const uint8_t* x, uint32_t H, uint32_t W, double* r);
double lorenz_ref_autocorr_at(const uint8_t* x, uint32_t H, uint32_t W, uint32_t u, uint32_t v);
void lorenz_ref_power_spectrum(const uint8_t* x, uint32_t H, uint32_t W, double* P);
double lorenz_ref_power_at(const uint8_t* x, uint32_t H, uint32_t W, uint32_t k, uint32_t l);
double lorenz_ref_spectral_flatness(const double* P, uint32_t H, uint32_t W);
/* One global block b of a message of length n, from that block's own bytes. */
int lorenz_ref_encrypt_block(const uint8_t* pw, size_t pw_len, const lref_params* prm, uint64_t n,
                             uint64_t b, const uint8_t* blk_pt, uint8_t* blk_ct);
/* block_ok (nullable): per-block verdict for [b0,b1); when given, only failing
 * blocks are zero-filled, otherwise the whole range is zero-filled on failure. */
int lorenz_ref_decrypt(const uint8_t* pw, size_t pw_len, const lref_params* prm, uint64_t n,
                       uint64_t b0, uint64_t b1, const uint8_t* ct, uint8_t* pt,
                       int64_t* first_bad, uint8_t* block_ok, int threads);

#ifdef __cplusplus
}
#endif
#endif
