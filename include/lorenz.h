/* lorenz.h — C ABI of the B200-native hot path of the parallel Lorenz-attractor
 * cipher of Marco, Martinez & Bruno, arXiv 1201.3114 ("Fast, parallel and secure
 * cryptography algorithm using Lorenz's attractor"): the per-block chaotic
 * operation mode.
 *
 * Library: paper_1201_3114_b200/csrc/liblorenz.so (CUDA, sm_100a). Python binding:
 * paper_1201_3114_b200/lorenz.py (same names, argument marshalling only).
 *
 * Citations: "P:n" = PAPER.md line n (section, equation); "S:n" = SPEC.md line n;
 * "Qn" = reading n of DESIGN.md §3. The operation every entry point computes is
 * defined in DESIGN.md §2; in short, for each block b of a message:
 *   key schedule  (§3.1, Eqs.2-7)   password -> a, a', lambda, r0, mu, alpha, k, Omega
 *   per character (§3.2, Steps 1-3) C_i = [P_i + R(alpha1,Omega1) + R(alpha2,Omega2)] mod 2^8
 *                                              (Eqs.8-9); Theta = P_i/10^{3+Omega3} added to r[mu3];
 *                                              n_it fixed-step RK4 steps of the Lorenz system (Eq.1, Q1-Q3);
 *                                              mu, alpha, Omega update; r += a'
 *   integrity     (§2)              16-byte sentinel "LORENZCHAOS-MAC1" appended to every
 *                                              block's plaintext; its ciphertext is the block tag (Q15)
 *   parallel mode (§5)              FAST: fixed B-byte blocks, block b keyed by
 *                                              SHA-256(pw || BE32 b)[0:18] (Q16); STRONG: one stream.
 *
 * Conventions shared by every call
 *   - All arithmetic is IEEE binary64 round-to-nearest with no fused multiply-add, in
 *     the operation order of DESIGN.md §2, so results are bit-identical on every
 *     conforming implementation (and to the CPU oracle in oracle/).
 *   - Device pointers are plain CUDA device addresses (e.g. torch.Tensor.data_ptr()),
 *     16-byte aligned; the caller owns every buffer. Any device-accessible address works,
 *     including mapped page-locked host memory (UVA): the chain kernels then read and write
 *     it over PCIe themselves, window by window (the direct mode of lorenz_encrypt_host).
 *     Pageable host memory is refused (LORENZ_E_ARG) by the chain and batch calls rather than
 *     left to fault inside a kernel. `cuda_stream` is a cudaStream_t
 *     (NULL = legacy default stream). Calls without the _async suffix enqueue their
 *     work on that stream and synchronise it before returning.
 *   - Errors are returned, never raised: no abort/exit. Argument errors are reported
 *     before anything is enqueued. After LORENZ_E_CUDA, lorenz_last_error() holds the
 *     CUDA error text of the calling thread.
 *   - Layout: block b of the message covers plaintext bytes [b*B, min(n,(b+1)*B)) and
 *     ciphertext bytes [b*(B+16), b*(B+16) + len_b + 16): its body then its 16-byte
 *     tag (Q21). STRONG is a single block with B = n.
 */
#ifndef LORENZ_H
#define LORENZ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LORENZ_TAG_BYTES 16
#define LORENZ_KEY_BYTES 384
#define LORENZ_ABI_VERSION 2

typedef enum {
  LORENZ_OK = 0,
  LORENZ_E_INTEGRITY = 1,  /* a recovered sentinel differs; mirrors SPEC exit code 1 */
  LORENZ_E_ARG = 2,        /* NULL / misaligned pointer, bad range or params                           */
  LORENZ_E_PASSWORD = 3,   /* password shorter than 3 bytes (Q17)                                 */
  LORENZ_E_LENGTH = 4,     /* ciphertext length inconsistent with the block size                 */
  LORENZ_E_DIVERGENCE = 5, /* guard: non-finite or |x|,|y|>100, z outside [-50,150] (Q18)                */
  LORENZ_E_CUDA = 6,       /* a CUDA runtime error; see lorenz_last_error()                              */
  LORENZ_E_IO = 7,         /* file open/read/write error (file calls); mirrors SPEC exit code 3  */
  LORENZ_E_FORMAT = 8      /* bad envelope magic / version / field                                */
} lorenz_status;

typedef enum { LORENZ_STRONG = 0, LORENZ_FAST = 1 } lorenz_mode;           /* P:446-448 §5 */
/* Q1; LORENZ_RK4_FMA (NEXT-3) is RK4 with fused multiply-adds at fixed sites
 * (DESIGN.md §2b): also IEEE-deterministic, but a different cipher definition. */
typedef enum { LORENZ_RK4 = 0, LORENZ_EULER = 1, LORENZ_RK4_FMA = 2 } lorenz_integrator;

typedef struct {
  uint32_t mode;       /* lorenz_mode                                                             */
  uint32_t n_it;       /* RK4 steps per character; 0 -> 3000 (STRONG) / 100 (FAST)      */
  uint32_t dt_code;    /* step h: 0 -> 0.01, 1 -> 0.005, 2 -> 0.02, 3 -> 0.027 (0 < h <= 0.027) */
  uint32_t block_size; /* FAST block size B: >= 1024 and a multiple of 16; 0 -> 1024. STRONG: ignored */
  uint32_t integrator; /* lorenz_integrator; LORENZ_EULER is the paper's own discretisation  */
  uint32_t variant;    /* NEXT-4 Step-3 reading: 0 = adopted reading Q13;
                          bits 0-1: 1 = literal textual order, 2 = cyclic index; bit 2: k2 = 7 - k1   */
} lorenz_params;

#define LORENZ_V_LITERAL 1u
#define LORENZ_V_CYCLIC 2u
#define LORENZ_V_DISTINCT_K 4u

/* Key: POD, caller-owned, trivially copyable, no heap. Holds the params, the exact
 * binary64 bit patterns of sigma, rho, beta, h, h/2, h/6, and the password:
 * STRONG: the normalised password (3..23 bytes; longer ones are replaced by
 * SHA-256(pw)[0:18]); FAST: the SHA-256 midstate of the raw password so the
 * device finishes SHA-256(pw || BE32 b) per block. */
typedef struct { uint8_t opaque[LORENZ_KEY_BYTES]; } lorenz_key;

/* Device-side result slot for the _async calls (caller-allocated device memory,
 * 32 bytes, 16-byte aligned; initialise with lorenz_result_init_async). */
typedef struct {
  uint8_t tag_xor[16];       /* XOR of the tags of the processed blocks (Q15)              */
  uint64_t first_bad;        /* min failing global block index, UINT64_MAX if none         */
  uint32_t status;           /* OR of per-lane flags: 1 = integrity, 4 = divergence         */
  uint32_t reserved;
} lorenz_result;

/* ---- host-only helpers (no device work) ---- */

/* Derive a key. pw: pw_len bytes (host). p: NULL -> FAST defaults.
 * Errors: LORENZ_E_PASSWORD if pw_len < 3; LORENZ_E_ARG for bad params/NULL.
 * Deterministic: same bytes and params -> bit-identical key. */
lorenz_status lorenz_keysetup(const uint8_t* pw, size_t pw_len, const lorenz_params* p,
                              lorenz_key* out);
/* Effective params stored in a key (defaults filled in). */
lorenz_status lorenz_key_params(const lorenz_key* k, lorenz_params* out);
/* FAST: max(1, ceil(n/B)); STRONG: 1. 0 for an invalid key. */
uint64_t lorenz_num_blocks(const lorenz_key* k, uint64_t n);
/* n + 16 * lorenz_num_blocks(k, n). */
uint64_t lorenz_ct_len(const lorenz_key* k, uint64_t n);
/* Inverse of lorenz_ct_len; LORENZ_E_LENGTH if no n maps to ct_len. */
lorenz_status lorenz_pt_len(const lorenz_key* k, uint64_t ct_len, uint64_t* n_out);
/* Launch plan of the chain kernel for global blocks [b0, b1) of an n-byte message (host
 * only, no device work; uses the current device's SM count, 148 without a device).
 * kind 0 = wave kernel: one lane per block, one warp per 32 blocks, grid = ceil(lanes / cta).
 * kind 1 = balanced kernel: grid = one CTA of `cta` threads per SM; the
 * lanes' 32-block units, (B+16)/16 chunks each, are dealt to `slots` resident warps,
 * `chunks_per_slot` chunks each, a unit cut by a slot boundary handing its chain states
 * from one warp to the next. Chooses exactly as the encrypt/decrypt/verify calls do
 * (lorenz_set_tuning overrides included). LORENZ_E_ARG on a NULL or bad key/out or an
 * out-of-range block range. */
typedef struct {
  uint32_t kind;            /* 0 wave, 1 balanced                                     */
  uint32_t cta;             /* threads per CTA                                        */
  uint64_t grid;            /* CTAs                                                   */
  uint64_t lanes;           /* b1 - b0 chains                                         */
  uint64_t slots;           /* balanced: warp slots sharing the units (0 for wave)    */
  uint64_t chunks_per_slot; /* balanced: 16-character chunks per slot (0 for wave); with a
                               skew, the slots of a CTA's warps w get chunks_per_slot +
                               (w / 4) * chunks_skew (later warps of a CTA run faster)     */
  uint64_t chunks_skew;     /* balanced: see above (0: equal slots)                     */
} lorenz_plan;
lorenz_status lorenz_launch_plan(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1,
                                 lorenz_plan* out);
const char* lorenz_status_string(lorenz_status s);

/* Tuning / test overrides of the chain kernels' launch plan (process-wide; normal use never
 * needs them, and the library reads no environment variables). Fields:
 *   schedule   0 automatic (the rule of DESIGN.md §4), 1 force the wave kernel, 2 force the
 *              balanced kernel (any size, RK4 / Euler / RK4-FMA);
 *   seg_slots  balanced kernel: warp slots (0 = SMs x warps per CTA; clamped to the 32-block
 *              units, so every unit spans at most two slots);
 *   seg_skew   balanced kernel: slot skew per warp group in per mille of a slot, 0..1000 (-1 = the
 *              default 8, 0 = equal slots);
 *   cta        wave kernel: threads per CTA (0 = automatic; 128, 256 or 512).
 * t = NULL restores every default. Thread-safe; applies to plans made after the call.
 * LORENZ_E_ARG for a field out of range (nothing is changed then). */
typedef struct {
  uint32_t schedule;
  uint32_t seg_slots;
  int32_t seg_skew;
  uint32_t cta;
} lorenz_tuning;
lorenz_status lorenz_set_tuning(const lorenz_tuning* t);
const char* lorenz_last_error(void);
int lorenz_abi_version(void);

/* ---- device calls: global blocks [b0, b1) of a message of total plaintext length n ----
 * pt / ct are DEVICE pointers to the start of the SLICE: pt = message + b0*B,
 * ct = ciphertext + b0*(B+16) (so a rank can hold only its own slice). The slice
 * holds min(n, b1*B) - b0*B plaintext bytes and that + 16*(b1-b0) ciphertext bytes.
 * pt and ct must not overlap. b0 == b1 is a no-op (tag_xor = 0). */

/* C = E_pi(P) (Eq.9, Steps 1-3). tag_xor (host, 16 B, nullable) receives the
 * XOR of the tags of blocks [b0,b1). */
lorenz_status lorenz_encrypt(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1,
                             const uint8_t* pt, uint8_t* ct, uint8_t tag_xor[16],
                             void* cuda_stream);

/* P = D_pi(C) (Eq.10; the chain advances with the recovered byte).
 * first_bad_block (host, nullable): min failing global block, -1 if none.
 * block_ok (DEVICE, nullable, b1-b0 bytes): per-block verdict 1/0. With block_ok,
 * only failing blocks' plaintext is zero-filled; without it, the whole slice is
 * zero-filled on failure (so unauthenticated plaintext is never released).
 * Returns LORENZ_E_INTEGRITY if any block fails. */
lorenz_status lorenz_decrypt(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1,
                             const uint8_t* ct, uint8_t* pt, int64_t* first_bad_block,
                             uint8_t* block_ok, void* cuda_stream);

/* Decrypt without writing plaintext: integrity check only.
 * tag_xor (host, nullable): XOR of the ciphertext's block tags. */
lorenz_status lorenz_verify(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1,
                            const uint8_t* ct, int64_t* first_bad_block, uint8_t tag_xor[16],
                            void* cuda_stream);

/* ---- asynchronous forms: enqueue and return; results accumulate into `res`
 * (device, see lorenz_result; 16-byte aligned, else LORENZ_E_ARG: the kernels update it with
 * 64-bit atomics). Safe inside CUDA graph capture. ---- */
lorenz_status lorenz_result_init_async(lorenz_result* res, void* cuda_stream);
lorenz_status lorenz_encrypt_async(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1,
                                   const uint8_t* pt, uint8_t* ct, lorenz_result* res,
                                   void* cuda_stream);
lorenz_status lorenz_decrypt_async(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1,
                                   const uint8_t* ct, uint8_t* pt, uint8_t* block_ok,
                                   lorenz_result* res, void* cuda_stream);
lorenz_status lorenz_verify_async(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1,
                                  const uint8_t* ct, lorenz_result* res, void* cuda_stream);

/* ---- batch (C5 sweeps): S independent messages of equal length n, one key each
 * (all keys must share mode/n_it/dt/B/integrator, else LORENZ_E_ARG). keys: HOST
 * array of S keys. Message s is at pts + s*n, its ciphertext at cts + s*ct_len(n),
 * its tag XOR at tags + 16*s (all DEVICE; tags 16-byte aligned, else LORENZ_E_ARG).
 * One launch, lane = (message, block). */
lorenz_status lorenz_encrypt_batch(const lorenz_key* keys, uint32_t S, uint64_t n,
                                   const uint8_t* pts, uint8_t* cts, uint8_t* tags,
                                   void* cuda_stream);

/* ---- C5 statistics (§4: histograms/entropy of the ciphertext; "slightly
 * different passwords"): integer-exact reductions on DEVICE buffers, enqueued on the stream.
 * `spans` is a HOST array (copied before return). ---- */
typedef struct {
  uint64_t a_off; /* byte offset of the span in buffer a */
  uint64_t b_off; /* byte offset of the span in buffer b (ignored by lorenz_histograms) */
  uint64_t len;   /* span length in bytes */
} lorenz_span;

/* For each of `count` spans: out[3i] = differing bits between a[a_off..] and
 * b[b_off..] over len bytes, out[3i+1] = differing bytes, out[3i+2] = bytes whose least
 * significant bits are equal. out: DEVICE uint64[3*count], overwritten. */
lorenz_status lorenz_compare_spans(const uint8_t* a, const uint8_t* b, const lorenz_span* spans,
                                   uint32_t count, uint64_t* out, void* cuda_stream);
/* 256-bin byte histogram of each span of a: hist: DEVICE uint64[256*count], overwritten. */
lorenz_status lorenz_histograms(const uint8_t* a, const lorenz_span* spans, uint32_t count,
                                uint64_t* hist, void* cuda_stream);

/* ---- NEXT-4 analysis: Fig.1 of the paper, frequency of the integer part and of
 * the decimal digit pairs 1-2, 3-4, 5-6 of the Lorenz coordinates. `lanes` trajectories start
 * at ic (DEVICE, lanes x 3 doubles, x y z), run `skip` transient steps, then every coordinate
 * of the state after each `stride` steps is binned, `samples` times:
 *   hist[(c*4 + kind)*128 + bin], c = x,y,z; kind 0: bin = trunc(v) + 64 (clamped to 0..127);
 *   kind k = 1..3: bin = floor(RN(|v| * 10^{2k})) mod 100.
 * hist: DEVICE uint64[3*4*128], overwritten. Same integrators / dt codes as the cipher. */
lorenz_status lorenz_digit_histograms(const double* ic, uint64_t lanes, uint32_t skip, uint32_t samples,
                                      uint32_t stride, uint32_t dt_code, uint32_t integrator,
                                      uint64_t* hist, void* cuda_stream);

/* ---- ragged batches (serving many messages of different lengths in one launch) ----
 * `count` FAST messages, message s of n[s] plaintext bytes under keys[s] (all keys with equal
 * params). Arrays n / *_off are HOST arrays of `count` entries; pts / cts / tags are DEVICE
 * pointers (16-byte aligned). Message s's plaintext is at pts + pt_off[s] and its ciphertext
 * (lorenz_ct_len(n[s]) bytes, blocks as in the single-message layout) at cts + ct_off[s]; every
 * offset a multiple of 16; output ranges must not overlap each other or the input. tags (16*count
 * bytes) receives each message's tag XOR (decrypt: of the received ciphertext). One launch over
 * all blocks of all messages (a lane finds its message by binary search over the block prefix
 * sums). Synchronous. Decrypt: first_bad (HOST, count entries) = the message's lowest failing
 * block or -1; a failing message's plaintext is zero-filled; LORENZ_E_INTEGRITY if any failed. */
lorenz_status lorenz_encrypt_ragged(const lorenz_key* keys, uint32_t count, const uint64_t* n,
                                    const uint64_t* pt_off, const uint64_t* ct_off, const uint8_t* pts,
                                    uint8_t* cts, uint8_t* tags, void* cuda_stream);
lorenz_status lorenz_decrypt_ragged(const lorenz_key* keys, uint32_t count, const uint64_t* n,
                                    const uint64_t* ct_off, const uint64_t* pt_off, const uint8_t* cts,
                                    uint8_t* pts, uint8_t* tags, int64_t* first_bad, void* cuda_stream);

/* ---- NEXT-4 §4 analysis: Fig.3 autocorrelation matrices and Fig.4 2-D Fourier
 * power spectra; readings Q25-Q27.
 * x: DEVICE pointer to an H x W byte matrix, row-major (e.g. the first H*W bytes of a
 * ciphertext); H and W powers of two in [2, 4096] (no zero padding; else LORENZ_E_ARG).
 * Outputs are DEVICE pointers (8-aligned), written stream-ordered on `cuda_stream`; a
 * workspace of 16*H*W bytes comes from the stream-ordered pool. FP64 FFTs: results agree
 * with the plain-sum definitions within the bounds of DESIGN.md §2e, not bit for bit.
 *
 * lorenz_autocorrelation: r[u*W + v] = sum_ij d[i][j] d[(i+u)%H][(j+v)%W] / sum_ij d[i][j]^2,
 *   d = x - mean(x) (normalised circular 2-D autocorrelation; r[0] = 1; a constant x gives
 *   r[0] = 1 and 0 elsewhere). r must not overlap x.
 * lorenz_power_spectrum: power[((k+H/2)%H)*W + (l+W/2)%W] = |F(k,l)|^2 / (HW)^2, F the 2-D DFT
 *   (DC-centred; sum of power = mean(x^2)). flatness (nullable, device double): geometric /
 *   arithmetic mean of the non-DC bins, 0 when they are all zero (deterministic reduction). */
lorenz_status lorenz_autocorrelation(const uint8_t* x, uint32_t H, uint32_t W, double* r, void* cuda_stream);
lorenz_status lorenz_power_spectrum(const uint8_t* x, uint32_t H, uint32_t W, double* power, double* flatness,
                                    void* cuda_stream);

/* ---- end to end from HOST buffers (the user-facing call of a file encryptor):
 * blocks [b0,b1) of an n-byte message; pt_host / ct_host are HOST pointers to the
 * slice starts (same slice convention as the device calls; [0, num_blocks) is the
 * whole message).
 * n_chunks = 0 (automatic) with both slices in page-locked memory mapped into the current
 * device's address space (cudaHostAlloc / cudaMallocHost, torch pin_memory(),
 * cudaHostRegister(..., cudaHostRegisterMapped)): DIRECT streaming — one chain launch reads
 * the input and writes the output over PCIe itself (no device buffers; the transfers overlap
 * the arithmetic window by window, so the call takes the kernel's time: 98.9 % of the device
 * rate at 64 MiB, 99.98 % at 1 GiB, profiles/e2e_probe_r02.jsonl).
 * Otherwise (pageable memory, or n_chunks > 0) the STAGED pipeline: host->device copies,
 * kernels and device->host copies are
 * pipelined over `n_chunks` block-aligned chunks (0 -> automatic: first and last chunk the
 * smallest that keep 2 warps of 32 blocks per SM sub-partition, middle chunks <= 128 MiB, one
 * chunk below twice that minimum; n_chunks > 0: equal chunks) on the current device. Chunk
 * kernels run one at a time, each overlapped with the neighbouring chunks' copies. Chunk c runs on internal stream c % S, S = min(8, chunks), whose
 * device buffers hold one chunk and are reused in stream order, so device memory is
 * bounded by ~2 x S chunks whatever the slice size (slices larger than HBM work).
 * Pinned host memory gives overlapped copies; pageable memory works but copies
 * synchronously. Buffers come from the stream-ordered pool (kept cached). Synchronous.
 * decrypt: on LORENZ_E_INTEGRITY the whole host plaintext slice is zero-filled. */
lorenz_status lorenz_encrypt_host(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1,
                                  const uint8_t* pt_host, uint8_t* ct_host, uint8_t tag_xor[16],
                                  uint32_t n_chunks);
lorenz_status lorenz_decrypt_host(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1,
                                  const uint8_t* ct_host, uint8_t* pt_host,
                                  int64_t* first_bad_block, uint32_t n_chunks);

/* ---- envelope + streaming file path (NEXT-2; SPEC envelope S:344-390) ----
 * File = 24-byte header || ciphertext (the concatenation of the blocks' body || tag).
 * Header (little-endian): "LZX1" | u8 version=1 | u8 mode | u8 flags (bits 0-1: integrator,
 * an extension; SPEC reserves the byte as 0 = RK4 here) | u8 dt_code | u32 n_it |
 * u32 chunk_size (= block size B; 0 in STRONG mode) | u64 payload_len (plaintext bytes). */
#define LORENZ_ENVELOPE_BYTES 24

/* Header of an n-byte message encrypted under k. */
lorenz_status lorenz_envelope_write(const lorenz_key* k, uint64_t n, uint8_t hdr[LORENZ_ENVELOPE_BYTES]);
/* Parse a header: params (for lorenz_keysetup with the password), payload length n and the
 * ciphertext length that must follow. LORENZ_E_LENGTH if len < 24; LORENZ_E_FORMAT for a
 * bad magic / version / mode / field combination. */
lorenz_status lorenz_envelope_read(const uint8_t* hdr, size_t len, lorenz_params* p, uint64_t* n,
                                   uint64_t* ct_len);

/* Encrypt the file at in_path into the envelope file out_path (HOST paths). The file is
 * streamed through the GPU in block-aligned chunks of about chunk_bytes (0 -> 32 MiB),
 * four chunks in flight (read -> H2D -> kernel -> D2H -> write), so files larger than
 * HBM work. The output is written to out_path + ".partial" and renamed on success.
 * tag_xor (nullable) receives the message digest. Uses the current CUDA device. */
lorenz_status lorenz_encrypt_file(const char* in_path, const char* out_path, const uint8_t* pw,
                                  size_t pw_len, const lorenz_params* p, uint64_t chunk_bytes,
                                  uint8_t tag_xor[16]);
/* Decrypt an envelope file. The params come from the header. On LORENZ_E_INTEGRITY no
 * output file is left behind (nothing unauthenticated is released) and *first_bad_block
 * (nullable) holds the first failing block; LORENZ_E_LENGTH for a truncated body. */
lorenz_status lorenz_decrypt_file(const char* in_path, const char* out_path, const uint8_t* pw,
                                  size_t pw_len, uint64_t chunk_bytes, int64_t* first_bad_block);

#ifdef __cplusplus
}
#endif
#endif /* LORENZ_H */
