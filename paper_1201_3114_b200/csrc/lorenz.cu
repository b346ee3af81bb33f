// lorenz.cu — host side of liblorenz.so: the C ABI of include/lorenz.h.
//
// Validates arguments, builds the per-launch constant block and password material
// from a lorenz_key, launches the sm_100a kernels of lorenz_device.cuh on the
// caller's stream, and reads back tag / verdict. No CPU fallback: every byte of
// ciphertext is produced on the GPU.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only; ranges are no-ops unless a profiler attaches

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/lorenz.h"
#include "lorenz_device.cuh"
#include "seg_launch.h"
#include "analysis.cuh"
#include "sha256.cuh"
#include "stats.cuh"

namespace {

constexpr uint32_t kMagic = 0x314B5A4Cu;  // "LZK1"

struct KeyImpl {
  uint32_t magic;
  uint32_t abi;
  lorenz_params prm;        // defaults filled in
  uint32_t pw_len;          // STRONG: normalised password length (3..23)
  double sigma, rho, beta;
  double h, h2, h6;         // step (P:187 range), h*0.5, h/6.0 — rounded once, here
  uint8_t pw[24];           // STRONG: normalised password
  uint32_t mid[8];          // FAST: SHA-256 midstate of the raw password's full blocks
  uint64_t raw_len;         // FAST: raw password length
  uint32_t tail_len;        // FAST: raw_len mod 64
  uint8_t tail[64];         // FAST: the raw password's last partial block
};
static_assert(sizeof(KeyImpl) <= LORENZ_KEY_BYTES, "key layout exceeds the ABI size");

thread_local std::string g_err;

// NVTX range over a host call (tracing for nsys / ncu --nvtx filters)
struct Trace {
  explicit Trace(const char* name) { nvtxRangePushA(name); }
  ~Trace() { nvtxRangePop(); }
};

const KeyImpl* impl(const lorenz_key* k) {
  if (!k) return nullptr;
  const KeyImpl* K = reinterpret_cast<const KeyImpl*>(k->opaque);
  return (K->magic == kMagic && K->abi == LORENZ_ABI_VERSION) ? K : nullptr;
}

bool cuda_ok(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return true;
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return false;
}

double dt_of(uint32_t code) {
  switch (code) {
    case 0: return 0.01;
    case 1: return 0.005;
    case 2: return 0.02;
    default: return 0.027;
  }
}

uint64_t nblocks(const KeyImpl* K, uint64_t n) {
  if (K->prm.mode == LORENZ_STRONG) return 1;
  const uint64_t B = K->prm.block_size;
  const uint64_t nb = (n + B - 1) / B;
  return nb ? nb : 1;
}

uint64_t block_B(const KeyImpl* K, uint64_t n) {
  return K->prm.mode == LORENZ_FAST ? K->prm.block_size : n;
}

// plaintext / ciphertext byte extents of blocks [b0,b1)
void slice_bytes(const KeyImpl* K, uint64_t n, uint64_t b0, uint64_t b1, uint64_t* pt_bytes,
                 uint64_t* ct_bytes) {
  const uint64_t B = block_B(K, n);
  const uint64_t hi = (K->prm.mode == LORENZ_FAST) ? ((b1 * B < n) ? b1 * B : n) : n;
  const uint64_t lo = (K->prm.mode == LORENZ_FAST) ? b0 * B : 0;
  *pt_bytes = hi - lo;
  *ct_bytes = hi - lo + 16 * (b1 - b0);
}

void put_words_be(const uint8_t* bytes, int nwords, uint32_t* w) {
  for (int i = 0; i < nwords; ++i)
    w[i] = (uint32_t)bytes[4 * i] << 24 | (uint32_t)bytes[4 * i + 1] << 16 |
           (uint32_t)bytes[4 * i + 2] << 8 | bytes[4 * i + 3];
}

lz::DevKey make_devkey(const KeyImpl* K) {
  lz::DevKey d;
  std::memset(&d, 0, sizeof d);
  if (K->prm.mode == LORENZ_FAST) {
    for (int i = 0; i < 8; ++i) d.mid[i] = K->mid[i];
    uint8_t fin[128] = {0};
    const uint32_t t = K->tail_len;
    std::memcpy(fin, K->tail, t);
    // fin[t..t+3] = BE32(b), filled per lane on the device
    fin[t + 4] = 0x80;
    const uint32_t nbk = (t + 4 + 1 + 8 <= 64) ? 1 : 2;
    const uint64_t bits = (K->raw_len + 4) * 8;
    for (int i = 0; i < 8; ++i) fin[64 * nbk - 1 - i] = (uint8_t)(bits >> (8 * i));
    put_words_be(fin, 32, d.fin);
    d.fin_blocks = nbk;
    d.b_off = t;
  } else {
    uint8_t pw[24] = {0};
    std::memcpy(pw, K->pw, K->pw_len);
    put_words_be(pw, 6, d.pw);
    d.pw_len = K->pw_len;
  }
  return d;
}

lz::DevConst make_const(const KeyImpl* K, uint64_t n, uint64_t b0, uint64_t lanes) {
  lz::DevConst C;
  std::memset(&C, 0, sizeof C);
  C.sigma = K->sigma; C.rho = K->rho; C.beta = K->beta;
  C.h = K->h; C.h2 = K->h2; C.h6 = K->h6;
  C.n = n;
  C.B = block_B(K, n);
  C.b0 = b0;
  C.lanes = lanes;
  C.nb = nblocks(K, n);
  C.n_it = K->prm.n_it;
  C.fast = K->prm.mode == LORENZ_FAST;
  C.variant = K->prm.variant;
  return C;
}

// SM count of the current device, cached per device (148 without a device).
int sm_count() {
  static std::atomic<int> cache[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return 148;
  }
  int n = cache[dev].load(std::memory_order_relaxed);
  if (!n) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;
    }
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// lorenz_set_tuning's overrides (process-wide); launch plans read a snapshot
std::mutex g_tuning_mu;
lorenz_tuning g_tuning = {0, 0, -1, 0};
lorenz_tuning tuning() {
  std::lock_guard<std::mutex> lk(g_tuning_mu);
  return g_tuning;
}

// CTA size for a launch of `lanes` chains (16 resident warps per SM either way). The kernel
// is FP64-pipe bound, so its makespan follows the largest number of warps any SM processes
// over the launch: 4 * ceil(CTAs/SMs) with 128-thread CTAs, 8 * ceil(CTAs/SMs) with 256.
// Take the smaller; on a tie 256 measured 0.3-3 % faster (tools/tune.py, 13 sizes from
// 16 MiB to 1 GiB: the rule picked the faster size at every one).
int chain_cta(uint64_t lanes, uint32_t integrator) {
  if (integrator == LORENZ_RK4_FMA) return 128;  // 5 CTAs/SM of 128 (see min_ctas)
  if (const uint32_t v = tuning().cta) return (int)v;  // lorenz_set_tuning: 128 | 256 | 512
  const uint64_t warps = (lanes + 31) / 32, sms = (uint64_t)sm_count();
  const uint64_t c128 = (warps + 3) / 4, c256 = (warps + 7) / 8;  // CTAs of 4 / 8 warps
  const uint64_t l128 = 4 * ((c128 + sms - 1) / sms), l256 = 8 * ((c256 + sms - 1) / sms);
  return l256 <= l128 ? 256 : 128;
}

template <int OP, int INTEG, int CTA>
cudaError_t launch_chain_cta(const lz::DevConst& C, const lz::DevKey& K, const lz::DevKey* Kb, const uint8_t* in,
                             uint8_t* out, lorenz_result* res, uint8_t* tags, uint8_t* block_ok, cudaStream_t st) {
  const uint64_t grid = (C.lanes + CTA - 1) / CTA;
  lz::lorenz_chain_kernel<OP, INTEG, CTA><<<(unsigned)grid, CTA, 0, st>>>(C, K, Kb, in, out, res, tags, block_ok);
  return cudaGetLastError();
}


// Balanced schedule (lz::lorenz_chain_seg_kernel, lorenz_device.cuh) for chain launches
// with two or more warps of chains per SM sub-partition (exceptions below): one CTA of 128 w
// threads per SM,
// S = SMs x 4 x w warp slots, w = min(4, warps per sub-partition) (tools/tune.py: 2 warps per
// sub-partition already keep the FP64 pipe 97 % busy, 4 reach 98 %). One CTA per SM because
// the warp schedulers favour the older of two co-resident CTAs (tools/seg_trace.py: with
// 2 x 256 threads per SM the second CTA's warps ran at half rate until the first finished, and
// slots cut across the two classes waited), while the warps of one CTA keep within ~3 %.
// Overrides for tests and tuning: lorenz_set_tuning (schedule, slots S clamped to U, skew).
bool seg_plan(const lz::DevConst& C, uint32_t integrator, lz::SegPlan* P, int* cta) {
  if (integrator > LORENZ_RK4_FMA) return false;
  const lorenz_tuning T = tuning();
  if (T.schedule == 1) return false;
  const uint64_t U = (C.lanes + 31) / 32, sms = (uint64_t)sm_count();
  const bool forced = T.schedule == 2;
  uint64_t w = std::min<uint64_t>(4, U / (4 * sms));
  if (!forced) {
    // The wave kernel wins (tools/tune.py) in one wave whose warps split evenly
    // over the SM sub-partitions (2 per sub-partition per 256-thread CTA) and, for Euler and
    // RK4-FMA, from 3 waves of 16 warps per SM on, where the dynamic CTA dispatch balances the
    // SMs. RK4 keeps the balanced kernel at every larger size (1 GiB: 98.05 % against 97.9 %).
    if (w < 2) return false;
    if (integrator == LORENZ_EULER && U > 3 * 16 * sms) return false;
    // RK4-FMA: the wave kernel runs 20 warps per SM (5 x 128 threads, <= 96 registers); with its
    // constants in uniform registers (integrate: no PIN for the FMA form) the balanced kernel
    // reaches 94.1-94.7 % at 12-16 warps and wins below three such waves (64 MiB 94.1 % vs 80.7 %,
    // 128 MiB 94.4 vs 92.5, 256 MiB 94.7 vs 94.0; equal at 512 MiB, 94.7 vs 95.0 at 1 GiB)
    if (integrator == LORENZ_RK4_FMA && U >= 3 * 20 * sms) return false;
    if (U <= 16 * sms) {
      const uint64_t per_smsp_max = 2 * ((((U + 7) / 8) + sms - 1) / sms);
      if (100 * U >= 99 * 4 * sms * per_smsp_max) return false;
    }
  }
  if (w < 2) w = 2;
  uint64_t S = 4 * w * sms;
  if (T.seg_slots) S = T.seg_slots;
  if (S > U) S = U;  // S <= U gives Cq >= Q: a unit spans at most two slots (the kernel relies on it)
  P->units = U;
  P->q = (uint32_t)((C.B + 16 + 15) / 16);
  P->slots = (uint32_t)S;
  P->cq = (U * P->q + S - 1) / S;
  P->wpc = 0;
  P->dq = 0;
  *cta = (int)(128 * w);
  // Skew: within a CTA, warps with a higher index progress faster (tools/seg_trace.py: the four
  // warp groups of a 512-thread CTA finished equal slots at 112.8 / 112.1 / 110.8 / 109.2 ms),
  // so each group of four warps gets `skew` per mille of the mean slot more than the previous
  // one and the slots finish together (tools/tune.py: 8 per mille, 1 GiB 97.95 % -> 98.05 %,
  // 128 MiB 97.45 % -> 97.96 %). Only for the default slot layout (S = SMs x warps per CTA),
  // and only while every slot keeps >= Q/8 chunks of slack over a unit (the two pieces of a
  // cut unit must not meet: with no slack, 1,184 units over 1,184 skewed slots ran at 61 %).
  const uint64_t wpc = 4 * w, G = sms;
  const uint64_t skew = T.seg_skew < 0 ? 8 : (uint64_t)T.seg_skew;
  if (skew && S == G * wpc) {
    const uint64_t UQ = U * P->q, ng = wpc / 4;
    const uint64_t dq = (UQ / S * skew + 500) / 1000;
    const uint64_t extra = G * 2 * dq * ng * (ng - 1);
    if (dq && UQ > extra) {
      const uint64_t cq = (UQ - extra + S - 1) / S;
      if (cq >= P->q + P->q / 8) {
        P->cq = cq;
        P->wpc = (uint32_t)wpc;
        P->dq = (uint32_t)dq;
      }
    }
  }
  return true;
}

template <int OP>
cudaError_t launch_chain(const lz::DevConst& C, const lz::DevKey& K, const lz::DevKey* Kb,
                         uint32_t integrator, const uint8_t* in, uint8_t* out, lorenz_result* res,
                         uint8_t* tags, uint8_t* block_ok, cudaStream_t st) {
  if (C.lanes == 0) return cudaSuccess;
  lz::SegPlan P;
  int scta = 0;
  if (seg_plan(C, integrator, &P, &scta)) {
    const cudaError_t e = lz::launch_seg_op<OP>(C, P, scta, integrator, K, Kb, in, out, res, tags, block_ok, st);
    if (e != cudaErrorNotReady) return e;  // cudaErrorNotReady: scratch allocation failed, fall through
  }
  const int cta = chain_cta(C.lanes, integrator);
  if (integrator == LORENZ_RK4_FMA)
    return launch_chain_cta<OP, LORENZ_RK4_FMA, 128>(C, K, Kb, in, out, res, tags, block_ok, st);
  if (integrator == LORENZ_EULER)
    return cta == 512   ? launch_chain_cta<OP, LORENZ_EULER, 512>(C, K, Kb, in, out, res, tags, block_ok, st)
           : cta == 256 ? launch_chain_cta<OP, LORENZ_EULER, 256>(C, K, Kb, in, out, res, tags, block_ok, st)
                        : launch_chain_cta<OP, LORENZ_EULER, 128>(C, K, Kb, in, out, res, tags, block_ok, st);
  return cta == 512   ? launch_chain_cta<OP, LORENZ_RK4, 512>(C, K, Kb, in, out, res, tags, block_ok, st)
         : cta == 256 ? launch_chain_cta<OP, LORENZ_RK4, 256>(C, K, Kb, in, out, res, tags, block_ok, st)
                      : launch_chain_cta<OP, LORENZ_RK4, 128>(C, K, Kb, in, out, res, tags, block_ok, st);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

bool overlap(const void* a, uint64_t na, const void* b, uint64_t nb) {
  if (!na || !nb) return false;
  const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return x < y + nb && y < x + na;
}

// Shared validation of the device block-range calls.
lorenz_status check_range(const KeyImpl* K, uint64_t n, uint64_t b0, uint64_t b1, const void* in,
                          uint64_t in_bytes, const void* out, uint64_t out_bytes) {
  if (!K) return LORENZ_E_ARG;
  const uint64_t nb = nblocks(K, n);
  if (b0 > b1 || b1 > nb) return LORENZ_E_ARG;
  if (K->prm.mode == LORENZ_FAST && nb > (1ULL << 32)) return LORENZ_E_ARG;  // BE32 block index
  if (in_bytes && (!in || !aligned16(in))) return LORENZ_E_ARG;
  if (out_bytes && (!out || !aligned16(out))) return LORENZ_E_ARG;
  if (overlap(in, in_bytes, out, out_bytes)) return LORENZ_E_ARG;
  return LORENZ_OK;
}

// Buffers the kernels dereference must be device-accessible: device or managed memory, or page-locked
// host memory mapped into the device's address space. Pageable host memory passed where a device
// pointer belongs would fault inside the kernel and kill the context: refuse it (LORENZ_E_ARG) instead.
bool device_accessible(const void* p, uint64_t len) {
  if (!len) return true;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return true;
  return a.type == cudaMemoryTypeHost && a.devicePointer != nullptr;
}

lorenz_status check_device(const void* a, uint64_t na, const void* b, uint64_t nb) {
  if (device_accessible(a, na) && device_accessible(b, nb)) return LORENZ_OK;
  g_err = "buffer not device-accessible (pageable host memory? use the _host calls)";
  return LORENZ_E_ARG;
}

lorenz_status finish_sync(lorenz_result* d_res, cudaStream_t st, lorenz_result* h_res) {
  if (!cuda_ok(cudaMemcpyAsync(h_res, d_res, sizeof *h_res, cudaMemcpyDeviceToHost, st), "readback"))
    return LORENZ_E_CUDA;
  if (!cuda_ok(cudaFreeAsync(d_res, st), "cudaFreeAsync")) return LORENZ_E_CUDA;
  if (!cuda_ok(cudaStreamSynchronize(st), "cudaStreamSynchronize")) return LORENZ_E_CUDA;
  if (h_res->status & lz::ST_DIVERGENCE) return LORENZ_E_DIVERGENCE;
  if (h_res->status & lz::ST_INTEGRITY) return LORENZ_E_INTEGRITY;
  return LORENZ_OK;
}

lorenz_status alloc_result(lorenz_result** d_res, cudaStream_t st) {
  if (!cuda_ok(lz::lib_malloc_async(reinterpret_cast<void**>(d_res), sizeof(lorenz_result), st), "cudaMallocAsync"))
    return LORENZ_E_CUDA;
  lz::result_init_kernel<<<1, 32, 0, st>>>(*d_res);
  return cuda_ok(cudaGetLastError(), "result_init") ? LORENZ_OK : LORENZ_E_CUDA;
}

}  // namespace

namespace lz {
void set_last_error(const std::string& s) { g_err = s; }  // shared with lorenz_io.cu, lorenz_spectra.cu
int device_sm_count() { return sm_count(); }             // shared with lorenz_spectra.cu

// The library's own stream-ordered pool, one per device, created on first use. Per-call scratch
// (result slots, key arrays, hand-over state, FFT workspaces, staged host-path buffers) comes
// from it; its release threshold keeps up to kPoolKeep bytes mapped across synchronisations so
// repeated calls do not remap pages, and everything above that goes back to the driver at the
// next synchronisation. The device's default pool and its policy are left alone.
constexpr uint64_t kPoolKeep = 256ull << 20;
cudaError_t lib_malloc_async(void** p, size_t bytes, cudaStream_t st) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  static bool tried[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, st);
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!tried[dev]) {
      tried[dev] = true;
      cudaMemPoolProps props;
      std::memset(&props, 0, sizeof props);
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      if (cudaMemPoolCreate(&pools[dev], &props) == cudaSuccess) {
        uint64_t keep = kPoolKeep;
        cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
      } else {  // no pool of our own (e.g. a device without stream-ordered pools): the default one
        cudaGetLastError();
        pools[dev] = nullptr;
      }
    }
    pool = pools[dev];
  }
  return pool ? cudaMallocFromPoolAsync(p, bytes, pool, st) : cudaMallocAsync(p, bytes, st);
}
}  // namespace lz

// ======================================================================== C ABI
extern "C" {


int lorenz_abi_version(void) { return LORENZ_ABI_VERSION; }

const char* lorenz_last_error(void) { return g_err.c_str(); }

const char* lorenz_status_string(lorenz_status s) {
  switch (s) {
    case LORENZ_OK: return "ok";
    case LORENZ_E_INTEGRITY: return "integrity check failed (a block's sentinel did not decrypt)";
    case LORENZ_E_ARG: return "invalid argument";
    case LORENZ_E_PASSWORD: return "password shorter than 3 bytes";
    case LORENZ_E_LENGTH: return "ciphertext length inconsistent with the block size";
    case LORENZ_E_DIVERGENCE: return "trajectory left the guard box";
    case LORENZ_E_CUDA: return "CUDA runtime error";
    case LORENZ_E_IO: return "file I/O error";
    case LORENZ_E_FORMAT: return "malformed envelope header";
  }
  return "unknown status";
}

lorenz_status lorenz_keysetup(const uint8_t* pw, size_t pw_len, const lorenz_params* p, lorenz_key* out) {
  if (!out || (!pw && pw_len)) return LORENZ_E_ARG;
  lorenz_params prm = p ? *p : lorenz_params{LORENZ_FAST, 0, 0, 0, LORENZ_RK4, 0};
  if (prm.mode > 1 || prm.dt_code > 3 || prm.integrator > 2) return LORENZ_E_ARG;
  if (prm.variant > 7 || (prm.variant & 3) == 3) return LORENZ_E_ARG;
  if (prm.n_it == 0) prm.n_it = prm.mode == LORENZ_FAST ? 100u : 3000u;
  if (prm.mode == LORENZ_FAST) {
    if (prm.block_size == 0) prm.block_size = 1024;
    if (prm.block_size < 1024 || prm.block_size % 16) return LORENZ_E_ARG;
  } else {
    prm.block_size = 0;
  }
  if (pw_len < 3) return LORENZ_E_PASSWORD;
  std::memset(out->opaque, 0, sizeof out->opaque);
  KeyImpl* K = reinterpret_cast<KeyImpl*>(out->opaque);
  K->magic = kMagic;
  K->abi = LORENZ_ABI_VERSION;
  K->prm = prm;
  volatile double three = 3.0, six = 6.0;  // computed at run time, RN, like the oracle
  K->sigma = 10.0;
  K->rho = 28.0;
  K->beta = 8.0 / three;
  K->h = dt_of(prm.dt_code);
  K->h2 = K->h * 0.5;
  K->h6 = K->h / six;
  if (prm.mode == LORENZ_STRONG) {
    if (pw_len > 23) {  // longer passwords are replaced by SHA-256(pw)[0:18]
      uint8_t d[32];
      lz::sha256_host(pw, pw_len, d);
      std::memcpy(K->pw, d, 18);
      K->pw_len = 18;
    } else {
      std::memcpy(K->pw, pw, pw_len);
      K->pw_len = (uint32_t)pw_len;
    }
  } else {
    lz::Sha256State s;
    s.init();
    uint64_t off = 0;
    uint32_t w[16];
    for (; off + 64 <= pw_len; off += 64) {
      put_words_be(pw + off, 16, w);
      s.compress(w);
    }
    for (int i = 0; i < 8; ++i) K->mid[i] = s.h[i];
    K->raw_len = pw_len;
    K->tail_len = (uint32_t)(pw_len - off);
    std::memcpy(K->tail, pw + off, K->tail_len);
  }
  return LORENZ_OK;
}

lorenz_status lorenz_set_tuning(const lorenz_tuning* t) {
  lorenz_tuning v = {0, 0, -1, 0};
  if (t) {
    if (t->schedule > 2 || t->seg_skew < -1 || t->seg_skew > 1000 ||
        (t->cta && t->cta != 128 && t->cta != 256 && t->cta != 512))
      return LORENZ_E_ARG;
    v = *t;
  }
  std::lock_guard<std::mutex> lk(g_tuning_mu);
  g_tuning = v;
  return LORENZ_OK;
}

lorenz_status lorenz_key_params(const lorenz_key* k, lorenz_params* out) {
  const KeyImpl* K = impl(k);
  if (!K || !out) return LORENZ_E_ARG;
  *out = K->prm;
  return LORENZ_OK;
}

lorenz_status lorenz_launch_plan(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1, lorenz_plan* out) {
  const KeyImpl* K = impl(k);
  if (!K || !out || b0 > b1 || b1 > nblocks(K, n)) return LORENZ_E_ARG;
  std::memset(out, 0, sizeof *out);
  const lz::DevConst C = make_const(K, n, b0, b1 - b0);
  out->lanes = C.lanes;
  if (C.lanes == 0) return LORENZ_OK;
  lz::SegPlan P;
  int cta = 0;
  if (seg_plan(C, K->prm.integrator, &P, &cta)) {
    out->kind = 1;
    out->cta = (uint32_t)cta;
    out->grid = (P.slots + cta / 32 - 1) / (cta / 32);
    out->slots = P.slots;
    out->chunks_per_slot = P.cq;
    out->chunks_skew = P.dq;
  } else {
    out->cta = (uint32_t)chain_cta(C.lanes, K->prm.integrator);
    out->grid = (C.lanes + out->cta - 1) / out->cta;
  }
  return LORENZ_OK;
}

uint64_t lorenz_num_blocks(const lorenz_key* k, uint64_t n) {
  const KeyImpl* K = impl(k);
  return K ? nblocks(K, n) : 0;
}

uint64_t lorenz_ct_len(const lorenz_key* k, uint64_t n) {
  const KeyImpl* K = impl(k);
  return K ? n + 16 * nblocks(K, n) : 0;
}

lorenz_status lorenz_pt_len(const lorenz_key* k, uint64_t ct_len, uint64_t* n_out) {
  const KeyImpl* K = impl(k);
  if (!K || !n_out) return LORENZ_E_ARG;
  if (ct_len < 16) return LORENZ_E_LENGTH;
  if (K->prm.mode == LORENZ_STRONG) { *n_out = ct_len - 16; return LORENZ_OK; }
  const uint64_t per = (uint64_t)K->prm.block_size + 16;
  const uint64_t nb = (ct_len + per - 1) / per;
  if (ct_len < 16 * nb) return LORENZ_E_LENGTH;
  const uint64_t n = ct_len - 16 * nb;
  if (nblocks(K, n) != nb) return LORENZ_E_LENGTH;
  *n_out = n;
  return LORENZ_OK;
}

lorenz_status lorenz_result_init_async(lorenz_result* res, void* stream) {
  if (!res || !aligned16(res)) return LORENZ_E_ARG;
  lz::result_init_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(res);
  return cuda_ok(cudaGetLastError(), "result_init") ? LORENZ_OK : LORENZ_E_CUDA;
}

lorenz_status lorenz_encrypt_async(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1,
                                   const uint8_t* pt, uint8_t* ct, lorenz_result* res, void* stream) {
  Trace tr("lorenz_encrypt");
  const KeyImpl* K = impl(k);
  if (!K || !res || !aligned16(res)) return LORENZ_E_ARG;  // 64-bit atomics on res
  uint64_t ptb = 0, ctb = 0;
  if (b0 < b1) slice_bytes(K, n, b0, b1, &ptb, &ctb);
  lorenz_status s = check_range(K, n, b0, b1, pt, ptb, ct, ctb);
  if (s != LORENZ_OK || b0 == b1) return s;
  if ((s = check_device(pt, ptb, ct, ctb)) != LORENZ_OK) return s;
  const lz::DevConst C = make_const(K, n, b0, b1 - b0);
  const lz::DevKey D = make_devkey(K);
  return cuda_ok(launch_chain<lz::OP_ENC>(C, D, nullptr, K->prm.integrator, pt, ct, res, nullptr, nullptr,
                                          (cudaStream_t)stream), "encrypt launch")
             ? LORENZ_OK : LORENZ_E_CUDA;
}

lorenz_status lorenz_decrypt_async(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1,
                                   const uint8_t* ct, uint8_t* pt, uint8_t* block_ok, lorenz_result* res,
                                   void* stream) {
  Trace tr("lorenz_decrypt");
  const KeyImpl* K = impl(k);
  if (!K || !res || !aligned16(res)) return LORENZ_E_ARG;  // 64-bit atomics on res
  uint64_t ptb = 0, ctb = 0;
  if (b0 < b1) slice_bytes(K, n, b0, b1, &ptb, &ctb);
  lorenz_status s = check_range(K, n, b0, b1, ct, ctb, pt, ptb);
  if (s != LORENZ_OK || b0 == b1) return s;
  if ((s = check_device(ct, ctb, pt, ptb)) != LORENZ_OK) return s;
  const lz::DevConst C = make_const(K, n, b0, b1 - b0);
  const lz::DevKey D = make_devkey(K);
  cudaStream_t st = (cudaStream_t)stream;
  if (!cuda_ok(launch_chain<lz::OP_DEC>(C, D, nullptr, K->prm.integrator, ct, pt, res, nullptr, block_ok, st),
               "decrypt launch"))
    return LORENZ_E_CUDA;
  if (!block_ok && ptb) {
    lz::zero_if_failed_kernel<<<256, 256, 0, st>>>(res, pt, ptb);
    if (!cuda_ok(cudaGetLastError(), "zero_if_failed")) return LORENZ_E_CUDA;
  }
  return LORENZ_OK;
}

lorenz_status lorenz_verify_async(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1, const uint8_t* ct,
                                  lorenz_result* res, void* stream) {
  Trace tr("lorenz_verify");
  const KeyImpl* K = impl(k);
  if (!K || !res || !aligned16(res)) return LORENZ_E_ARG;  // 64-bit atomics on res
  uint64_t ptb = 0, ctb = 0;
  if (b0 < b1) slice_bytes(K, n, b0, b1, &ptb, &ctb);
  lorenz_status s = check_range(K, n, b0, b1, ct, ctb, nullptr, 0);
  if (s != LORENZ_OK || b0 == b1) return s;
  if ((s = check_device(ct, ctb, nullptr, 0)) != LORENZ_OK) return s;
  const lz::DevConst C = make_const(K, n, b0, b1 - b0);
  const lz::DevKey D = make_devkey(K);
  return cuda_ok(launch_chain<lz::OP_VERIFY>(C, D, nullptr, K->prm.integrator, ct, nullptr, res, nullptr,
                                             nullptr, (cudaStream_t)stream), "verify launch")
             ? LORENZ_OK : LORENZ_E_CUDA;
}

lorenz_status lorenz_encrypt(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1, const uint8_t* pt,
                             uint8_t* ct, uint8_t tag_xor[16], void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const KeyImpl* K = impl(k);
  if (!K) return LORENZ_E_ARG;
  if (tag_xor) std::memset(tag_xor, 0, 16);
  uint64_t ptb = 0, ctb = 0;
  if (b0 < b1) slice_bytes(K, n, b0, b1, &ptb, &ctb);
  lorenz_status s = check_range(K, n, b0, b1, pt, ptb, ct, ctb);
  if (s != LORENZ_OK || b0 == b1) return s;
  lorenz_result* d_res = nullptr;
  if ((s = alloc_result(&d_res, st)) != LORENZ_OK) return s;
  s = lorenz_encrypt_async(k, n, b0, b1, pt, ct, d_res, stream);
  lorenz_result h;
  lorenz_status f = finish_sync(d_res, st, &h);
  if (s != LORENZ_OK) return s;
  if (f == LORENZ_OK && tag_xor) std::memcpy(tag_xor, h.tag_xor, 16);
  return f;
}

lorenz_status lorenz_decrypt(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1, const uint8_t* ct,
                             uint8_t* pt, int64_t* first_bad_block, uint8_t* block_ok, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const KeyImpl* K = impl(k);
  if (!K) return LORENZ_E_ARG;
  if (first_bad_block) *first_bad_block = -1;
  uint64_t ptb = 0, ctb = 0;
  if (b0 < b1) slice_bytes(K, n, b0, b1, &ptb, &ctb);
  lorenz_status s = check_range(K, n, b0, b1, ct, ctb, pt, ptb);
  if (s != LORENZ_OK || b0 == b1) return s;
  lorenz_result* d_res = nullptr;
  if ((s = alloc_result(&d_res, st)) != LORENZ_OK) return s;
  s = lorenz_decrypt_async(k, n, b0, b1, ct, pt, block_ok, d_res, stream);
  lorenz_result h;
  lorenz_status f = finish_sync(d_res, st, &h);
  if (s != LORENZ_OK) return s;
  if (first_bad_block && h.first_bad != ~0ULL) *first_bad_block = (int64_t)h.first_bad;
  return f;
}

lorenz_status lorenz_verify(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1, const uint8_t* ct,
                            int64_t* first_bad_block, uint8_t tag_xor[16], void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const KeyImpl* K = impl(k);
  if (!K) return LORENZ_E_ARG;
  if (first_bad_block) *first_bad_block = -1;
  if (tag_xor) std::memset(tag_xor, 0, 16);
  uint64_t ptb = 0, ctb = 0;
  if (b0 < b1) slice_bytes(K, n, b0, b1, &ptb, &ctb);
  lorenz_status s = check_range(K, n, b0, b1, ct, ctb, nullptr, 0);
  if (s != LORENZ_OK || b0 == b1) return s;
  lorenz_result* d_res = nullptr;
  if ((s = alloc_result(&d_res, st)) != LORENZ_OK) return s;
  s = lorenz_verify_async(k, n, b0, b1, ct, d_res, stream);
  lorenz_result h;
  lorenz_status f = finish_sync(d_res, st, &h);
  if (s != LORENZ_OK) return s;
  if (first_bad_block && h.first_bad != ~0ULL) *first_bad_block = (int64_t)h.first_bad;
  if (tag_xor && f != LORENZ_E_CUDA) std::memcpy(tag_xor, h.tag_xor, 16);
  return f;
}

lorenz_status lorenz_encrypt_batch(const lorenz_key* keys, uint32_t S, uint64_t n, const uint8_t* pts,
                                   uint8_t* cts, uint8_t* tags, void* stream) {
  Trace tr("lorenz_encrypt_batch");
  if (!keys || S == 0) return LORENZ_E_ARG;
  const KeyImpl* K0 = impl(&keys[0]);
  if (!K0) return LORENZ_E_ARG;
  for (uint32_t s = 1; s < S; ++s) {
    const KeyImpl* Ks = impl(&keys[s]);
    if (!Ks || std::memcmp(&Ks->prm, &K0->prm, sizeof K0->prm) != 0) return LORENZ_E_ARG;
  }
  const uint64_t nb = nblocks(K0, n), ctl = n + 16 * nb;
  if (K0->prm.mode == LORENZ_FAST && nb > (1ULL << 32)) return LORENZ_E_ARG;
  if ((n && (!pts || !aligned16(pts) || n % 16)) || !cts || !aligned16(cts) || !tags || !aligned16(tags))
    return LORENZ_E_ARG;
  if (overlap(pts, n * S, cts, ctl * S)) return LORENZ_E_ARG;
  if (check_device(pts, n * S, cts, ctl * S) != LORENZ_OK || check_device(tags, 16ull * S, nullptr, 0) != LORENZ_OK)
    return LORENZ_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  lz::DevKey* d_keys = nullptr;
  std::vector<lz::DevKey> h_keys(S);  // pageable: the H2D below is staged before it returns
  for (uint32_t s = 0; s < S; ++s) h_keys[s] = make_devkey(impl(&keys[s]));
  lorenz_status ret = LORENZ_OK;
  lorenz_result* d_res = nullptr;
  do {
    if (!cuda_ok(lz::lib_malloc_async(reinterpret_cast<void**>(&d_keys), sizeof(lz::DevKey) * S, st), "alloc keys")) {
      ret = LORENZ_E_CUDA; break;
    }
    if (!cuda_ok(cudaMemcpyAsync(d_keys, h_keys.data(), sizeof(lz::DevKey) * S, cudaMemcpyHostToDevice, st),
                 "keys H2D") ||
        !cuda_ok(cudaMemsetAsync(tags, 0, 16ull * S, st), "tags memset")) {
      ret = LORENZ_E_CUDA; break;
    }
    if ((ret = alloc_result(&d_res, st)) != LORENZ_OK) break;
    lz::DevConst C = make_const(K0, n, 0, nb * S);
    C.batch = 1;
    C.in_msg_stride = n;
    C.out_msg_stride = ctl;
    lz::DevKey dummy;
    std::memset(&dummy, 0, sizeof dummy);
    if (!cuda_ok(launch_chain<lz::OP_ENC>(C, dummy, d_keys, K0->prm.integrator, pts, cts, d_res, tags, nullptr, st),
                 "batch launch")) {
      ret = LORENZ_E_CUDA; break;
    }
  } while (0);
  if (d_keys) cudaFreeAsync(d_keys, st);
  if (d_res) {
    lorenz_result h;
    lorenz_status f = finish_sync(d_res, st, &h);
    if (ret == LORENZ_OK) ret = f;
  } else {
    cudaStreamSynchronize(st);
  }
  return ret;
}

// ---------------------------------------------------------------- ragged batches (serving)
}  // extern "C"
namespace {
// count messages of different lengths, one launch over all their blocks (DevConst.batch = 2)
lorenz_status ragged(const lorenz_key* keys, uint32_t count, const uint64_t* n, const uint64_t* in_off,
                     const uint64_t* out_off, const uint8_t* in, uint8_t* out, uint8_t* tags, int64_t* first_bad,
                     bool decrypt, cudaStream_t st) {
  if (!keys || count == 0 || count > (1u << 30) || !n || !in_off || !out_off || !in || !out || !tags ||
      !aligned16(in) || !aligned16(out) || !aligned16(tags) || (decrypt && !first_bad))
    return LORENZ_E_ARG;
  const KeyImpl* K0 = impl(&keys[0]);
  if (!K0 || K0->prm.mode != LORENZ_FAST) return LORENZ_E_ARG;
  for (uint32_t s = 1; s < count; ++s) {
    const KeyImpl* Ks = impl(&keys[s]);
    if (!Ks || std::memcmp(&Ks->prm, &K0->prm, sizeof K0->prm) != 0) return LORENZ_E_ARG;
  }
  // host tables: block prefix sums, lengths, offsets; per-message extents for the overlap checks
  std::vector<uint64_t> tab(4ull * count + 1);
  uint64_t* blk = tab.data();
  uint64_t *len = blk + count + 1, *ioff = len + count, *ooff = ioff + count;
  std::vector<std::pair<uint64_t, uint64_t>> outs(count);
  uint64_t in_end = 0, out_end = 0;
  blk[0] = 0;
  for (uint32_t s = 0; s < count; ++s) {
    const uint64_t nb = nblocks(K0, n[s]), ctl = n[s] + 16 * nb;
    if ((in_off[s] | out_off[s]) & 15) return LORENZ_E_ARG;  // 16-byte aligned message starts
    const uint64_t ib = decrypt ? ctl : n[s], ob = decrypt ? n[s] : ctl;
    blk[s + 1] = blk[s] + nb;
    len[s] = n[s];
    ioff[s] = in_off[s];
    ooff[s] = out_off[s];
    in_end = std::max(in_end, in_off[s] + ib);
    out_end = std::max(out_end, out_off[s] + ob);
    outs[s] = {out_off[s], out_off[s] + ob};
  }
  // non-empty output ranges must be disjoint: sorted by start, each starts at or after the
  // furthest end so far (an empty range in between must not hide an overlap)
  outs.erase(std::remove_if(outs.begin(), outs.end(), [](const std::pair<uint64_t, uint64_t>& r) {
               return r.second <= r.first;
             }), outs.end());
  std::sort(outs.begin(), outs.end());
  uint64_t max_end = 0;
  for (size_t s = 0; s < outs.size(); ++s) {
    if (s && outs[s].first < max_end) {
      g_err = "ragged batch: output ranges overlap";
      return LORENZ_E_ARG;
    }
    max_end = std::max(max_end, outs[s].second);
  }
  if (overlap(in, in_end, out, out_end)) return LORENZ_E_ARG;
  const uint64_t lanes = blk[count];
  std::vector<lz::DevKey> h_keys(count);
  for (uint32_t s = 0; s < count; ++s) h_keys[s] = make_devkey(impl(&keys[s]));
  lz::DevKey* d_keys = nullptr;
  uint64_t* d_tab = nullptr;  // blk | len | in | out | bad
  lorenz_result* d_res = nullptr;
  lorenz_status ret = LORENZ_OK;
  std::vector<uint64_t> bad(count, ~0ULL);
  do {
    if (!cuda_ok(lz::lib_malloc_async(reinterpret_cast<void**>(&d_keys), sizeof(lz::DevKey) * count, st), "alloc") ||
        !cuda_ok(lz::lib_malloc_async(reinterpret_cast<void**>(&d_tab), 8 * (5ull * count + 1), st), "alloc")) {
      ret = LORENZ_E_CUDA; break;
    }
    if (!cuda_ok(cudaMemcpyAsync(d_keys, h_keys.data(), sizeof(lz::DevKey) * count, cudaMemcpyHostToDevice, st),
                 "keys H2D") ||
        !cuda_ok(cudaMemcpyAsync(d_tab, tab.data(), 8 * tab.size(), cudaMemcpyHostToDevice, st), "tables H2D") ||
        !cuda_ok(cudaMemsetAsync(d_tab + tab.size(), 0xFF, 8ull * count, st), "verdicts") ||
        !cuda_ok(cudaMemsetAsync(tags, 0, 16ull * count, st), "tags memset")) {
      ret = LORENZ_E_CUDA; break;
    }
    if ((ret = alloc_result(&d_res, st)) != LORENZ_OK) break;
    lz::DevConst C = make_const(K0, 0, 0, lanes);
    C.batch = 2;
    C.count = count;
    C.rag_blk = d_tab;
    C.rag_len = d_tab + count + 1;
    C.rag_in = d_tab + 2ull * count + 1;
    C.rag_out = d_tab + 3ull * count + 1;
    C.rag_bad = reinterpret_cast<unsigned long long*>(d_tab + 4ull * count + 1);
    lz::DevKey dummy;
    std::memset(&dummy, 0, sizeof dummy);
    const cudaError_t e =
        decrypt ? launch_chain<lz::OP_DEC>(C, dummy, d_keys, K0->prm.integrator, in, out, d_res, tags, nullptr, st)
                : launch_chain<lz::OP_ENC>(C, dummy, d_keys, K0->prm.integrator, in, out, d_res, tags, nullptr, st);
    if (!cuda_ok(e, "ragged launch")) { ret = LORENZ_E_CUDA; break; }
    if (decrypt &&
        !cuda_ok(cudaMemcpyAsync(bad.data(), C.rag_bad, 8ull * count, cudaMemcpyDeviceToHost, st), "verdicts D2H")) {
      ret = LORENZ_E_CUDA; break;
    }
  } while (0);
  if (d_keys) cudaFreeAsync(d_keys, st);
  if (d_tab) cudaFreeAsync(d_tab, st);
  if (d_res) {
    lorenz_result h;
    lorenz_status f = finish_sync(d_res, st, &h);  // synchronises the stream (verdicts are on the host)
    if (ret == LORENZ_OK || (ret == LORENZ_E_INTEGRITY && f != LORENZ_E_INTEGRITY)) ret = f;
  } else {
    cudaStreamSynchronize(st);
  }
  if (decrypt && (ret == LORENZ_OK || ret == LORENZ_E_INTEGRITY)) {
    bool any = false;
    for (uint32_t s = 0; s < count; ++s) {
      first_bad[s] = bad[s] == ~0ULL ? -1 : (int64_t)bad[s];
      if (bad[s] != ~0ULL && n[s]) {  // never release a failing message's plaintext
        any = true;
        if (!cuda_ok(cudaMemsetAsync(out + out_off[s], 0, n[s], st), "zero")) ret = LORENZ_E_CUDA;
      }
    }
    if (any) {
      cudaStreamSynchronize(st);
      if (ret == LORENZ_OK) ret = LORENZ_E_INTEGRITY;
    }
  }
  return ret;
}
}  // namespace
extern "C" {

lorenz_status lorenz_encrypt_ragged(const lorenz_key* keys, uint32_t count, const uint64_t* n, const uint64_t* pt_off,
                                    const uint64_t* ct_off, const uint8_t* pts, uint8_t* cts, uint8_t* tags,
                                    void* stream) {
  Trace tr("lorenz_encrypt_ragged");
  return ragged(keys, count, n, pt_off, ct_off, pts, cts, tags, nullptr, false, (cudaStream_t)stream);
}

lorenz_status lorenz_decrypt_ragged(const lorenz_key* keys, uint32_t count, const uint64_t* n, const uint64_t* ct_off,
                                    const uint64_t* pt_off, const uint8_t* cts, uint8_t* pts, uint8_t* tags,
                                    int64_t* first_bad, void* stream) {
  Trace tr("lorenz_decrypt_ragged");
  return ragged(keys, count, n, ct_off, pt_off, cts, pts, tags, first_bad, true, (cudaStream_t)stream);
}

// ---------------------------------------------------------------- NEXT-4 analysis (Fig.1)
lorenz_status lorenz_digit_histograms(const double* ic, uint64_t lanes, uint32_t skip, uint32_t samples,
                                      uint32_t stride, uint32_t dt_code, uint32_t integrator, uint64_t* hist,
                                      void* stream) {
  Trace tr("lorenz_digit_histograms");
  if (!hist || (lanes && !ic) || dt_code > 3 || integrator > 2 || lanes > (1ULL << 40)) return LORENZ_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (!cuda_ok(cudaMemsetAsync(hist, 0, sizeof(uint64_t) * lz::kHistBins, st), "memset")) return LORENZ_E_CUDA;
  if (lanes == 0) return LORENZ_OK;
  lorenz_key k;  // the constants exactly as a key holds them
  lorenz_params p{LORENZ_FAST, 1, dt_code, 0, integrator, 0};
  const uint8_t dummy[3] = {'a', 'b', 'c'};
  lorenz_status s = lorenz_keysetup(dummy, 3, &p, &k);
  if (s != LORENZ_OK) return s;
  const lz::DevConst C = make_const(impl(&k), 0, 0, lanes);
  const unsigned grid = (unsigned)((lanes + lz::kCta - 1) / lz::kCta);
  auto* h = reinterpret_cast<unsigned long long*>(hist);
  if (integrator == LORENZ_EULER)
    lz::digit_hist_kernel<LORENZ_EULER><<<grid, lz::kCta, 0, st>>>(C, ic, lanes, skip, samples, stride, h);
  else if (integrator == LORENZ_RK4_FMA)
    lz::digit_hist_kernel<LORENZ_RK4_FMA><<<grid, lz::kCta, 0, st>>>(C, ic, lanes, skip, samples, stride, h);
  else
    lz::digit_hist_kernel<LORENZ_RK4><<<grid, lz::kCta, 0, st>>>(C, ic, lanes, skip, samples, stride, h);
  return cuda_ok(cudaGetLastError(), "digit_hist") ? LORENZ_OK : LORENZ_E_CUDA;
}

// ---------------------------------------------------------------- C5 statistics
}  // extern "C"
namespace {
// spans: HOST array; copied to a stream-ordered device buffer. grid.x covers the longest span.
template <typename Launch>
lorenz_status span_launch(const lorenz_span* spans, uint32_t count, uint64_t* out, uint64_t out_words,
                          cudaStream_t st, Launch launch) {
  if (!cuda_ok(cudaMemsetAsync(out, 0, sizeof(uint64_t) * out_words, st), "memset")) return LORENZ_E_CUDA;
  uint64_t mx = 0;
  for (uint32_t i = 0; i < count; ++i) mx = spans[i].len > mx ? spans[i].len : mx;
  const uint64_t tiles = (mx + lz::kStatTile - 1) / lz::kStatTile;
  if (!tiles) return LORENZ_OK;
  lorenz_span* d = nullptr;
  if (!cuda_ok(lz::lib_malloc_async(reinterpret_cast<void**>(&d), sizeof(lorenz_span) * count, st), "alloc spans"))
    return LORENZ_E_CUDA;
  lorenz_status ret = LORENZ_OK;
  if (!cuda_ok(cudaMemcpyAsync(d, spans, sizeof(lorenz_span) * count, cudaMemcpyHostToDevice, st), "spans H2D"))
    ret = LORENZ_E_CUDA;
  if (ret == LORENZ_OK) {
    launch(dim3((unsigned)tiles, count), d);
    if (!cuda_ok(cudaGetLastError(), "stats kernel")) ret = LORENZ_E_CUDA;
  }
  cudaFreeAsync(d, st);
  return ret;
}
}  // namespace
extern "C" {

lorenz_status lorenz_compare_spans(const uint8_t* a, const uint8_t* b, const lorenz_span* spans, uint32_t count,
                                   uint64_t* out, void* stream) {
  if (!a || !b || !spans || !out || count == 0 || count > 65535) return LORENZ_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  return span_launch(spans, count, out, 3ull * count, st, [&](dim3 g, const lorenz_span* d) {
    lz::compare_spans_kernel<<<g, lz::kStatCta, 0, st>>>(a, b, d, out);
  });
}

lorenz_status lorenz_histograms(const uint8_t* a, const lorenz_span* spans, uint32_t count, uint64_t* hist,
                                void* stream) {
  if (!a || !spans || !hist || count == 0 || count > 65535) return LORENZ_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  return span_launch(spans, count, hist, 256ull * count, st, [&](dim3 g, const lorenz_span* d) {
    lz::histogram_kernel<<<g, lz::kStatCta, 0, st>>>(a, d, hist);
  });
}

// ---------------------------------------------------------------- host-buffer end to end
namespace {
struct HostPipe {
  // one stream per chunk (up to 8): chunk c's H2D, kernel and D2H are stream-ordered; events
  // chain the H2Ds and the kernels across streams in chunk order, so copies overlap kernels
  static constexpr int kStreams = 8;
  cudaStream_t st[kStreams] = {};
  cudaEvent_t ev[kStreams] = {};
  cudaEvent_t cp[kStreams] = {};  // "chunk c's H2D done": chains the H2Ds in chunk order
  cudaEvent_t kd[kStreams] = {};  // "chunk c's kernel done": chains the kernels in chunk order
  int n = 0;                      // streams in use by the current call (one per ring slot)
  bool ready = false;
  // The streams and events are created once per host thread and device (host_pipe below):
  // creating eight streams per call cost ~0.6 ms, 2 % of a 64 MiB call.
  bool init() {
    for (int i = 0; i < kStreams; ++i) {
      if (!cuda_ok(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking), "stream create")) return false;
      if (!cuda_ok(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "event create")) return false;
      if (!cuda_ok(cudaEventCreateWithFlags(&cp[i], cudaEventDisableTiming), "event create")) return false;
      if (!cuda_ok(cudaEventCreateWithFlags(&kd[i], cudaEventDisableTiming), "event create")) return false;
    }
    ready = true;
    return true;
  }
  void use(int slots) { n = slots < 1 ? 1 : (slots > kStreams ? kStreams : slots); }
  // all streams wait for stream 0's work so far
  void fan_out() {
    cudaEventRecord(ev[0], st[0]);
    for (int i = 1; i < n; ++i) cudaStreamWaitEvent(st[i], ev[0], 0);
  }
  // stream 0 waits for every stream
  void fan_in() {
    for (int i = 1; i < n; ++i) {
      cudaEventRecord(ev[i], st[i]);
      cudaStreamWaitEvent(st[0], ev[i], 0);
    }
  }
  ~HostPipe() {
    for (int i = 0; i < kStreams; ++i) {
      if (st[i]) cudaStreamDestroy(st[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
      if (cp[i]) cudaEventDestroy(cp[i]);
      if (kd[i]) cudaEventDestroy(kd[i]);
    }
  }
};

// This host thread's pipe for the current device (nullptr if its streams cannot be created).
HostPipe* host_pipe() {
  static thread_local HostPipe pipes[16];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
  HostPipe& P = pipes[dev];
  if (!P.ready && !P.init()) return nullptr;
  return &P;
}

constexpr uint64_t kHostChunk = 128ull << 20;  // upper bound of an automatic host-path chunk

// The device address of host bytes [p, p + len) if they are page-locked memory mapped into the
// current device's address space as one contiguous range, else nullptr (pageable memory, or
// another device's non-portable allocation).
const uint8_t* device_alias(const void* p, uint64_t len) {
  if (!p || !len) return nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  auto alias = [dev](const void* q) -> const uint8_t* {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, q) != cudaSuccess) {
      cudaGetLastError();  // pageable memory on older drivers: not an error of the call
      return nullptr;
    }
    if (a.type != cudaMemoryTypeHost || !a.devicePointer || a.device != dev) return nullptr;
    return static_cast<const uint8_t*>(a.devicePointer);
  };
  const uint8_t* d0 = alias(p);
  const uint8_t* d1 = alias(static_cast<const uint8_t*>(p) + (len - 1));
  return (d0 && d1 && d1 - d0 == (ptrdiff_t)(len - 1)) ? d0 : nullptr;
}

}  // namespace

// Blocks [B0,B1) from host slices: chunked H2D -> kernel -> D2H over HostPipe's streams.
// The slice is cut into block-aligned chunks (plan below); chunk c runs on slot c % S
// (S = min(8, chunks)), each slot owning a stream and device buffers sized for one chunk. Chunk c + S reuses the slot's buffers only
// after chunk c's D2H (same stream), so the host never waits and device memory stays bounded
// (≈ 8 x 2 x 128 MiB) whatever the message size: messages larger than HBM work.
static lorenz_status host_range(const lorenz_key* k, uint64_t n, uint64_t B0, uint64_t B1, const uint8_t* in_host,
                                uint8_t* out_host, bool decrypt, lorenz_result* h_res, uint32_t n_chunks) {
  Trace tr(decrypt ? "lorenz_decrypt_host" : "lorenz_encrypt_host");
  const KeyImpl* K = impl(k);
  if (!K) return LORENZ_E_ARG;
  uint64_t ptb = 0, ctb = 0;
  if (B0 < B1) slice_bytes(K, n, B0, B1, &ptb, &ctb);
  const uint64_t inb = decrypt ? ctb : ptb, outb = decrypt ? ptb : ctb;
  lorenz_status ret = check_range(K, n, B0, B1, in_host, inb, out_host, outb);
  if (ret != LORENZ_OK || B0 == B1) return ret;
  // Direct streaming (automatic mode): when both host slices are page-locked and mapped into
  // this device's address space (cudaHostAlloc, torch pin_memory, cudaHostRegister with
  // cudaHostRegisterMapped), ONE chain launch reads its input and writes its output over PCIe
  // itself. The kernel consumes its input at the FP64 rate (~2.4 GB/s per GPU at n_it = 100,
  // a few % of the link) and every block's characters are spread over the whole launch, so the
  // transfers hide under the arithmetic from the first window to the last — no copy is left
  // outside the kernel, whatever the slice size (the staged pipeline below always exposes its
  // first H2D and last D2H).
  if (n_chunks == 0) {
    const uint8_t* din = device_alias(in_host, inb);
    uint8_t* dout = const_cast<uint8_t*>(device_alias(out_host, outb));
    if (din && dout) {
      HostPipe* PP = host_pipe();
      if (!PP) return LORENZ_E_CUDA;
      cudaStream_t st = PP->st[0];
      lorenz_result* d_res = nullptr;
      if ((ret = alloc_result(&d_res, st)) != LORENZ_OK) return ret;
      ret = decrypt ? lorenz_decrypt_async(k, n, B0, B1, din, dout, nullptr, d_res, st)
                    : lorenz_encrypt_async(k, n, B0, B1, din, dout, d_res, st);
      const lorenz_status f = finish_sync(d_res, st, h_res);
      if (ret == LORENZ_OK) ret = f;
      if (decrypt && ret == LORENZ_E_INTEGRITY && outb) std::memset(out_host, 0, outb);  // never release it
      return ret;
    }
  }
  const uint64_t nbk = B1 - B0;
  const uint64_t Bsz = block_B(K, n);
  // Chunk plan: block boundaries cut[0..C]. The chunk kernels run one after another (each is a
  // launch of its own, so the library's schedule choice applies to it), overlapped with the next
  // chunk's H2D and the previous chunk's D2H. n_chunks > 0: C equal chunks. Automatic: the first
  // and the last chunk — whose copies nothing overlaps — are the smallest that still give 2 warps
  // per SM sub-partition (8 x SMs units of 32 blocks); the middle is cut into chunks of at most
  // kHostChunk bytes (and at least that minimum). Slices under two minimal chunks: one chunk.
  std::vector<uint64_t> cut;
  if (n_chunks) {
    const uint64_t C = std::min<uint64_t>(n_chunks, nbk);
    for (uint64_t c = 0; c <= C; ++c) cut.push_back(B0 + (uint64_t)((unsigned __int128)nbk * c / C));
  } else {
    const uint64_t edge = 32 * 8 * (uint64_t)sm_count();
    cut.push_back(B0);
    if (nbk >= 2 * edge) {
      const uint64_t mid = nbk - 2 * edge;
      if (mid < edge) {
        cut.push_back(B0 + nbk / 2);
      } else {
        const uint64_t maxb = std::max<uint64_t>(edge, kHostChunk / std::max<uint64_t>(Bsz, 1));
        const uint64_t M = (mid + maxb - 1) / maxb;
        cut.push_back(B0 + edge);
        for (uint64_t i = 1; i < M; ++i) cut.push_back(B0 + edge + (uint64_t)((unsigned __int128)mid * i / M));
        cut.push_back(B1 - edge);
      }
    }
    cut.push_back(B1);
  }
  const uint64_t C = cut.size() - 1;
  const uint32_t S = (uint32_t)std::min<uint64_t>(C, HostPipe::kStreams);
  uint64_t cap_in = 16, cap_out = 16, cap_blk = 1;  // the largest chunk
  for (uint64_t c = 0; c < C; ++c) {
    const uint64_t b0 = cut[c], b1 = cut[c + 1];
    uint64_t cp, cc;
    slice_bytes(K, n, b0, b1, &cp, &cc);
    cap_in = std::max(cap_in, decrypt ? cc : cp);
    cap_out = std::max(cap_out, decrypt ? cp : cc);
    cap_blk = std::max(cap_blk, b1 - b0);
  }
  HostPipe* PP = host_pipe();
  if (!PP) return LORENZ_E_CUDA;
  HostPipe& P = *PP;
  P.use((int)S);
  uint8_t *d_in[HostPipe::kStreams] = {}, *d_out[HostPipe::kStreams] = {}, *d_ok[HostPipe::kStreams] = {};
  lorenz_result* d_res = nullptr;
  cudaStream_t s0 = P.st[0];
  for (uint32_t i = 0; i < S && ret == LORENZ_OK; ++i)
    if (!cuda_ok(lz::lib_malloc_async(reinterpret_cast<void**>(&d_in[i]), cap_in, s0), "alloc in") ||
        !cuda_ok(lz::lib_malloc_async(reinterpret_cast<void**>(&d_out[i]), cap_out, s0), "alloc out") ||
        (decrypt && !cuda_ok(lz::lib_malloc_async(reinterpret_cast<void**>(&d_ok[i]), cap_blk, s0), "alloc ok")))
      ret = LORENZ_E_CUDA;
  if (ret == LORENZ_OK) ret = alloc_result(&d_res, s0);
  if (ret == LORENZ_OK) {
    P.fan_out();
    for (uint64_t c = 0; c < C && ret == LORENZ_OK; ++c) {
      const uint64_t b0 = cut[c], b1 = cut[c + 1];
      if (b0 == b1) continue;
      const uint32_t sl = (uint32_t)(c % S);
      cudaStream_t st = P.st[sl];
      uint64_t cp, cc;
      slice_bytes(K, n, b0, b1, &cp, &cc);
      const uint64_t poff = (b0 - B0) * Bsz, coff = poff + 16 * (b0 - B0);  // offsets inside the slice
      const uint64_t ioff = decrypt ? coff : poff, ooff = decrypt ? poff : coff;
      const uint64_t ib = decrypt ? cc : cp, ob = decrypt ? cp : cc;
      // H2Ds in chunk order (the copy engines would otherwise share their bandwidth between the
      // streams' copies and delay the first chunk's kernel)
      if (c > 0) cudaStreamWaitEvent(st, P.cp[(c - 1) % S], 0);
      if (ib && !cuda_ok(cudaMemcpyAsync(d_in[sl], in_host + ioff, ib, cudaMemcpyHostToDevice, st), "H2D")) {
        ret = LORENZ_E_CUDA;
        break;
      }
      cudaEventRecord(P.cp[sl], st);
      if (c > 0) cudaStreamWaitEvent(st, P.kd[(c - 1) % S], 0);  // kernels in chunk order, one at a time
      ret = decrypt ? lorenz_decrypt_async(k, n, b0, b1, d_in[sl], d_out[sl], d_ok[sl], d_res, st)
                    : lorenz_encrypt_async(k, n, b0, b1, d_in[sl], d_out[sl], d_res, st);
      cudaEventRecord(P.kd[sl], st);
      if (ret == LORENZ_OK && ob &&
          !cuda_ok(cudaMemcpyAsync(out_host + ooff, d_out[sl], ob, cudaMemcpyDeviceToHost, st), "D2H"))
        ret = LORENZ_E_CUDA;
    }
    P.fan_in();
  }
  for (uint32_t i = 0; i < S; ++i) {
    if (d_in[i]) cudaFreeAsync(d_in[i], s0);
    if (d_out[i]) cudaFreeAsync(d_out[i], s0);
    if (d_ok[i]) cudaFreeAsync(d_ok[i], s0);
  }
  if (d_res) {
    lorenz_status f = finish_sync(d_res, s0, h_res);
    if (ret == LORENZ_OK) ret = f;
  } else {
    cudaStreamSynchronize(s0);
  }
  if (decrypt && ret == LORENZ_E_INTEGRITY && outb) std::memset(out_host, 0, outb);  // never release it
  return ret;
}

lorenz_status lorenz_encrypt_host(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1, const uint8_t* pt_host,
                                  uint8_t* ct_host, uint8_t tag_xor[16], uint32_t n_chunks) {
  if (tag_xor) std::memset(tag_xor, 0, 16);
  lorenz_result h;
  std::memset(&h, 0, sizeof h);
  lorenz_status ret = host_range(k, n, b0, b1, pt_host, ct_host, false, &h, n_chunks);
  if (ret == LORENZ_OK && tag_xor) std::memcpy(tag_xor, h.tag_xor, 16);
  return ret;
}

lorenz_status lorenz_decrypt_host(const lorenz_key* k, uint64_t n, uint64_t b0, uint64_t b1, const uint8_t* ct_host,
                                  uint8_t* pt_host, int64_t* first_bad_block, uint32_t n_chunks) {
  if (first_bad_block) *first_bad_block = -1;
  lorenz_result h;
  std::memset(&h, 0, sizeof h);
  h.first_bad = ~0ULL;
  lorenz_status ret = host_range(k, n, b0, b1, ct_host, pt_host, true, &h, n_chunks);
  if (first_bad_block && h.first_bad != ~0ULL) *first_bad_block = (int64_t)h.first_bad;
  return ret;
}

}  // extern "C"
