// lorenz_spectra.cu — host side of the NEXT-4 analysis calls lorenz_power_spectrum and
// lorenz_autocorrelation (include/lorenz.h): the FFT pass plans and launches of spectra.cuh.
// A translation unit of its own so the FFT instantiations compile beside the chain kernels
// (build.py).
#include <cuda.h>
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled (the driver entry point, fetched at run time)
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <mutex>
#include <string>

#include "../../include/lorenz.h"
#include "seg_launch.h"
#include "spectra.cuh"

namespace lz {
void set_last_error(const std::string& s);  // lorenz.cu
int device_sm_count();                      // lorenz.cu
}  // namespace lz

namespace {
bool cuda_ok(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return true;
  lz::set_last_error(std::string(what) + ": " + cudaGetErrorString(e));
  return false;
}
int sm_count() { return lz::device_sm_count(); }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
struct Trace {
  explicit Trace(const char* name) { nvtxRangePushA(name); }
  ~Trace() { nvtxRangePop(); }
};
}  // namespace

namespace {
bool fft_side(uint32_t v) { return v >= 2 && v <= 4096 && (v & (v - 1)) == 0; }
uint32_t ilog2(uint32_t v) { return 31u - (uint32_t)__builtin_clz(v); }

// workspace row pitch (elements). Padding it (2..256 elements) measured no difference at 4096^2,
// so the workspace is dense.
uint64_t fft_ws_pitch(uint32_t W) { return W; }

lz::FftPass fft_rows(uint32_t H, uint32_t W, uint64_t in_pitch, uint64_t out_pitch) {
  lz::FftPass p = lz::fft_plan(W, ilog2(W), H, true);
  p.rows = 1;
  p.in_pitch = in_pitch;
  p.out_pitch = out_pitch;
  p.H = H;
  p.W = W;
  return p;
}
lz::FftPass fft_cols(uint32_t H, uint32_t W, uint64_t in_pitch, uint64_t out_pitch) {
  lz::FftPass p = lz::fft_plan(H, ilog2(H), W, false);
  p.rows = 0;
  p.in_pitch = in_pitch;
  p.out_pitch = out_pitch;
  p.H = H;
  p.W = W;
  return p;
}

// one 1-D FFT pass over the batch; n >= 1024 runs the persistent prefetching kernel (complex input,
// or 16-byte aligned byte rows). *grid_out = the grid used (one flatness partial per CTA).
template <int IN, int OUT>
bool fft_launch(const lz::FftPass& p, const uint8_t* bytes, const double2* cin, double2* cout, double* rout,
                const unsigned long long* sum, double* lag0, cudaStream_t st, unsigned* grid_out = nullptr) {
  const size_t smem = lz::fft_smem_bytes(
      p, OUT == lz::FFT_OUT_R2C || OUT == lz::FFT_OUT_HALF_SPECTRUM || OUT == lz::FFT_OUT_POWER_FFT);
  const unsigned tiles = (p.nseq + p.S - 1) / p.S, cta = lz::fft_cta(p.n, p.rows != 0);
  const bool persist =
      p.logn >= 10 && OUT <= lz::FFT_OUT_REAL && IN <= lz::FFT_IN_COMPLEX &&  // plain modes only
      (IN == lz::FFT_IN_COMPLEX || (p.rows && p.in_pitch == p.n && aligned16(bytes)));
  auto go = [&](auto kernel) {
    if (!cuda_ok(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "fft smem"))
      return false;
    unsigned grid = tiles;
    if (persist) {
      int occ = 0;
      if (!cuda_ok(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, (int)cta, smem), "fft occupancy"))
        return false;
      grid = std::min<unsigned>(tiles, (unsigned)std::max(1, occ) * (unsigned)sm_count());
    }
    if (grid_out) *grid_out = grid;
    kernel<<<grid, cta, smem, st>>>(p, bytes, cin, cout, rout, sum, lag0);
    return cuda_ok(cudaGetLastError(), "fft pass");
  };
  switch (p.logn) {
    case 1: return go(lz::fft_pass_kernel<IN, OUT, 1, 256>);
    case 2: return go(lz::fft_pass_kernel<IN, OUT, 2, 256>);
    case 3: return go(lz::fft_pass_kernel<IN, OUT, 3, 256>);
    case 4: return go(lz::fft_pass_kernel<IN, OUT, 4, 256>);
    case 5: return go(lz::fft_pass_kernel<IN, OUT, 5, 256>);
    case 6: return go(lz::fft_pass_kernel<IN, OUT, 6, 256>);
    case 7: return go(lz::fft_pass_kernel<IN, OUT, 7, 256>);
    case 8: return go(lz::fft_pass_kernel<IN, OUT, 8, 256>);
    case 9: return go(lz::fft_pass_kernel<IN, OUT, 9, 256>);
    case 10:
      return persist ? go(lz::fft_persistent_kernel<IN, OUT, 10, 256>) : go(lz::fft_pass_kernel<IN, OUT, 10, 256>);
    case 11:
      if (cta == 128 && !persist) return go(lz::fft_pass_kernel<IN, OUT, 11, 128>);
      return persist ? go(lz::fft_persistent_kernel<IN, OUT, 11, 256>) : go(lz::fft_pass_kernel<IN, OUT, 11, 256>);
    default:
      if (cta == 512)
        return persist ? go(lz::fft_persistent_kernel<IN, OUT, 12, 512>) : go(lz::fft_pass_kernel<IN, OUT, 12, 512>);
      return persist ? go(lz::fft_persistent_kernel<IN, OUT, 12, 256>) : go(lz::fft_pass_kernel<IN, OUT, 12, 256>);
  }
}



// The four-step column transform of the power spectrum (spectra.cuh "four-step column transform"):
// H = 16 H2 for H = 2048, 4096, with at least 8 packed columns.
bool four_step_cols(uint32_t H, uint32_t M) { return (H == 2048 || H == 4096) && M >= 8; }

// stage 2 at H2 = 256: 8 columns per 128-thread CTA (against 16 per 256: 4096^2 spectrum 0.189 -> 0.188 ms)
#ifndef LZ_S2_CTA
#define LZ_S2_CTA 128
#endif
lz::FftPass four_step_stage2(uint32_t H, uint32_t W, uint32_t M) {
  const uint32_t H2 = H / 16;
  lz::FftPass c = lz::fft_plan(H2, ilog2(H2), M, false);
  if (LZ_S2_CTA == 128 && H2 == 256 && c.S == 16) {  // 8 columns per 128-thread CTA
    c.S = 8;
    c.logS = 3;
    c.pitch = H2 + H2 / 16;
    c.pitch += (1 - c.pitch % 8 + 8) % 8;  // pitch = 1 (mod 8): fft_plan's rule for 8 sequences per phase
  }
  c.rows = 0;
  c.in_pitch = M;
  c.out_pitch = M;
  c.H = H;
  c.W = W;
  c.kmul = 16;
  c.ysplit = 1;
  c.in_y_off = (uint64_t)H2 * M;
  return c;
}

// stage 1 -> stage 2 (16 blocks of H2 rows) -> the packed column's unpacking, whose last CTA combines the
// flatness partials (stage 2's CTAs, then the unpacking's) when flatness != null
bool four_step_spectrum(uint32_t H, uint32_t W, uint32_t M, double scale, double2* ws, double2* col0,
                        double* power, double2* part, unsigned* ctr, double* flatness, cudaStream_t st) {
  const uint32_t H2 = H / 16;
  lz::FftPass c = four_step_stage2(H, W, M);
  c.scale = scale;
  c.part = part;
  c.col0_out = col0;
  lz::FftPass s1 = c;
  const dim3 g1(H2 / 32, (M + 7) / 8);
  if (H == 4096) lz::fft_col_stage1_kernel<12><<<g1, 256, 0, st>>>(s1, ws, ctr);
  else lz::fft_col_stage1_kernel<11><<<g1, 256, 0, st>>>(s1, ws, ctr);
  if (!cuda_ok(cudaGetLastError(), "fft stage 1")) return false;
  const size_t smem = lz::fft_smem_bytes(c, true);
  const dim3 g2((c.nseq + c.S - 1) / c.S, 16);
  auto go = [&](auto kernel, unsigned cta) {
    if (!cuda_ok(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "fft smem"))
      return false;
    kernel<<<g2, cta, smem, st>>>(c, nullptr, ws, nullptr, power, nullptr, nullptr);
    return cuda_ok(cudaGetLastError(), "fft stage 2");
  };
  const bool ok =
      H2 == 256 ? (c.S == 8 ? go(lz::fft_pass_kernel<lz::FFT_IN_COMPLEX, lz::FFT_OUT_HALF_SPECTRUM, 8, 128>, 128)
                            : go(lz::fft_pass_kernel<lz::FFT_IN_COMPLEX, lz::FFT_OUT_HALF_SPECTRUM, 8, 256>, 256))
                : go(lz::fft_pass_kernel<lz::FFT_IN_COMPLEX, lz::FFT_OUT_HALF_SPECTRUM, 7, 256>, 256);
  if (!ok) return false;
  const unsigned g3 = H / 256;
  lz::col0_unpack_kernel<256><<<g3, 256, 0, st>>>(c, col0, power, part ? part + g2.x * g2.y : nullptr, ctr, part,
                                                  g2.x * g2.y + g3, (uint64_t)H * W - 1, flatness);
  return cuda_ok(cudaGetLastError(), "fft col0 unpack");
}

// The TMA column pass (spectra.cuh fft_col_tma_kernel): a tensor map over the H x M double2
// workspace seen as H rows of 2 M doubles, boxes of 256 rows x 2 doubles. cuTensorMapEncodeTiled is a
// driver call; the runtime hands out its entry point (no link against libcuda).
#ifndef LZ_COL_TMA
#define LZ_COL_TMA 1
#endif
bool col_tensor_map(CUtensorMap* map, double2* ws, uint32_t H, uint32_t M) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    else
      cudaGetLastError();
  });
  if (!encode) return false;
  const cuuint64_t dims[2] = {2ull * M, H};
  const cuuint64_t strides[1] = {(cuuint64_t)M * sizeof(double2)};
  const cuuint32_t box[2] = {2, 256}, estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, ws, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the autocorrelation's fused column pass over M packed columns of H = 2048 or 4096 rows with TMA; false
// (nothing launched) when the tensor map cannot be built, and the caller runs fft_pass_kernel instead
bool col_power_fft_tma(const lz::FftPass& cols, double2* ws, uint32_t H, uint32_t M, cudaStream_t st, bool* launched) {
  *launched = false;
  if (!LZ_COL_TMA || (H != 4096 && H != 2048)) return true;
  CUtensorMap map;
  if (!col_tensor_map(&map, ws, H, M)) return true;
  lz::FftPass c = cols;
  c.S = 1;
  c.logS = 0;
  c.T = H / 16;
  c.pitch = H + H / 16;
  const size_t smem = (size_t)c.pitch * sizeof(double2) + 128;  // + alignment slack (TMA: 128-byte boxes)
  auto go = [&](auto kernel) {
    if (!cuda_ok(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "fft smem"))
      return false;
    kernel<<<M, H / 16, smem, st>>>(c, map);
    *launched = true;
    return cuda_ok(cudaGetLastError(), "fft column pass (TMA)");
  };
  return H == 4096 ? go(lz::fft_col_tma_kernel<12>) : go(lz::fft_col_tma_kernel<11>);
}

lorenz_status spectra_args(const uint8_t* x, uint32_t H, uint32_t W, const double* out) {
  if (!x || !out || !fft_side(H) || !fft_side(W) || (reinterpret_cast<uintptr_t>(out) & 7)) {
    lz::set_last_error("H and W must be powers of two in [2, 4096]; x and out non-null device pointers, out 8-aligned");
    return LORENZ_E_ARG;
  }
  return LORENZ_OK;
}
}  // namespace
extern "C" {

lorenz_status lorenz_power_spectrum(const uint8_t* x, uint32_t H, uint32_t W, double* power, double* flatness,
                                    void* stream) {
  Trace tr("lorenz_power_spectrum");
  lorenz_status ret = spectra_args(x, H, W, power);
  if (ret != LORENZ_OK) return ret;
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t N = (uint64_t)H * W;
  double2* ws = nullptr;
  double2* part = nullptr;
  // real input: W-point row transforms as W/2-point complex FFTs of byte pairs (FFT_IN_PAIRS ->
  // FFT_OUT_R2C), then W/2 packed columns whose powers are written at (k, l) and (-k, -l)
  // (FFT_OUT_HALF_SPECTRUM): half the FFT work and the workspace of the complex path. W = 2 keeps
  // the complex path.
  const bool r2c = W >= 4;
  const uint32_t M = r2c ? W / 2 : W;
  const uint64_t NW = (uint64_t)H * M;
  if (!cuda_ok(lz::lib_malloc_async(reinterpret_cast<void**>(&ws), NW * sizeof(double2), st), "alloc fft"))
    return LORENZ_E_CUDA;
  lz::FftPass rows = fft_rows(H, M, W, M), cols = fft_cols(H, M, M, W);
  rows.W = cols.W = W;
  cols.scale = std::ldexp(1.0, -2 * (int)ilog2((uint32_t)N));  // 1 / N^2
  const bool four = r2c && four_step_cols(H, M);
  uint32_t tiles = (cols.nseq + cols.S - 1) / cols.S;  // >= the column pass's grid
  if (four) {
    const lz::FftPass c2 = four_step_stage2(H, W, M);
    tiles = 16 * ((c2.nseq + c2.S - 1) / c2.S) + H / 256;
  }
  unsigned nparts = 0;  // one flatness partial per column CTA
  // (+ 16 bytes: the four-step's CTA counter)
  bool ok = !flatness || cuda_ok(lz::lib_malloc_async(reinterpret_cast<void**>(&part), (tiles + 1) * sizeof(double2), st),
                                 "alloc");
  double2* col0 = nullptr;  // the four-step's packed column U[k]
  ok = ok && (!four || cuda_ok(lz::lib_malloc_async(reinterpret_cast<void**>(&col0), H * sizeof(double2), st), "alloc"));
  cols.part = flatness ? part : nullptr;
  if (four)
    ok = ok &&
         fft_launch<lz::FFT_IN_PAIRS, lz::FFT_OUT_R2C>(rows, x, nullptr, ws, nullptr, nullptr, nullptr, st) &&
         four_step_spectrum(H, W, M, cols.scale, ws, col0, power, cols.part,
                            part ? reinterpret_cast<unsigned*>(part + tiles) : nullptr, flatness, st);
  else if (r2c)
    ok = ok &&
         fft_launch<lz::FFT_IN_PAIRS, lz::FFT_OUT_R2C>(rows, x, nullptr, ws, nullptr, nullptr, nullptr, st) &&
         fft_launch<lz::FFT_IN_COMPLEX, lz::FFT_OUT_HALF_SPECTRUM>(cols, nullptr, ws, ws, power, nullptr, nullptr,
                                                                   st, &nparts);
  else
    ok = ok &&
         fft_launch<lz::FFT_IN_BYTES, lz::FFT_OUT_COMPLEX>(rows, x, nullptr, ws, nullptr, nullptr, nullptr, st) &&
         fft_launch<lz::FFT_IN_COMPLEX, lz::FFT_OUT_SPECTRUM>(cols, nullptr, ws, ws, power, nullptr, nullptr, st,
                                                              &nparts);
  if (ok && flatness && !four) {  // (the four-step path's col0_unpack_kernel combines them)
    lz::flatness_final_kernel<<<1, lz::kFftCta, 0, st>>>(part, nparts, N - 1, flatness);
    ok = cuda_ok(cudaGetLastError(), "flatness");
  }
  cudaFreeAsync(ws, st);
  if (part) cudaFreeAsync(part, st);
  if (col0) cudaFreeAsync(col0, st);
  return ok ? LORENZ_OK : LORENZ_E_CUDA;
}

lorenz_status lorenz_autocorrelation(const uint8_t* x, uint32_t H, uint32_t W, double* r, void* stream) {
  Trace tr("lorenz_autocorrelation");
  lorenz_status ret = spectra_args(x, H, W, r);
  if (ret != LORENZ_OK) return ret;
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t N = (uint64_t)H * W;
  double2* ws = nullptr;
  unsigned long long* aux = nullptr;  // [0] = byte sum, [1] = lag-0 value (double bits), [2] = sum of squares
  // real input (W >= 4): R2C rows of centred byte pairs -> one fused column pass (transform, |.|^2,
  // transform: FFT_OUT_POWER_FFT) over the W/2 packed columns -> C2R rows -> normalisation.
  // Three transform passes over a half-size workspace instead of four full ones; W = 2 keeps the
  // complex path.
  const bool r2c = W >= 4;
  const uint32_t M = r2c ? W / 2 : W;
  const uint64_t Pw = r2c ? M : fft_ws_pitch(W), NW = (uint64_t)H * Pw;
  if (!cuda_ok(lz::lib_malloc_async(reinterpret_cast<void**>(&ws), NW * sizeof(double2), st), "alloc fft") ||
      !cuda_ok(lz::lib_malloc_async(reinterpret_cast<void**>(&aux), 32, st), "alloc aux")) {
    if (ws) cudaFreeAsync(ws, st);
    return LORENZ_E_CUDA;
  }
  double* lag0 = reinterpret_cast<double*>(aux + 1);
  const unsigned sgrid = (unsigned)std::min<uint64_t>(4ull * sm_count(), (N + lz::kFftCta - 1) / lz::kFftCta);
  bool ok = cuda_ok(cudaMemsetAsync(aux, 0, 32, st), "memset");
  if (ok) {
    lz::byte_sum_kernel<<<sgrid, lz::kFftCta, 0, st>>>(x, N, aux);
    ok = cuda_ok(cudaGetLastError(), "byte sum");
  }
  if (ok && r2c) {
    lz::FftPass rows1 = fft_rows(H, M, W, M), cols = fft_cols(H, M, M, M);
    lz::FftPass rows2 = fft_rows(H, M, M, M);
    rows1.W = cols.W = rows2.W = W;
    cols.packed0 = 1;
    bool tma = false;
    ok = fft_launch<lz::FFT_IN_PAIRS_CENTRED, lz::FFT_OUT_R2C>(rows1, x, nullptr, ws, nullptr, aux, nullptr, st) &&
         col_power_fft_tma(cols, ws, H, M, st, &tma) &&
         (tma || fft_launch<lz::FFT_IN_COMPLEX, lz::FFT_OUT_POWER_FFT>(cols, nullptr, ws, ws, nullptr, nullptr, nullptr,
                                                                       st)) &&
         fft_launch<lz::FFT_IN_C2R, lz::FFT_OUT_REAL_PAIRS>(rows2, nullptr, ws, nullptr, r, aux, nullptr, st);
  } else if (ok) {
    const lz::FftPass rows1 = fft_rows(H, W, W, Pw), cols1 = fft_cols(H, W, Pw, Pw);
    const lz::FftPass rows2 = fft_rows(H, W, Pw, Pw), cols2 = fft_cols(H, W, Pw, W);
    ok = fft_launch<lz::FFT_IN_CENTRED, lz::FFT_OUT_COMPLEX>(rows1, x, nullptr, ws, nullptr, aux, nullptr, st) &&
         fft_launch<lz::FFT_IN_COMPLEX, lz::FFT_OUT_POWER>(cols1, nullptr, ws, ws, nullptr, nullptr, nullptr, st) &&
         fft_launch<lz::FFT_IN_COMPLEX, lz::FFT_OUT_COMPLEX>(rows2, nullptr, ws, ws, nullptr, nullptr, nullptr, st) &&
         fft_launch<lz::FFT_IN_COMPLEX, lz::FFT_OUT_REAL>(cols2, nullptr, ws, nullptr, r, nullptr, lag0, st);
  }
  if (ok && !r2c) {  // the real-input pipeline normalises in its last pass (FFT_OUT_REAL_PAIRS)
    lz::autocorr_normalise_kernel<<<sgrid, lz::kFftCta, 0, st>>>(r, N, lag0);
    ok = cuda_ok(cudaGetLastError(), "normalise");
  }
  cudaFreeAsync(ws, st);
  cudaFreeAsync(aux, st);
  return ok ? LORENZ_OK : LORENZ_E_CUDA;
}

}  // extern "C"
