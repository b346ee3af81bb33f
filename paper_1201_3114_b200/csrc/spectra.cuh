// spectra.cuh — NEXT-4 analysis kernels for the paper's §4 figures: the autocorrelation
// matrices of Fig.3 and the 2-D Fourier power spectra of Fig.4,
// readings Q25-Q27.
//
// Both are 2-D FFTs of an H x W byte matrix (powers of two, 2..4096), FP64:
//   power spectrum  P = |FFT2(x)|^2 / (HW)^2, DC-centred;
//   autocorrelation r = Re FFT2(|FFT2(x - mean)|^2) / (its lag-0 value)   (Wiener-Khinchin;
//                   FFT instead of the inverse FFT: the input is real, so only a conjugation
//                   differs and Re is unchanged).
// One pass = one batch of 1-D FFTs of length n along rows (stride 1) or columns (stride W):
// a CTA loads C sequences into shared memory in bit-reversed order (coalesced along the
// contiguous axis), runs the log2(n) radix-2 DIT stages in place against a per-CTA
// twiddle table (sincospi of exact dyadic arguments), and writes back through a fused epilogue
// (|F|^2, the DC shift and 1/N^2 scaling, or the real part). HBM / shared-memory bound:
// 5 log2(n) flops per element per pass against 32 bytes of HBM traffic.
#pragma once
#include <cstdint>

namespace lz {

constexpr int kFftCta = 256;
constexpr uint32_t kFftElems = 4096;  // complex elements per CTA (64 KiB + padding + twiddles)

enum FftIn : int { FFT_IN_BYTES = 0, FFT_IN_CENTRED = 1, FFT_IN_COMPLEX = 2 };
enum FftOut : int { FFT_OUT_COMPLEX = 0, FFT_OUT_POWER = 1, FFT_OUT_SPECTRUM = 2, FFT_OUT_REAL = 3 };

struct FftPass {
  uint32_t n, logn;   // FFT length (power of two) and log2(n)
  uint32_t nseq, C;   // sequences in the batch, sequences per CTA
  uint64_t stride;    // elements between consecutive points of a sequence (1 = rows)
  uint64_t dist;      // elements between consecutive sequences
  uint32_t H, W;      // matrix shape (for the DC shift)
  double scale;       // FFT_OUT_SPECTRUM: 1 / (HW)^2 (a power of two: exact)
};

__host__ __device__ inline uint32_t fft_seq_per_cta(uint32_t n, uint32_t nseq) {
  const uint32_t c = n >= kFftElems ? 1u : kFftElems / n;
  return c < nseq ? c : nseq;
}
__host__ __device__ inline size_t fft_smem_bytes(uint32_t n, uint32_t C) {
  return (size_t)C * (n + 1) * 16 + (size_t)(n / 2) * 16;  // padded sequences + twiddles
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

// element e of the CTA's tile -> (sequence s in the CTA, point k): the contiguous axis is the
// fastest-varying thread index, so global loads / stores coalesce along rows or along columns
__device__ __forceinline__ void fft_map(const FftPass& p, uint32_t e, uint32_t& s, uint32_t& k) {
  if (p.stride == 1) { s = e >> p.logn; k = e & (p.n - 1); }
  else { s = e % p.C; k = e / p.C; }
}

template <int IN, int OUT>
__global__ void __launch_bounds__(kFftCta)
    fft_pass_kernel(const FftPass p, const uint8_t* __restrict__ bytes, const double2* cin, double2* cout,
                    double* __restrict__ rout, const unsigned long long* __restrict__ sum, double* __restrict__ lag0) {
  extern __shared__ double2 fsm[];
  double2* tw = fsm + (size_t)p.C * (p.n + 1);
  const uint32_t n = p.n, half = n >> 1, row = n + 1;
  const uint64_t seq0 = (uint64_t)blockIdx.x * p.C;
  const uint32_t C = (seq0 + p.C <= p.nseq) ? p.C : (uint32_t)(p.nseq - seq0);
  for (uint32_t t = threadIdx.x; t < half; t += kFftCta) {  // exp(-2 pi i t / n)
    double s, c;
    sincospi(__ddiv_rn(2.0 * t, (double)n), &s, &c);
    tw[t] = make_double2(c, -s);
  }
  double mean = 0.0;
  if (IN == FFT_IN_CENTRED) mean = __ddiv_rn((double)*sum, (double)p.H * (double)p.W);  // exact: HW = 2^k
  const uint32_t E = C * n;
  for (uint32_t e = threadIdx.x; e < E; e += kFftCta) {
    uint32_t s, k;
    fft_map(p, e, s, k);
    const uint64_t g = (seq0 + s) * p.dist + (uint64_t)k * p.stride;
    double2 v;
    if (IN == FFT_IN_COMPLEX) v = cin[g];
    else if (IN == FFT_IN_CENTRED) v = make_double2(__dsub_rn((double)bytes[g], mean), 0.0);  // exact
    else v = make_double2((double)bytes[g], 0.0);
    fsm[s * row + (__brev(k) >> (32 - p.logn))] = v;
  }
  __syncthreads();
  // radix-2 DIT, in place; stage with half-size m uses twiddle index j * (n / 2m)
  for (uint32_t lm = 0; lm < p.logn; ++lm) {
    const uint32_t m = 1u << lm, tshift = p.logn - 1 - lm;
    for (uint32_t b = threadIdx.x; b < C * half; b += kFftCta) {
      const uint32_t s = b >> (p.logn - 1), q = b & (half - 1);
      const uint32_t j = q & (m - 1), i0 = ((q >> lm) << (lm + 1)) + j;
      double2* xs = fsm + s * row;
      const double2 a = xs[i0], t = cmul(tw[j << tshift], xs[i0 + m]);
      xs[i0] = make_double2(__dadd_rn(a.x, t.x), __dadd_rn(a.y, t.y));
      xs[i0 + m] = make_double2(__dsub_rn(a.x, t.x), __dsub_rn(a.y, t.y));
    }
    __syncthreads();
  }
  for (uint32_t e = threadIdx.x; e < E; e += kFftCta) {
    uint32_t s, k;
    fft_map(p, e, s, k);
    const uint64_t g = (seq0 + s) * p.dist + (uint64_t)k * p.stride;
    const double2 v = fsm[s * row + k];
    if (OUT == FFT_OUT_COMPLEX) {
      cout[g] = v;
    } else if (OUT == FFT_OUT_POWER) {
      cout[g] = make_double2(__dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y)), 0.0);
    } else if (OUT == FFT_OUT_SPECTRUM) {
      const uint64_t i = g / p.W, jj = g % p.W;  // frequency (k, l) -> DC-centred position
      const uint64_t o = ((i + p.H / 2) & (p.H - 1)) * p.W + ((jj + p.W / 2) & (p.W - 1));
      rout[o] = __dmul_rn(__dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y)), p.scale);
    } else {
      rout[g] = v.x;
      if (g == 0) *lag0 = v.x;
    }
  }
}

// sum of the H*W bytes (the mean of the autocorrelation's centring; < 2^36, exact)
__global__ void __launch_bounds__(kFftCta) byte_sum_kernel(const uint8_t* __restrict__ x, uint64_t n,
                                                           unsigned long long* __restrict__ out) {
  unsigned long long acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * kFftCta + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kFftCta)
    acc += x[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// r = c / c(0,0); a zero-variance input (c(0,0) = 0 exactly) gives the S:436 convention (Q25)
__global__ void __launch_bounds__(kFftCta) autocorr_normalise_kernel(double* __restrict__ r, uint64_t n,
                                                                     const double* __restrict__ lag0) {
  const double c0 = *lag0;
  for (uint64_t i = (uint64_t)blockIdx.x * kFftCta + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kFftCta)
    r[i] = c0 == 0.0 ? (i == 0 ? 1.0 : 0.0) : __ddiv_rn(r[i], c0);
}

// spectral flatness of a DC-centred spectrum: per-CTA partial (sum log P, sum P) over the non-DC
// bins in a fixed grid-stride order, then one CTA combines the partials in index order
// (deterministic: the same bits every run)
constexpr int kFlatCtas = 296;
__global__ void __launch_bounds__(kFftCta) flatness_partial_kernel(const double* __restrict__ P, uint64_t n,
                                                                   uint64_t dc, double2* __restrict__ part) {
  __shared__ double2 red[kFftCta / 32];
  double sl = 0.0, sp = 0.0;
  for (uint64_t i = (uint64_t)blockIdx.x * kFftCta + threadIdx.x; i < n; i += (uint64_t)kFlatCtas * kFftCta)
    if (i != dc) {
      sl = __dadd_rn(sl, log(P[i]));
      sp = __dadd_rn(sp, P[i]);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sl = __dadd_rn(sl, __shfl_xor_sync(0xffffffffu, sl, o));
    sp = __dadd_rn(sp, __shfl_xor_sync(0xffffffffu, sp, o));
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_double2(sl, sp);
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 a = red[0];
    for (int w = 1; w < kFftCta / 32; ++w) a = make_double2(__dadd_rn(a.x, red[w].x), __dadd_rn(a.y, red[w].y));
    part[blockIdx.x] = a;
  }
}

__global__ void flatness_final_kernel(const double2* __restrict__ part, uint64_t bins, double* __restrict__ out) {
  if (threadIdx.x) return;
  double sl = 0.0, sp = 0.0;
  for (int b = 0; b < kFlatCtas; ++b) {
    sl = __dadd_rn(sl, part[b].x);
    sp = __dadd_rn(sp, part[b].y);
  }
  const double M = (double)bins;
  *out = sp == 0.0 ? 0.0 : __ddiv_rn(exp(__ddiv_rn(sl, M)), __ddiv_rn(sp, M));
}

}  // namespace lz
