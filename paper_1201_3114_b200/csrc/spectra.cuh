// spectra.cuh — NEXT-4 analysis kernels for the paper's §4 figures: the autocorrelation
// matrices of Fig.3 and the 2-D Fourier power spectra of Fig.4,
// readings Q25-Q27.
//
// Both are 2-D FFTs of an H x W byte matrix (powers of two, 2..4096), FP64:
//   power spectrum  P = |FFT2(x)|^2 / (HW)^2, DC-centred;
//   autocorrelation r = Re FFT2(|FFT2(x - mean)|^2) / (its lag-0 value)   (Wiener-Khinchin;
//                   FFT instead of the inverse FFT: the input is real, so only a conjugation
//                   differs and Re is unchanged).
// One pass = one batch of 1-D FFTs of length n = 2^L along rows (stride 1) or columns
// (stride W), as Stockham autosort radix-16 passes (the last one radix 2^(L mod 4) when L is
// not a multiple of 4) held in registers: each thread owns 16 elements (n >= 16) or a whole
// sequence (n < 16). The first pass reads HBM directly (coalesced along the contiguous axis),
// the last pass writes HBM directly through a fused epilogue (|F|^2, the DC shift and 1/N^2
// scaling, or the real part); between passes the tile is exchanged through shared memory
// (padded by one element per 16 against bank conflicts). Twiddles exp(-2 pi i m / n) come from
// a per-call table (sincospi of exact dyadic arguments, L1/L2-resident); the in-register
// 2..16-point DFTs use compile-time constants. At n = 4096: 3 passes, 2 exchanges.
// HBM-bound: 16 B read + 16 B written per element per 1-D pass (bytes / doubles at the ends).
#pragma once
#include <cuda.h>  // CUtensorMap (fft_col_tma_kernel)

#include <cstdint>

namespace lz {

constexpr int kFftCtaThreads = 256;
constexpr int kFftCta = 256;  // the reductions (byte sums, flatness, col0 unpacking)

// FFT_IN_PAIRS: a real row of 2n bytes read as n complex values x[2m] + i x[2m+1] (real-to-complex)
// FFT_IN_PAIRS_CENTRED: the same with the mean subtracted (exact).
// FFT_IN_C2R: a Hermitian half spectrum Q[0..n] (Q[0] + i Q[n] packed in element 0, both real)
//   pre-processed so that one n-point FFT yields the real 2n-point transform (see c2r_load).
// FFT_IN_SMEM_DENSE: the tile is already in shared memory, unpadded (a TMA load; fft_col_tma_kernel).
enum FftIn : int {
  FFT_IN_BYTES = 0, FFT_IN_CENTRED = 1, FFT_IN_COMPLEX = 2, FFT_IN_PAIRS = 3, FFT_IN_PAIRS_CENTRED = 4,
  FFT_IN_C2R = 5, FFT_IN_SMEM_DENSE = 6
};
// FFT_OUT_R2C: unpack the row's half spectrum X[0..n] (2n-point real DFT) from the n-point complex
//   FFT of the pairs, stored as n complex values with X[0] + i X[n] packed in element 0.
// FFT_OUT_HALF_SPECTRUM: column pass over those n packed columns: |F|^2 / N^2 at (k, l) and at its
//   mirror (-k, W-l) (real input: P(k,l) = P(-k,-l)); column 0 unpacks the DC and Nyquist columns.
// FFT_OUT_POWER_FFT: column pass fusing transform -> |.|^2 (packed DC / Nyquist column unpacked) ->
//   transform again (the autocorrelation's two column transforms in one HBM round trip).
// FFT_OUT_REAL_PAIRS: the C2R row output R[m] -> real samples (2m, 2m+1) = (Re R, -Im R), divided by the
//   exact lag-0 value (lag0_exact; r(0,0) = 1): the autocorrelation normalised in its last pass.
enum FftOut : int {
  FFT_OUT_COMPLEX = 0, FFT_OUT_POWER = 1, FFT_OUT_SPECTRUM = 2, FFT_OUT_REAL = 3,
  FFT_OUT_R2C = 4, FFT_OUT_HALF_SPECTRUM = 5, FFT_OUT_POWER_FFT = 6, FFT_OUT_REAL_PAIRS = 7,
  FFT_OUT_SMEM = 8,  // the last pass leaves the transform in shared memory, natural order, unpadded (for a TMA store)
  FFT_OUT_POWER_SMEM = 9  // the last pass leaves |X|^2 (as (P, 0)) in the exchange tile: power_in_place fused
};

struct FftPass {
  uint32_t n, logn;     // FFT length (power of two, 2..4096) and log2(n)
  uint32_t nseq;        // sequences in the batch
  uint32_t T, S;        // threads per sequence (n/16, or 1 when n < 16), sequences per CTA
  uint32_t logS;        // log2(S) (S is a power of two)
  uint32_t pitch;       // shared-memory elements per sequence (n + n/16)
  uint32_t npass;       // Stockham passes
  uint32_t rlog[4];     // log2 of each pass's radix
  uint32_t rows;        // 1: sequences are rows (element (seq, idx)); 0: columns (element (idx, seq))
  uint64_t in_pitch;    // row pitch (elements) of the input matrix
  uint64_t out_pitch;   // row pitch of a complex (workspace) output
  uint32_t H, W;        // matrix shape (for the DC shift)
  double scale;         // FFT_OUT_SPECTRUM: 1 / (HW)^2 (a power of two: exact)
  uint32_t packed0;     // FFT_OUT_POWER_FFT: sequence 0 holds the packed DC + i Nyquist column
  double2* part;        // FFT_OUT_SPECTRUM (nullable): per-CTA (sum log P, sum P) over non-DC bins
  uint32_t kmul, kadd;  // columns: output position pos is row pos * kmul + kadd (1, 0 for a whole column);
                        // ysplit: kadd = blockIdx.y (stage 2 of the four-step column transform)
  uint32_t ysplit;      // 1: the grid's y index selects a block of n rows (input offset in_y_off) and the
                        // output rows pos * kmul + blockIdx.y
  uint64_t in_y_off;    // input element offset per blockIdx.y
  double2* col0_out;    // stage 2 (nullable): sequence 0's transform U[k] goes here instead of P
};

// CTA threads: 256, except 512 for 4096-point column passes (S = 2 adjacent columns per CTA,
// so every 32-byte sector a warp touches is fully used) and 128 for 2048-point row passes
// 2048-point row passes (W = 4096): one row per 128-thread CTA, four CTAs per SM (measured against two
// rows per 256-thread CTA: 4096^2 spectrum 0.189 -> 0.184 ms, autocorrelation 0.259 -> 0.253 ms)
#ifndef LZ_ROW_CTA
#define LZ_ROW_CTA 128
#endif
inline uint32_t fft_cta(uint32_t n, bool rows) {
  if (rows && n >= 2048) return LZ_ROW_CTA;
  return (!rows && n >= 4096) ? 512 : 256;
}

inline FftPass fft_plan(uint32_t n, uint32_t logn, uint32_t nseq, bool rows) {
  FftPass p{};
  p.n = n;
  p.logn = logn;
  p.nseq = nseq;
  p.T = n >= 16 ? n / 16 : 1;
  const uint32_t S = fft_cta(n, rows) / p.T;
  p.S = S < nseq ? S : nseq;
  p.logS = 0;
  while ((1u << p.logS) < p.S) ++p.logS;
  // shared pitch: the padded sequence (+1 per 16) plus an offset that puts the k sequences an
  // 8-thread shared-memory phase touches (k = 8/T rows, or min(8, S) columns) 128/k bytes apart,
  // so the phase's 16-byte accesses fall in distinct bank groups
  const uint32_t k = rows ? (p.T >= 8 ? 1 : 8 / p.T) : (p.S < 8 ? p.S : 8);
  p.pitch = n + n / 16;
  if (k > 1) p.pitch += ((8 / k) - p.pitch % 8 + 8) % 8;  // pitch = 8/k (mod 8)
  p.kmul = 1;
  p.kadd = 0;
  p.ysplit = 0;
  p.in_y_off = 0;
  p.col0_out = nullptr;
  p.npass = 0;
  uint32_t L = logn;
  while (L >= 4) { p.rlog[p.npass++] = 4; L -= 4; }
  if (L) p.rlog[p.npass++] = L;
  return p;
}
// exchange tile (>= 2 passes) or shared-memory epilogue (R2C / half-spectrum modes)
inline size_t fft_smem_bytes(const FftPass& p, bool epilogue = false) {
  return (p.npass > 1 || epilogue) ? (size_t)p.S * p.pitch * 16 : 0;
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)); }
// complex product with fused multiply-adds (4 FP64 pipe ops instead of 6; the FFTs are
// analysis arithmetic with a tolerance, not part of the bit-exact cipher)
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)), __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}

// exp(-2 pi i m / n) from sincospi of the exact dyadic argument 2m/n (each CTA builds its own
// 64 + n/64-entry shared tables with it; no global twiddle table)
__device__ __forceinline__ double2 twiddle_exact(uint32_t m, uint32_t n) {
  double sn, cs;
  sincospi(__ddiv_rn(2.0 * m, (double)n), &sn, &cs);
  return make_double2(cs, -sn);
}

// x * exp(-2 pi i m / 16), m a compile-time constant after unrolling: 1 and -i are free
__device__ __forceinline__ double2 rot16(double2 x, int m) {
  constexpr double C1 = 0.92387953251128673848, C2 = 0.70710678118654752440, C3 = 0.38268343236508978178;
  switch (m) {
    case 0: return x;
    case 4: return make_double2(x.y, -x.x);
    case 2: return make_double2(__dmul_rn(__dadd_rn(x.x, x.y), C2), __dmul_rn(__dsub_rn(x.y, x.x), C2));
    case 6: return make_double2(__dmul_rn(__dsub_rn(x.y, x.x), C2), __dmul_rn(-__dadd_rn(x.x, x.y), C2));
    case 1: return cmul(x, make_double2(C1, -C3));
    case 3: return cmul(x, make_double2(C3, -C1));
    case 5: return cmul(x, make_double2(-C3, -C1));
    default: return cmul(x, make_double2(-C1, -C3));  // 7
  }
}

// in-register R-point DFT (decimation in frequency): y_u lands in a[O + bitrev_R(u)]
template <int R>
__device__ __forceinline__ void dft_dif(double2 (&a)[16], const int O) {  // O: constant after unrolling
#pragma unroll
  for (int h = R / 2; h >= 1; h >>= 1)
#pragma unroll
    for (int b = 0; b < R; b += 2 * h)
#pragma unroll
      for (int j = 0; j < h; ++j) {
        const double2 u = a[O + b + j], v = a[O + b + j + h];
        a[O + b + j] = cadd(u, v);
        a[O + b + j + h] = rot16(csub(u, v), j * (16 / (2 * h)));
      }
}

template <int R>
__device__ __forceinline__ int bitrev_c(int u) {
  int r = 0;
#pragma unroll
  for (int b = 1; b < R; b <<= 1) r = (r << 1) | ((u & b) ? 1 : 0);
  return r;
}

__device__ __forceinline__ uint32_t fft_pad(uint32_t i) { return i + (i >> 4); }

// flatness accumulator of one thread: sum P, and sum log P kept as a product of frexp mantissas
// (each in [1/2, 1): at most 16 per thread, so no underflow) plus an exponent sum -> one log per
// thread instead of one per bin
struct FlatAcc {
  double sp = 0.0, mprod = 1.0;
  int esum = 0;
  // P = m 2^e, m in [1/2, 1): exponent field split off with integer ops for normal P >= 0;
  // zero and subnormals take frexp (P = 0 -> m = 0: log -> -inf, geometric mean 0)
  __device__ __forceinline__ static double split(double P, int& e) {
    const long long b = __double_as_longlong(P);
    const int ef = (int)(b >> 52) & 0x7ff;
    if (ef != 0) {
      e = ef - 1022;
      return __longlong_as_double((b & 0x800fffffffffffffLL) | 0x3fe0000000000000LL);
    }
    return frexp(P, &e);
  }
  __device__ __forceinline__ void add(double P) {
    int e;
    const double m = split(P, e);
    mprod = __dmul_rn(mprod, m);
    esum += e;
    sp = __dadd_rn(sp, P);
  }
  // a bin counted twice (a half-spectrum bin and its mirror): one step of each dependent chain
  __device__ __forceinline__ void add2(double P) {
    int e;
    const double m = split(P, e);
    mprod = __dmul_rn(mprod, __dmul_rn(m, m));  // m^2 >= 1/4: 16 per thread stay far from underflow
    esum += 2 * e;
    sp = __dadd_rn(sp, __dmul_rn(P, 2.0));      // exact doubling
  }
  __device__ __forceinline__ double sum_log() const {
    return __dadd_rn(log(mprod), __dmul_rn((double)esum, 0.69314718055994530942));
  }
};

// the kernel's operands and per-CTA constants
struct FftIo {
  const uint8_t* bytes;  // FFT_IN_BYTES / FFT_IN_CENTRED input (global)
  const uint8_t* sb;     // the same bytes staged in shared memory (row passes), or null
  uint64_t seq0;         // first sequence of the CTA (index origin of sb)
  const double2* cin;
  double2* cout;
  double* rout;
  double* lag0;
  double mean;
  const double2* tlo;    // shared: exp(-2 pi i m / n), m < 64, at tw_lo(m)
  const double2* thi;    // shared: exp(-2 pi i 64 m / n), m < n / 64
  const double2* t2lo;   // shared (R2C / C2R): exp(-2 pi i m / 2n), m < 64
  const double2* t2hi;   // shared (R2C / C2R): exp(-2 pi i 64 m / 2n), m < 2n / 64
  double c0 = 0.0;       // FFT_OUT_REAL_PAIRS: the unnormalised lag-0 value (lag0_exact) and its reciprocal
  double inv_c0 = 0.0;
};

// The lag-0 value of the real-input autocorrelation pipeline's unnormalised output: the second
// forward transform scales by N and the C2R pre-processing by 1/2, so it is (N/2) c(0,0) with
// c(0,0) = sum_ij (x_ij - mean)^2 = (N sum x^2 - (sum x)^2) / N, i.e. (N sum x^2 - (sum x)^2) / 2,
// from the exact byte sums; the only rounding is the 128-bit integer's conversion to binary64
// (the normaliser, fused into the last pass instead of a separate pass over r)
__device__ __forceinline__ double lag0_exact(const unsigned long long* sums, uint64_t N) {
  const unsigned __int128 num = (unsigned __int128)N * sums[2] - (unsigned __int128)sums[0] * sums[0];
  return __dmul_rn((double)num, 0.5);
}

template <int N>
__device__ __forceinline__ double2 twid2(const FftIo& io, uint32_t m) {  // exp(-2 pi i m / 2N)
  if (2 * N <= 64) return io.t2lo[m];
  return cmul(io.t2lo[m & 63], io.t2hi[m >> 6]);
}

// exp(-2 pi i m / n) = tlo[m mod 64] * thi[m / 64] (n <= 4096: two 64-entry shared tables). The low
// table holds entry m at tw_lo(m) = m + m/8: a Stockham pass's twiddle steps are multiples of 8, 16
// or 32 across a warp (pass 2 of a 2048-point row: m = 8 k), which in an unpadded table of 16-byte
// entries all fall in one bank group (an 8-way conflict); one pad entry per 8 spreads them out.
#ifndef LZ_TW_PAD
#define LZ_TW_PAD 1
#endif
__host__ __device__ constexpr uint32_t tw_lo(uint32_t m) { return LZ_TW_PAD ? m + (m >> 3) : m; }
constexpr uint32_t kTwLo = tw_lo(63) + 1;  // low-table entries (72 with the padding)
template <int N>
__host__ __device__ constexpr int tw_entries() { return (int)kTwLo + (N > 64 ? N / 64 : 1); }
// every CTA fills its own tables from sincospi of exact dyadic arguments (twiddle_exact)
template <int N>
__device__ __forceinline__ void fill_twiddles(double2* tws, uint32_t t0, uint32_t nt) {
  for (uint32_t i = t0; i < 64 + (N > 64 ? N / 64 : 0); i += nt)
    if (i < 64) { if (i < (uint32_t)N) tws[tw_lo(i)] = twiddle_exact(i, N); }
    else tws[kTwLo + i - 64] = twiddle_exact(64 * (i - 64), N);
}
template <int N>
__device__ __forceinline__ double2 twid(const FftIo& io, uint32_t m) {
  if (N <= 64) return io.tlo[tw_lo(m)];
  return cmul(io.tlo[tw_lo(m & 63)], io.thi[m >> 6]);
}

template <int IN, int N>
__device__ __forceinline__ double2 fft_load(const FftPass& p, const FftIo& io, uint64_t seq, uint32_t idx) {
  if (IN == FFT_IN_PAIRS || IN == FFT_IN_PAIRS_CENTRED) {  // rows only: bytes 2 idx, 2 idx + 1 of row seq
    const uint8_t* r = io.sb ? io.sb + (seq - io.seq0) * 2 * N : io.bytes + seq * p.in_pitch;
    if (IN == FFT_IN_PAIRS) return make_double2((double)r[2 * idx], (double)r[2 * idx + 1]);
    return make_double2(__dsub_rn((double)r[2 * idx], io.mean), __dsub_rn((double)r[2 * idx + 1], io.mean));
  }
  if (IN == FFT_IN_C2R) {  // rows only: V[l] = Ge - i Go, Ge = (Q[l] + conj Q[n-l]) / 2, Go = w (Q[l] - conj Q[n-l]) / 2
    const double2* q = io.cin + seq * p.in_pitch;
    const double2 a = q[idx];
    if (idx == 0) {  // Q[0], Q[n] real, packed in element 0
      return make_double2(__dmul_rn(__dadd_rn(a.x, a.y), 0.5), __dmul_rn(__dsub_rn(a.y, a.x), 0.5));
    }
    const double2 b = q[N - idx];  // conj(b) = conj Q[n-l]
    const double2 ge = make_double2(__dmul_rn(__dadd_rn(a.x, b.x), 0.5), __dmul_rn(__dsub_rn(a.y, b.y), 0.5));
    const double2 d = make_double2(__dmul_rn(__dsub_rn(a.x, b.x), 0.5), __dmul_rn(__dadd_rn(a.y, b.y), 0.5));
    const double2 go = cmul(twid2<N>(io, idx), d);
    return make_double2(__dadd_rn(ge.x, go.y), __dsub_rn(ge.y, go.x));  // ge - i go
  }
  const uint64_t g = p.rows ? seq * p.in_pitch + idx : (uint64_t)idx * p.in_pitch + seq;
  if (IN == FFT_IN_COMPLEX) return io.cin[g + (p.ysplit ? blockIdx.y * p.in_y_off : 0)];
  const double b = io.sb ? (double)io.sb[(seq - io.seq0) * N + idx] : (double)io.bytes[g];
  return make_double2(IN == FFT_IN_CENTRED ? __dsub_rn(b, io.mean) : b, 0.0);  // exact (HW = 2^k)
}

template <int OUT>
__device__ __forceinline__ void fft_store(const FftPass& p, const FftIo& io, uint64_t seq, uint32_t pos, double2 v,
                                          FlatAcc& acc) {
  const uint64_t i = p.rows ? seq : (uint64_t)pos * p.kmul + (p.ysplit ? blockIdx.y : p.kadd);  // (row, column)
  const uint64_t j = p.rows ? pos : seq;
  if (OUT == FFT_OUT_COMPLEX) {
    io.cout[i * p.out_pitch + j] = v;
  } else if (OUT == FFT_OUT_POWER) {
    io.cout[i * p.out_pitch + j] = make_double2(__dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y)), 0.0);
  } else if (OUT == FFT_OUT_SPECTRUM) {  // frequency (k, l) = (i, j) -> DC-centred position
    const uint64_t o = ((i + p.H / 2) & (p.H - 1)) * p.W + ((j + p.W / 2) & (p.W - 1));
    const double P = __dmul_rn(__dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y)), p.scale);
    io.rout[o] = P;
    if (p.part && (i | j) != 0) acc.add(P);  // flatness over the non-DC bins
  } else if (OUT == FFT_OUT_REAL_PAIRS) {  // rows only: r at (seq, 2 pos), (seq, 2 pos + 1), normalised
    double2 o = make_double2(0.0, 0.0);     // a zero-variance input: r = 0 off the origin
    if (io.c0 > 0.0) o = make_double2(__dmul_rn(v.x, io.inv_c0), -__dmul_rn(v.y, io.inv_c0));
    if (seq == 0 && pos == 0) o.x = 1.0;    // r(0,0) = 1 (Q25)
    reinterpret_cast<double2*>(io.rout + seq * p.W)[pos] = o;
  } else if (OUT == FFT_OUT_HALF_SPECTRUM) {  // column j in [1, W/2): (k, j) and its mirror (-k, W - j)
    const double P = __dmul_rn(__dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y)), p.scale);
    const uint64_t i2 = (p.H - i) & (p.H - 1), j2 = p.W - j;
    io.rout[((i + p.H / 2) & (p.H - 1)) * p.W + ((j + p.W / 2) & (p.W - 1))] = P;
    io.rout[((i2 + p.H / 2) & (p.H - 1)) * p.W + ((j2 + p.W / 2) & (p.W - 1))] = P;
    if (p.part) acc.add2(P);
  } else {
    io.rout[i * p.W + j] = v.x;
    if ((i | j) == 0) *io.lag0 = v.x;
  }
}

#ifndef LZ_C2R_PAIRED
#define LZ_C2R_PAIRED 1
#endif
// The C2R pre-processing done in registers (FFT_IN_C2R, first pass of radix R < 16: fft_passes then
// runs the remainder radix first). The first pass gives thread tid the G/2 groups j = tid + g T and
// their mirrors j' = NR - j (NR/2 for j = 0): the inputs l = j + t NR and N - l = j' + (R - 1 - t) NR
// are then in the same thread, which loads Q[l] and Q[N - l] once each and forms V[l] and V[N - l]
// from them (fft_load's formulas; exp(-2 pi i (N - l) / 2N) = -conj exp(-2 pi i l / 2N)). Measured
// at 4096^2: the C2R row pass 107 -> 72 us. (The same pairing for the R2C unpacking in the last
// pass measured slower, 70 -> 80 us, and is not used.)
__device__ __forceinline__ double2 c2r_v(double2 a, double2 b, double2 w) {  // a = Q[l], b = Q[N - l]
  const double2 ge = make_double2(__dmul_rn(__dadd_rn(a.x, b.x), 0.5), __dmul_rn(__dsub_rn(a.y, b.y), 0.5));
  const double2 d = make_double2(__dmul_rn(__dsub_rn(a.x, b.x), 0.5), __dmul_rn(__dadd_rn(a.y, b.y), 0.5));
  const double2 go = cmul(w, d);
  return make_double2(__dadd_rn(ge.x, go.y), __dsub_rn(ge.y, go.x));  // ge - i go
}
template <int N>
__device__ __forceinline__ void c2r_pair(const FftIo& io, double2& A, double2& B, uint32_t l) {
  const double2 a = A, b = B, w = twid2<N>(io, l);
  A = c2r_v(a, b, w);
  B = c2r_v(b, a, make_double2(-w.x, w.y));
}
template <int R, int N>
__device__ __forceinline__ void c2r_registers(const FftIo& io, double2 (&a)[16], uint32_t tid) {
  constexpr int G = 16 / R, T = N / 16, NR = N / R;
#pragma unroll
  for (int g = 0; g < G / 2; ++g) {
    const uint32_t j = tid + g * T;
    const int gm = g + G / 2;
    if (g > 0 || j != 0) {
#pragma unroll
      for (int t = 0; t < R; ++t) c2r_pair<N>(io, a[g * R + t], a[gm * R + R - 1 - t], j + t * NR);
    } else {
      const double2 q0 = a[0];  // Q[0] + i Q[N], both real
      a[0] = make_double2(__dmul_rn(__dadd_rn(q0.x, q0.y), 0.5), __dmul_rn(__dsub_rn(q0.y, q0.x), 0.5));
      {
        const double2 h = a[R / 2];  // l = N/2 pairs with itself
        a[R / 2] = c2r_v(h, h, twid2<N>(io, N / 2));
      }
#pragma unroll
      for (int t = 1; t < R / 2; ++t) c2r_pair<N>(io, a[t], a[R - t], t * NR);
#pragma unroll
      for (int t = 0; t < R / 2; ++t) c2r_pair<N>(io, a[gm * R + t], a[gm * R + R - 1 - t], NR / 2 + t * NR);
    }
  }
}

// one Stockham pass of radix R after sub-transforms of length LS: group j (< N/R) takes
// x[j + t N/R], t < R, multiplies by exp(-2 pi i t k / (LS R)), k = j mod LS, does the R-point
// DFT and writes y_u to (j - k) R + k + u LS. Everything but the thread's indices is static.
// SMEM_SRC: the first pass reads a tile already prefetched into Xs (complex input) or the byte
// stage; `pre` is called by every thread of the last pass once the tile is no longer read (the
// persistent kernel prefetches its next tile there, overlapping the last pass and its stores).
template <int R, int N, int LS, bool FIRST, bool LAST, int IN, int OUT, bool SMEM_SRC, typename Pre>
__device__ __forceinline__ void fft_pass(const FftPass& p, const FftIo& io, double2 (&a)[16], double2* Xs,
                                         uint32_t tid, uint64_t seq, bool active, bool valid, FlatAcc& acc,
                                         const Pre& pre) {
  constexpr int E = N < 16 ? N : 16, G = E / R, T = N / E, NR = N / R;
  constexpr bool FROM_XS = !FIRST || (SMEM_SRC && (IN == FFT_IN_COMPLEX || IN == FFT_IN_SMEM_DENSE));
  // the unpadded tile of a TMA load / store is read by the first pass and written by the last one at
  // consecutive indices across a warp (idx = j + t NR, pos = j + u LS): conflict-free without padding
  constexpr bool DENSE_RD = FIRST && IN == FFT_IN_SMEM_DENSE, DENSE_WR = LAST && OUT == FFT_OUT_SMEM;
  constexpr bool PAIRED_IN = LZ_C2R_PAIRED && FIRST && IN == FFT_IN_C2R && N > 16 && G >= 2;  // c2r_registers
  // group g's j: tid + g T, or for PAIRED_IN's second half the mirror NR - j of the first half's j
  // (NR/2 for j = 0), so that the thread holds the input at l and N - l together
  auto jof = [&](int g) -> uint32_t {
    if (!PAIRED_IN || g < G / 2) return tid + g * T;
    const uint32_t jj = tid + (g - G / 2) * T;
    return jj ? NR - jj : NR / 2;
  };
#pragma unroll
  for (int g = 0; g < G && active; ++g) {
    const uint32_t j = jof(g);
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const uint32_t idx = j + t * NR;
      if (PAIRED_IN) a[g * R + t] = valid ? io.cin[seq * p.in_pitch + idx] : make_double2(0.0, 0.0);
      else if (!FROM_XS) a[g * R + t] = valid ? fft_load<IN, N>(p, io, seq, idx) : make_double2(0.0, 0.0);
      else a[g * R + t] = Xs[DENSE_RD ? idx : fft_pad(idx)];
    }
  }
  if constexpr (PAIRED_IN)
    if (active) c2r_registers<R, N>(io, a, tid);
  if (FROM_XS) __syncthreads();  // every read of this pass done before anyone overwrites the tile
  if (LAST) pre();
#pragma unroll
  for (int g = 0; g < G && active; ++g) {
    const uint32_t j = jof(g), k = j & (LS - 1);
    if (LS > 1 && k) {
      // w^t for t < R from w, w^2, w^4, w^8 only: w^t = w^(t&3) * w^(t&12) (at most two extra
      // complex products per factor); each w^(2^i) is itself a product of two shared-table entries
      const uint32_t step = k * (N / (LS * R));
      const double2 one = make_double2(1.0, 0.0);
      const double2 w1 = twid<N>(io, step);
      const double2 w2 = R > 2 ? twid<N>(io, 2 * step) : one;
      const double2 w3 = R > 2 ? cmul(w1, w2) : one;
      const double2 w4 = R > 4 ? twid<N>(io, 4 * step) : one;
      const double2 w8 = R > 8 ? twid<N>(io, 8 * step) : one;
      const double2 w12 = R > 8 ? cmul(w4, w8) : one;
#pragma unroll
      for (int t = 1; t < R; ++t) {
        const int lo = t & 3, hi = t & 12;
        const double2 wl = lo == 1 ? w1 : lo == 2 ? w2 : w3;
        const double2 wh = hi == 4 ? w4 : hi == 8 ? w8 : w12;
        const double2 w = lo == 0 ? wh : hi == 0 ? wl : cmul(wl, wh);
        a[g * R + t] = cmul(a[g * R + t], w);
      }
    }
    dft_dif<R>(a, g * R);
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const uint32_t pos = (j - k) * R + k + u * LS;
      const double2 v = a[g * R + bitrev_c<R>(u)];
      if (LAST && !(OUT == FFT_OUT_R2C || OUT == FFT_OUT_POWER_FFT || OUT == FFT_OUT_SMEM || OUT == FFT_OUT_POWER_SMEM ||
                    (OUT == FFT_OUT_HALF_SPECTRUM && seq == 0))) {
        if (valid) fft_store<OUT>(p, io, seq, pos, v, acc);
      } else {
        if (LAST && OUT == FFT_OUT_POWER_SMEM)
          Xs[fft_pad(pos)] = make_double2(__dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y)), 0.0);
        else
          Xs[DENSE_WR ? pos : fft_pad(pos)] = v;  // exchange, or the input of a shared-memory epilogue
      }
    }
  }
  if (!LAST || OUT == FFT_OUT_R2C || OUT == FFT_OUT_HALF_SPECTRUM || OUT == FFT_OUT_POWER_FFT || OUT == FFT_OUT_SMEM ||
      OUT == FFT_OUT_POWER_SMEM)
    __syncthreads();
}

// the passes of an N = 2^LOGN transform: radix 16 while >= 4 bits remain, then the remainder
template <int LOGN, int DONE, int IN, int OUT, bool SMEM_SRC = false, typename Pre = void (*)()>
__device__ __forceinline__ void fft_passes(const FftPass& p, const FftIo& io, double2 (&a)[16], double2* Xs,
                                           uint32_t tid, uint64_t seq, bool active, bool valid, FlatAcc& acc,
                                           const Pre& pre) {
  // C2R input (c2r_registers) runs the remainder radix first, so that its first pass has >= 2 groups
  constexpr bool REMF = LZ_C2R_PAIRED && IN == FFT_IN_C2R && LOGN > 4 && (LOGN & 3) != 0;
  constexpr int REM = LOGN - DONE, RL = (REMF && DONE == 0) ? (LOGN & 3) : (REM >= 4 ? 4 : REM);
  fft_pass<1 << RL, 1 << LOGN, 1 << DONE, DONE == 0, REM == RL, IN, OUT, SMEM_SRC>(p, io, a, Xs, tid, seq, active,
                                                                                    valid, acc, pre);
  if constexpr (REM > RL)
    fft_passes<LOGN, DONE + RL, IN, OUT, SMEM_SRC>(p, io, a, Xs, tid, seq, active, valid, acc, pre);
}

__device__ __forceinline__ void no_prefetch() {}

// per-CTA flatness partial (sum log P, sum P): warp shuffles then warps in order (deterministic)
template <int CTA>
__device__ __forceinline__ void flat_partial(const FlatAcc& fa, double2* part) {
  {
    __shared__ double2 red[CTA / 32];
    double2 acc = make_double2(fa.sum_log(), fa.sp);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      acc = make_double2(__dadd_rn(acc.x, __shfl_xor_sync(0xffffffffu, acc.x, o)),
                         __dadd_rn(acc.y, __shfl_xor_sync(0xffffffffu, acc.y, o)));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double2 t = red[0];
      for (int w = 1; w < CTA / 32; ++w) t = make_double2(__dadd_rn(t.x, red[w].x), __dadd_rn(t.y, red[w].y));
      part[blockIdx.x + (uint64_t)gridDim.x * blockIdx.y] = t;
    }
  }
}

// spectral flatness = exp(mean log P) / mean P over the non-DC bins, from the per-CTA partials
// of the spectrum's column pass, combined in index order (deterministic: same bits every run) by one
// kFftCta-thread CTA (flatness_final_kernel, or the last CTA of col0_unpack_kernel)
__device__ __forceinline__ void flatness_combine(const double2* part, uint32_t nparts, uint64_t bins, double* out) {
  __shared__ double2 red[kFftCta];
  double sl = 0.0, sp = 0.0;
  for (uint32_t b = threadIdx.x; b < nparts; b += kFftCta) {  // fixed assignment and order
    const double2 v = __ldcg(part + b);                        // (L2: partials of other CTAs)
    sl = __dadd_rn(sl, v.x);
    sp = __dadd_rn(sp, v.y);
  }
  red[threadIdx.x] = make_double2(sl, sp);
  __syncthreads();
  for (int h = kFftCta / 2; h > 0; h >>= 1) {
    if ((int)threadIdx.x < h)
      red[threadIdx.x] = make_double2(__dadd_rn(red[threadIdx.x].x, red[threadIdx.x + h].x),
                                      __dadd_rn(red[threadIdx.x].y, red[threadIdx.x + h].y));
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double M = (double)bins;
    *out = red[0].y == 0.0 ? 0.0 : __ddiv_rn(exp(__ddiv_rn(red[0].x, M)), __ddiv_rn(red[0].y, M));
  }
}
// FFT_OUT_R2C epilogue: Z = the n-point FFT of z[m] = x[2m] + i x[2m+1] is in Xs (natural order).
// With a = Z[l], b = conj(Z[n-l]): Fe = (a + b)/2, Fo = -i (a - b)/2, w = exp(-2 pi i l / 2n):
// X[l] = Fe + w Fo and X[n-l] = conj(Fe - w Fo); X[0] = Re Z0 + Im Z0 and X[n] = Re Z0 - Im Z0 are
// stored packed as X[0] + i X[n] in element 0.
template <int N>
__device__ __forceinline__ void r2c_epilogue(const FftPass& p, const FftIo& io, const double2* Xs, uint32_t tid,
                                             uint64_t seq, bool valid, const double2* t2lo, const double2* t2hi) {
  constexpr int T = N < 16 ? 1 : N / 16;
  if (!valid) return;
  double2* y = io.cout + seq * p.out_pitch;
  for (uint32_t l = tid; l <= N / 2; l += T) {
    const double2 a = Xs[fft_pad(l)], bz = Xs[fft_pad((N - l) & (N - 1))];
    if (l == 0) {
      y[0] = make_double2(__dadd_rn(a.x, a.y), __dsub_rn(a.x, a.y));
      continue;
    }
    const double2 fe = make_double2(__dmul_rn(__dadd_rn(a.x, bz.x), 0.5), __dmul_rn(__dsub_rn(a.y, bz.y), 0.5));
    const double2 fo = make_double2(__dmul_rn(__dadd_rn(a.y, bz.y), 0.5), __dmul_rn(__dsub_rn(bz.x, a.x), 0.5));
    const double2 w = (2 * N <= 64) ? t2lo[l] : cmul(t2lo[l & 63], t2hi[l >> 6]);
    const double2 wf = cmul(w, fo);
    y[l] = make_double2(__dadd_rn(fe.x, wf.x), __dadd_rn(fe.y, wf.y));
    if (l != N / 2) y[N - l] = make_double2(__dsub_rn(fe.x, wf.x), __dsub_rn(wf.y, fe.y));
  }
}

// FFT_OUT_HALF_SPECTRUM epilogue for column 0 (sequence 0): U = FFT(X[.,0] + i X[.,W/2]) is in Xs.
// A[k] = (U[k] + conj(U[-k]))/2 and B[k] = -i (U[k] - conj(U[-k]))/2 are the spectra of the DC and
// Nyquist columns: P(k, 0) = |A|^2 / N^2, P(k, W/2) = |B|^2 / N^2.
template <int N>
__device__ __forceinline__ void half_col0_epilogue(const FftPass& p, const FftIo& io, const double2* Xs,
                                                   uint32_t tid, FlatAcc& acc) {
  constexpr int T = N < 16 ? 1 : N / 16;
  for (uint32_t k = tid; k < N; k += T) {
    const double2 a = Xs[fft_pad(k)], bz = Xs[fft_pad((N - k) & (N - 1))];
    const double2 A = make_double2(__dmul_rn(__dadd_rn(a.x, bz.x), 0.5), __dmul_rn(__dsub_rn(a.y, bz.y), 0.5));
    const double2 Bv = make_double2(__dmul_rn(__dadd_rn(a.y, bz.y), 0.5), __dmul_rn(__dsub_rn(bz.x, a.x), 0.5));
    const double P0 = __dmul_rn(__dadd_rn(__dmul_rn(A.x, A.x), __dmul_rn(A.y, A.y)), p.scale);
    const double P1 = __dmul_rn(__dadd_rn(__dmul_rn(Bv.x, Bv.x), __dmul_rn(Bv.y, Bv.y)), p.scale);
    const uint64_t row = ((k + p.H / 2) & (p.H - 1)) * p.W;
    io.rout[row + p.W / 2] = P0;  // column 0 -> centred column W/2
    io.rout[row] = P1;            // column W/2 -> centred column 0
    if (p.part) {
      if (k != 0) acc.add(P0);
      acc.add(P1);
    }
  }
}

// FFT_OUT_POWER_FFT middle step, in place in Xs: X -> |X|^2 (as (P, 0)); the packed column 0
// (sequence 0 when p.packed0) -> (|A|^2, |B|^2) with A, B the DC / Nyquist column spectra
// (A[k] = (U[k] + conj U[-k]) / 2, B[k] = -i (U[k] - conj U[-k]) / 2; both even in k).
template <int N>
__device__ __forceinline__ void power_in_place(const FftPass& p, double2* Xs, uint32_t tid, uint64_t seq,
                                               bool active) {
  constexpr int T = N < 16 ? 1 : N / 16;
  if (!active) return;
  for (uint32_t k = tid; k <= N / 2; k += T) {
    const uint32_t k2 = (N - k) & (N - 1);
    const double2 a = Xs[fft_pad(k)], bz = Xs[fft_pad(k2)];
    double2 va, vb;
    if (p.packed0 && seq == 0) {
      const double2 A = make_double2(__dmul_rn(__dadd_rn(a.x, bz.x), 0.5), __dmul_rn(__dsub_rn(a.y, bz.y), 0.5));
      const double2 Bv = make_double2(__dmul_rn(__dadd_rn(a.y, bz.y), 0.5), __dmul_rn(__dsub_rn(bz.x, a.x), 0.5));
      va = vb = make_double2(__dadd_rn(__dmul_rn(A.x, A.x), __dmul_rn(A.y, A.y)),
                             __dadd_rn(__dmul_rn(Bv.x, Bv.x), __dmul_rn(Bv.y, Bv.y)));
    } else {
      va = make_double2(__dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y)), 0.0);
      vb = make_double2(__dadd_rn(__dmul_rn(bz.x, bz.x), __dmul_rn(bz.y, bz.y)), 0.0);
    }
    Xs[fft_pad(k)] = va;
    Xs[fft_pad(k2)] = vb;
  }
}

// CTA = S sequences x T = N/16 threads (T = 1 when N < 16); rows: a sequence's threads are
// adjacent; columns: adjacent threads take adjacent columns (coalescing). Byte-input row passes
// first stage the CTA's rows (S N = 4096 bytes) in shared memory with one 16-byte load per thread.
template <int IN, int OUT, int LOGN, int CTA>
__global__ void __launch_bounds__(CTA, 512 / CTA)
    fft_pass_kernel(const FftPass p, const uint8_t* __restrict__ bytes, const double2* cin, double2* cout,
                    double* __restrict__ rout, const unsigned long long* __restrict__ sum, double* __restrict__ lag0) {
  constexpr int N = 1 << LOGN, T = N < 16 ? 1 : N / 16;
  extern __shared__ double2 fsm[];
  uint32_t s, tid;
  if (p.rows) { s = threadIdx.x / T; tid = threadIdx.x % T; }
  else { s = threadIdx.x & (p.S - 1); tid = threadIdx.x >> p.logS; }
  const uint64_t seq0 = (uint64_t)blockIdx.x * p.S, seq = seq0 + s;
  const bool active = s < p.S && tid < (uint32_t)T;  // (a CTA narrower than 256 threads leaves some idle)
  const bool valid = active && seq < p.nseq;
  double2* Xs = fsm + (size_t)(active ? s : 0) * p.pitch;
  __shared__ double2 tws[tw_entries<N>()];
  fill_twiddles<N>(tws, threadIdx.x, CTA);
  FftIo io{bytes, nullptr, seq0, cin, cout, rout, lag0, 0.0, tws, tws + kTwLo, nullptr, nullptr};
  if (IN == FFT_IN_CENTRED || IN == FFT_IN_PAIRS_CENTRED)
    io.mean = __ddiv_rn((double)*sum, (double)p.H * (double)p.W);
  if (OUT == FFT_OUT_REAL_PAIRS) {
    io.c0 = lag0_exact(sum, (uint64_t)p.H * p.W);
    io.inv_c0 = io.c0 > 0.0 ? __drcp_rn(io.c0) : 0.0;
  }
  if constexpr ((IN == FFT_IN_BYTES || IN == FFT_IN_CENTRED || IN == FFT_IN_PAIRS || IN == FFT_IN_PAIRS_CENTRED) &&
                N >= 16) {
    constexpr int BPE = (IN == FFT_IN_PAIRS || IN == FFT_IN_PAIRS_CENTRED) ? 2 : 1;  // bytes per element
    __shared__ uint4 stage[CTA * BPE];                // S N BPE = CTA * 16 * BPE bytes
    if (p.rows && p.in_pitch == (uint64_t)N * BPE && (reinterpret_cast<uintptr_t>(bytes) & 15) == 0) {
      const uint64_t rows = (p.nseq - seq0 < p.S) ? p.nseq - seq0 : p.S;
      const uint4* src = reinterpret_cast<const uint4*>(bytes + seq0 * N * BPE);
#pragma unroll
      for (int q = 0; q < BPE; ++q) {
        const uint32_t i = threadIdx.x + q * CTA;
        if ((uint64_t)i * 16 < rows * N * BPE) stage[i] = __ldg(src + i);
      }
      io.sb = reinterpret_cast<const uint8_t*>(stage);
    }
  }
  constexpr bool TW2 = OUT == FFT_OUT_R2C || IN == FFT_IN_C2R;
  __shared__ double2 tw2s[TW2 ? 64 + (2 * N > 64 ? 2 * N / 64 : 1) : 1];
  if (TW2)
    for (uint32_t i = threadIdx.x; i < 64 + (2 * N > 64 ? 2 * N / 64 : 0); i += CTA)
      if (i < 64) { if (i < 2u * N) tw2s[i] = twiddle_exact(i, 2 * N); }
      else tw2s[i] = twiddle_exact(64 * (i - 64), 2 * N);
  io.t2lo = tw2s;
  io.t2hi = tw2s + 64;
  __syncthreads();  // twiddle tables (and the staged bytes) visible to the CTA
  double2 a[16];
  FlatAcc fa;
  fft_passes<LOGN, 0, IN, OUT>(p, io, a, Xs, tid, seq, active, valid, fa, no_prefetch);
  if constexpr (OUT == FFT_OUT_POWER_FFT) {  // |.|^2 in shared memory, then the second transform
    power_in_place<N>(p, Xs, tid, seq, valid);
    __syncthreads();
    fft_passes<LOGN, 0, FFT_IN_COMPLEX, FFT_OUT_COMPLEX, true>(p, io, a, Xs, tid, seq, active, valid, fa,
                                                                no_prefetch);
  }
  if constexpr (OUT == FFT_OUT_R2C) r2c_epilogue<N>(p, io, Xs, tid, seq, valid, tw2s, tw2s + 64);
  if constexpr (OUT == FFT_OUT_HALF_SPECTRUM)
    if (seq0 == 0 && s == 0 && active) {
      if (p.col0_out) {  // four-step stage 2: U[k] of the packed column, k = pos kmul + blockIdx.y
        for (uint32_t k2 = tid; k2 < (uint32_t)N; k2 += T) p.col0_out[(uint64_t)k2 * p.kmul + blockIdx.y] = Xs[fft_pad(k2)];
      } else {
        half_col0_epilogue<N>(p, io, Xs, tid, fa);
      }
    }
  if ((OUT == FFT_OUT_SPECTRUM || OUT == FFT_OUT_HALF_SPECTRUM) && p.part) flat_partial<CTA>(fa, p.part);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// issue the asynchronous copy of tile `tile` (S sequences of the batch) into shared memory:
// complex input -> the padded exchange tile, bytes -> the 16-byte-per-thread stage
template <int IN, int N, int LOGN, int CTA>
__device__ __forceinline__ void fft_prefetch(const FftPass& p, const uint8_t* bytes, const double2* cin,
                                             double2* fsm, uint4* stage, uint64_t tile) {
  const uint64_t seq0 = tile * p.S;
  const uint32_t nS = (uint32_t)((p.nseq - seq0 < p.S) ? p.nseq - seq0 : p.S);
  if (IN == FFT_IN_COMPLEX) {
    for (uint32_t e = threadIdx.x; e < (p.S << LOGN); e += CTA) {
      const uint32_t s = p.rows ? e / N : e & (p.S - 1), idx = p.rows ? e % N : e >> p.logS;
      if (s >= nS) continue;
      const uint64_t g = p.rows ? (seq0 + s) * p.in_pitch + idx : (uint64_t)idx * p.in_pitch + seq0 + s;
      cp_async16(fsm + (size_t)s * p.pitch + fft_pad(idx), cin + g);
    }
  } else if ((uint64_t)threadIdx.x * 16 < (uint64_t)nS * N) {  // rows, pitch N, 16-byte aligned
    cp_async16(stage + threadIdx.x, bytes + seq0 * N + 16 * (uint64_t)threadIdx.x);
  }
  cp_async_commit();
}

// Persistent variant for n >= 1024: each CTA loops over tiles (grid = resident CTAs) and
// prefetches tile i+1 with cp.async while tile i's last pass computes and stores, so loads
// overlap compute even at one 512-thread CTA per SM. The first pass reads the prefetched tile.
template <int IN, int OUT, int LOGN, int CTA>
__global__ void __launch_bounds__(CTA, 512 / CTA)
    fft_persistent_kernel(const FftPass p, const uint8_t* __restrict__ bytes, const double2* cin, double2* cout,
                          double* __restrict__ rout, const unsigned long long* __restrict__ sum,
                          double* __restrict__ lag0) {
  constexpr int N = 1 << LOGN, T = N / 16;
  static_assert(N >= 256, "persistent FFT needs >= 2 passes");
  extern __shared__ double2 fsm[];
  __shared__ uint4 stage[CTA];
  __shared__ double2 tws[tw_entries<N>()];
  uint32_t s, tid;
  if (p.rows) { s = threadIdx.x / T; tid = threadIdx.x % T; }
  else { s = threadIdx.x & (p.S - 1); tid = threadIdx.x >> p.logS; }
  const bool active = s < p.S && tid < (uint32_t)T;
  double2* Xs = fsm + (size_t)(active ? s : 0) * p.pitch;
  const uint64_t tiles = (p.nseq + p.S - 1) / p.S;
  uint64_t tile = blockIdx.x;
  if (tile < tiles) fft_prefetch<IN, N, LOGN, CTA>(p, bytes, cin, fsm, stage, tile);
  fill_twiddles<N>(tws, threadIdx.x, CTA);
  FftIo io{bytes, reinterpret_cast<const uint8_t*>(stage), 0, cin, cout, rout, lag0, 0.0, tws, tws + kTwLo};
  if (IN == FFT_IN_CENTRED) io.mean = __ddiv_rn((double)*sum, (double)p.H * (double)p.W);
  double2 a[16];
  FlatAcc fa;
  for (; tile < tiles; tile += gridDim.x) {
    cp_async_wait_all();
    __syncthreads();  // the tile (and the twiddles) visible to the CTA
    io.seq0 = tile * p.S;
    const uint64_t seq = io.seq0 + s;
    const bool valid = active && seq < p.nseq;
    const uint64_t next = tile + gridDim.x;
    auto pre = [&]() {
      if (next < tiles) fft_prefetch<IN, N, LOGN, CTA>(p, bytes, cin, fsm, stage, next);
    };
    fft_passes<LOGN, 0, IN, OUT, true>(p, io, a, Xs, tid, seq, active, valid, fa, pre);
  }
  if (OUT == FFT_OUT_SPECTRUM && p.part) flat_partial<CTA>(fa, p.part);
}


// ---------------------------------------------------------------- TMA column transform
// The autocorrelation's fused column pass (FFT_OUT_POWER_FFT: transform, |.|^2, transform) for
// H = 4096 (2048) with the Tensor Memory Accelerator: one column per 256 (128)-thread CTA, two (four)
// CTAs per SM. The column is read row segment by row segment, 16 bytes per row; plain loads cost the
// LSU one L1 wavefront per row (a warp's 32 rows = 32 wavefronts: the LSU-bound 2-column kernel), TMA
// moves the same bytes without them. The tensor map views the workspace as H rows of 2 M doubles; a box is
// 256 rows x one column (2 doubles = 16 bytes), 4 KB landing unpadded (TMA destinations are 128-byte
// aligned) at tile offset 256 b, N/256 boxes per column completing on one mbarrier. The first pass
// reads the unpadded tile (FFT_IN_SMEM_DENSE) and the exchanges after it use the padded layout; the
// second transform's last pass writes the unpadded tile (FFT_OUT_SMEM) and the same boxes go back with
// TMA stores. The 32-byte sectors a column half-uses are completed from L2 by the neighbouring
// column's CTA, which runs beside it.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"(map), "r"(c0), "r"(c1), "r"(smem_u32(src)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra DONE;\n bra LAB_WAIT;\n DONE:\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

template <int LOGN>
__global__ void __launch_bounds__((1 << LOGN) / 16, 8192 / (1 << LOGN))
    fft_col_tma_kernel(const FftPass p, const __grid_constant__ CUtensorMap map) {
  constexpr int N = 1 << LOGN, T = N / 16, BOX = 256, NB = N / BOX;  // one column per T-thread CTA
  static_assert(N == 2048 || N == 4096, "TMA column pass: 2048 or 4096 rows");
  extern __shared__ __align__(128) double2 fsm_raw[];  // N + N/16 elements (padded exchanges) + 128 B of slack
  double2* fsm = reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(fsm_raw) + 127) & ~uintptr_t(127));
  __shared__ double2 tws[tw_entries<N>()];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t tid = threadIdx.x;
  const uint64_t seq = blockIdx.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (tid < 32) {  // warp 0 issues the column's N/BOX box loads
    if (tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(N * 16)
                   : "memory");
    if (tid < (uint32_t)NB) tma_load_2d(fsm + BOX * tid, &map, 2 * (int)seq, BOX * (int)tid, &bar);
  }
  fill_twiddles<N>(tws, tid, T);
  __syncthreads();  // twiddle tables
  mbar_wait(&bar, 0);
  FftIo io{nullptr, nullptr, seq, nullptr, nullptr, nullptr, nullptr, 0.0, tws, tws + kTwLo, nullptr, nullptr};
  double2 a[16];
  FlatAcc fa;
#ifndef LZ_TMA_FUSED_POWER
#define LZ_TMA_FUSED_POWER 1
#endif
  // H = 4096 (121 -> 114 us); at 2048 rows the fused form measured no faster and is not compiled
  if (seq == 0 || !LZ_TMA_FUSED_POWER || LOGN != 12) {  // packed DC / Nyquist column: |A|^2, |B|^2 need X[k], X[-k]
    fft_passes<LOGN, 0, FFT_IN_SMEM_DENSE, FFT_OUT_POWER_FFT, true>(p, io, a, fsm, tid, seq, true, true, fa,
                                                                    no_prefetch);
    power_in_place<N>(p, fsm, tid, seq, true);
    __syncthreads();
  } else {  // every other column: |X[k]|^2 elementwise, written by the last pass itself
    fft_passes<LOGN, 0, FFT_IN_SMEM_DENSE, FFT_OUT_POWER_SMEM, true>(p, io, a, fsm, tid, seq, true, true, fa,
                                                                     no_prefetch);
  }
  fft_passes<LOGN, 0, FFT_IN_COMPLEX, FFT_OUT_SMEM, true>(p, io, a, fsm, tid, seq, true, true, fa, no_prefetch);
  // (fft_pass ended with a barrier after the tile writes) generic-proxy writes -> the TMA engine
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (tid < 32) {
    if (tid < (uint32_t)NB) tma_store_2d(&map, 2 * (int)seq, BOX * (int)tid, fsm + BOX * tid);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the tile is read before the CTA exits
  }
}

// ---------------------------------------------------------------- four-step column transform
// The power spectrum's column transforms for H = 16 H2 (H = 2048, 4096): stage 1 below, then stage 2 =
// fft_pass_kernel<FFT_IN_COMPLEX, FFT_OUT_HALF_SPECTRUM, log2 H2> with ysplit (blockIdx.y = k1), then
// col0_unpack_kernel. With n = H2 n1 + n2 and k = k1 + 16 k2:
//   X[k1 + 16 k2] = sum_{n2} W_H2^{n2 k2} ( W_H^{n2 k1} sum_{n1<16} x[H2 n1 + n2] W_16^{n1 k1} ).
// Stage 1 does the 16-point DFTs and twiddles in registers, one thread per (n2, column), a warp covering
// 4 n2 x 8 adjacent columns (128-byte row segments), and writes y[k1] in place at row H2 k1 + n2 (it
// reads exactly the 16 elements it writes); stage 2 runs the H2-point transforms over H2 consecutive
// rows per k1, 16 columns per CTA, and writes P at rows k1 + 16 k2. The single-pass alternative moves
// 32-byte row segments of 2 columns and is bound by the LSU.
template <int LOGN>
__global__ void __launch_bounds__(256) fft_col_stage1_kernel(const FftPass p, double2* __restrict__ ws, unsigned* ctr) {
  constexpr int N = 1 << LOGN, N2 = N / 16;
  if (ctr && (blockIdx.x | blockIdx.y | threadIdx.x) == 0) *ctr = 0;  // col0_unpack_kernel's CTA counter
  __shared__ double2 tw[64 + N / 64];
  for (uint32_t i = threadIdx.x; i < 64 + N / 64; i += 256) tw[i] = twiddle_exact(i < 64 ? i : 64 * (i - 64), N);
  __syncthreads();
  const uint32_t c = threadIdx.x & 7, n2 = blockIdx.x * 32 + (threadIdx.x >> 3);
  const uint64_t col = (uint64_t)blockIdx.y * 8 + c;
  if (n2 >= (uint32_t)N2 || col >= p.nseq) return;
  double2 a[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) a[t] = ws[(uint64_t)(N2 * t + n2) * p.in_pitch + col];
  dft_dif<16>(a, 0);  // y_u in a[bitrev16(u)]
  auto tw_at = [&](uint32_t m) { return cmul(tw[m & 63], tw[64 + (m >> 6)]); };  // exp(-2 pi i m / N), m < N
  const double2 one = make_double2(1.0, 0.0);
  const double2 w1 = n2 ? tw_at(n2) : one, w2 = n2 ? tw_at(2 * n2) : one, w4 = n2 ? tw_at(4 * n2) : one;
  const double2 w8 = n2 ? tw_at(8 * n2) : one, w3 = cmul(w1, w2), w12 = cmul(w4, w8);
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    double2 v = a[bitrev_c<16>(u)];
    if (u) {
      const int lo = u & 3, hi = u & 12;
      const double2 wl = lo == 1 ? w1 : lo == 2 ? w2 : w3;
      const double2 wh = hi == 4 ? w4 : hi == 8 ? w8 : w12;
      v = cmul(v, lo == 0 ? wh : hi == 0 ? wl : cmul(wl, wh));
    }
    ws[(uint64_t)(N2 * u + n2) * p.in_pitch + col] = v;
  }
}

// The packed DC / Nyquist column after stage 2 (U[k] gathered from the 16 k1 blocks): the same
// unpacking as half_col0_epilogue; CTA b's flatness partial goes to part[b]. With flat != null the
// last CTA to finish (a counter stage 1 zeroed) combines all nparts partials from all_parts into the
// flatness (flatness_combine: the same order and bits as flatness_final_kernel, one launch fewer).
template <int CTA>
__global__ void __launch_bounds__(CTA) col0_unpack_kernel(const FftPass p, const double2* __restrict__ u,
                                                          double* __restrict__ rout, double2* part, unsigned* ctr,
                                                          const double2* all_parts, uint32_t nparts, uint64_t bins,
                                                          double* flat) {
  static_assert(CTA == kFftCta, "flatness_combine runs on this CTA");
  FlatAcc fa;
  const uint32_t N = p.H;
  for (uint32_t k = blockIdx.x * CTA + threadIdx.x; k < N; k += CTA * gridDim.x) {
    const double2 a = u[k], bz = u[(N - k) & (N - 1)];
    const double2 A = make_double2(__dmul_rn(__dadd_rn(a.x, bz.x), 0.5), __dmul_rn(__dsub_rn(a.y, bz.y), 0.5));
    const double2 Bv = make_double2(__dmul_rn(__dadd_rn(a.y, bz.y), 0.5), __dmul_rn(__dsub_rn(bz.x, a.x), 0.5));
    const double P0 = __dmul_rn(__dadd_rn(__dmul_rn(A.x, A.x), __dmul_rn(A.y, A.y)), p.scale);
    const double P1 = __dmul_rn(__dadd_rn(__dmul_rn(Bv.x, Bv.x), __dmul_rn(Bv.y, Bv.y)), p.scale);
    const uint64_t row = ((k + p.H / 2) & (p.H - 1)) * p.W;
    rout[row + p.W / 2] = P0;  // column 0 -> centred column W/2
    rout[row] = P1;            // column W/2 -> centred column 0
    if (part) {
      if (k != 0) fa.add(P0);
      fa.add(P1);
    }
  }
  if (part) flat_partial<CTA>(fa, part);
  if (flat) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
      __threadfence();  // this CTA's partial visible before it is counted
      last = atomicAdd(ctr, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      flatness_combine(all_parts, nparts, bins, flat);
    }
  }
}


// sum of the H*W bytes (the mean of the autocorrelation's centring; < 2^36, exact) in out[0] and
// the sum of their squares (< 2^44, exact) in out[2]
__global__ void __launch_bounds__(kFftCta) byte_sum_kernel(const uint8_t* __restrict__ x, uint64_t n,
                                                           unsigned long long* __restrict__ out) {
  unsigned long long acc = 0, acc2 = 0;
  const uint64_t t0 = (uint64_t)blockIdx.x * kFftCta + threadIdx.x, step = (uint64_t)gridDim.x * kFftCta;
  if ((reinterpret_cast<uintptr_t>(x) & 15) == 0 && n % 16 == 0) {  // 16 bytes per load, SAD / dp4a sums
#pragma unroll 4
    for (uint64_t i = t0; i < n / 16; i += step) {  // (unrolled: four independent 16-byte loads in flight)
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(x) + i);
      acc += __vsadu4(v.x, 0u) + __vsadu4(v.y, 0u) + __vsadu4(v.z, 0u) + __vsadu4(v.w, 0u);
      acc2 += __dp4a(v.x, v.x, 0u) + __dp4a(v.y, v.y, 0u) + __dp4a(v.z, v.z, 0u) + __dp4a(v.w, v.w, 0u);
    }
  } else {
    for (uint64_t i = t0; i < n; i += step) {
      acc += x[i];
      acc2 += (unsigned)x[i] * x[i];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
    acc2 += __shfl_xor_sync(0xffffffffu, acc2, o);
  }
  // the CTA's warps combined in shared memory, then one atomic per sum per CTA (one per warp queued
  // ~9,500 same-address atomics at L2 and took 10 us even when the bytes sat in L2)
  __shared__ unsigned long long red[2][kFftCta / 32];
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = acc;
    red[1][threadIdx.x >> 5] = acc2;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    unsigned long long t = 0;
#pragma unroll
    for (int w = 0; w < kFftCta / 32; ++w) t += red[threadIdx.x][w];
    if (t) atomicAdd(out + 2 * threadIdx.x, t);
  }
}

// r = c / c(0,0); a zero-variance input (c(0,0) = 0 exactly) gives the S:436 convention (Q25)
__global__ void __launch_bounds__(kFftCta) autocorr_normalise_kernel(double* __restrict__ r, uint64_t n,
                                                                     const double* __restrict__ lag0) {
  const double c0 = *lag0;
  const uint64_t t0 = (uint64_t)blockIdx.x * kFftCta + threadIdx.x, step = (uint64_t)gridDim.x * kFftCta;
  if (c0 != 0.0 && (reinterpret_cast<uintptr_t>(r) & 15) == 0 && n % 2 == 0) {  // 16-byte accesses
    double2* r2 = reinterpret_cast<double2*>(r);
    for (uint64_t i = t0; i < n / 2; i += step) {
      const double2 v = r2[i];
      r2[i] = make_double2(__ddiv_rn(v.x, c0), __ddiv_rn(v.y, c0));
    }
  } else {
    for (uint64_t i = t0; i < n; i += step) r[i] = c0 == 0.0 ? (i == 0 ? 1.0 : 0.0) : __ddiv_rn(r[i], c0);
  }
}

// spectral flatness: see flatness_combine
__global__ void __launch_bounds__(kFftCta) flatness_final_kernel(const double2* __restrict__ part, uint32_t nparts,
                                                                 uint64_t bins, double* __restrict__ out) {
  flatness_combine(part, nparts, bins, out);
}

}  // namespace lz
