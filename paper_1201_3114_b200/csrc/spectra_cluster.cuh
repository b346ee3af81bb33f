// spectra_cluster.cuh — the column pass of the large 2-D transforms (H = 4 M rows, M = 512 or
// 1024) as one 4-CTA thread-block cluster per group of COLS adjacent packed columns (NEXT-4,
// Figs. 3-4).
//
// Why a cluster: an FP64 complex column of 4096 points is 64 KB, so one SM holds at most two of
// them and the single-CTA column pass (spectra.cuh) reads and writes 32-byte row segments at a
// 32 KiB stride — 16 L1 wavefronts per warp access, and the LSU, not HBM, set its speed
// (long-scoreboard and lg-throttle stalls, 1.6 TB/s). Here the four CTAs of a cluster split the
// rows instead: CTA r holds rows [r M, (r+1) M) of COLS columns (COLS x 16 B = 128-byte row
// segments at COLS = 8), and the transform is the four-step split N = 4 x M:
//
//   DIF (forward):  X[r + 4 k2] = FFT_M( W_N^{n2 r} sum_{n1<4} x[n1 M + n2] W_4^{n1 r} )[k2]
//     -> the radix-4 step reads the same (column, n2) element of all four CTAs' shared memory
//        (distributed shared memory), then each CTA runs M-point FFTs of its own residue class;
//   DIT (the autocorrelation's second transform, input in that residue layout):
//     X2[m1 + M m2] = sum_{r<4} W_4^{r m2} (W_N^{r m1} FFT_M(P[r + 4 k2])[m1])
//     -> M-point FFTs first, twiddle, then the radix-4 step across the cluster, CTA m2 writing
//        rows [m2 M, (m2+1) M) contiguously.
//
// The packed DC / Nyquist column (sequence 0) pairs U[k] with U[-k], which lives in CTA (4-r) & 3:
// read across the cluster as well. Same arithmetic as the single-CTA pass (FMA complex products
// at the same sites, the same twiddle tables), within the bounds of §2e.
#pragma once
#include <cooperative_groups.h>

#include "spectra.cuh"

namespace lz {

namespace cg = cooperative_groups;

constexpr int kClusterRanks = 4;

template <int COLS>
__host__ __device__ constexpr int log2c() {
  return COLS <= 1 ? 0 : 1 + log2c<COLS / 2>();
}

// Local plan of the cluster column pass: M-point column FFTs, COLS sequences per CTA.
inline FftPass fft_plan_cluster(uint32_t M, uint32_t LM, uint32_t nseq, uint32_t cols) {
  FftPass p = fft_plan(M, LM, nseq, false);
  p.S = cols;
  p.logS = 0;
  while ((1u << p.logS) < cols) ++p.logS;
  const uint32_t k = cols < 8 ? cols : 8;  // sequences one 8-thread shared-memory phase touches
  p.pitch = M + M / 16;
  if (k > 1) p.pitch += ((8 / k) - p.pitch % 8 + 8) % 8;
  p.kmul = kClusterRanks;
  return p;
}
inline size_t fft_cluster_smem_bytes(const FftPass& p) { return (size_t)p.S * p.pitch * sizeof(double2); }

// sum_{n1<4} x_{n1} W_4^{n1 r}, W_4 = exp(-2 pi i / 4) = -i; r is CTA-uniform
__device__ __forceinline__ double2 radix4_row(double2 x0, double2 x1, double2 x2, double2 x3, uint32_t r) {
  const double2 s02 = cadd(x0, x2), d02 = csub(x0, x2), s13 = cadd(x1, x3), d13 = csub(x1, x3);
  if (r == 0) return cadd(s02, s13);
  if (r == 2) return csub(s02, s13);
  if (r == 1) return make_double2(__dadd_rn(d02.x, d13.y), __dsub_rn(d02.y, d13.x));  // d02 - i d13
  return make_double2(__dsub_rn(d02.x, d13.y), __dadd_rn(d02.y, d13.x));              // d02 + i d13
}

// 32-bit shared::cluster address of `smem` in the CTA of cluster rank `rank` (mapa), and a 16-byte
// load from such an address: one register per address instead of a 64-bit generic pointer
__device__ __forceinline__ uint32_t cluster_base(const void* smem, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"((uint32_t)__cvta_generic_to_shared(smem)), "r"(rank));
  return out;
}
__device__ __forceinline__ double2 ld_cluster(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
  return v;
}

// exp(-2 pi i m / N) from the N-point tables (m < N)
template <int N>
__device__ __forceinline__ double2 twN(const double2* lo, const double2* hi, uint32_t m) {
  return N <= 64 ? lo[m] : cmul(lo[m & 63], hi[m >> 6]);
}

// OUT: FFT_OUT_HALF_SPECTRUM (power spectrum: P at (k, j) and (-k, W - j), the packed column 0
// unpacked) or FFT_OUT_POWER_FFT (autocorrelation: transform, |.|^2, transform, in place).
// LOGN = log2 H; grid = 4 x (packed columns / COLS); CTA = COLS x M / 16 threads.
template <int OUT, int LOGN, int COLS>
__global__ void __cluster_dims__(kClusterRanks, 1, 1) __launch_bounds__(COLS * (1 << (LOGN - 2)) / 16, 1)
    fft_col_cluster_kernel(const FftPass p, const double2* cin, double2* cout, double* __restrict__ rout) {
  constexpr int N = 1 << LOGN, LM = LOGN - 2, M = 1 << LM, T = M / 16, CTA = T * COLS, LC = log2c<COLS>();
  constexpr int PER = M * COLS / CTA;  // elements per thread in the element-wise steps (16)
  static_assert(OUT == FFT_OUT_HALF_SPECTRUM || OUT == FFT_OUT_POWER_FFT, "cluster column modes");
  static_assert(PER == 16 && M >= 256, "M-point local transforms of 16 elements per thread");
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t r = cluster.block_rank();
  const uint64_t col0 = (uint64_t)(blockIdx.x / kClusterRanks) * COLS;
  extern __shared__ double2 fsm[];
  __shared__ double2 twm[64 + M / 64];   // M-point twiddles of the local passes
  __shared__ double2 twn[64 + N / 64];   // N-point twiddles of the four-step split
  for (uint32_t i = threadIdx.x; i < 64 + M / 64; i += CTA) twm[i] = twiddle_exact(i < 64 ? i : 64 * (i - 64), M);
  for (uint32_t i = threadIdx.x; i < 64 + N / 64; i += CTA) twn[i] = twiddle_exact(i < 64 ? i : 64 * (i - 64), N);

  // ---- load rows [r M, (r+1) M) of the group's columns: COLS x 16 B contiguous per row ----
  {
    double2 v[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const uint32_t e = threadIdx.x + q * CTA, row = e >> LC, c = e & (COLS - 1);
      v[q] = cin[(uint64_t)(r * M + row) * p.in_pitch + col0 + c];
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const uint32_t e = threadIdx.x + q * CTA, row = e >> LC, c = e & (COLS - 1);
      fsm[c * p.pitch + fft_pad(row)] = v[q];
    }
  }
  cluster.sync();  // every CTA's rows are in place (and the twiddle tables)

  // ---- DIF radix-4 step across the cluster: y = W_N^{n2 r} sum_n1 x_{n1} W_4^{n1 r} ----
  // In two halves of 8 elements per thread (register pressure): every CTA reads half h of all four
  // tiles, the cluster synchronises, each CTA overwrites half h of its own tile, and so on — half
  // 1's positions are never written before every CTA has read them.
  {
    uint32_t xb[kClusterRanks];
#pragma unroll
    for (int k = 0; k < kClusterRanks; ++k) xb[k] = cluster_base(fsm, k);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double2 y[PER / 2];
#pragma unroll
      for (int q = 0; q < PER / 2; ++q) {
        const uint32_t e = threadIdx.x + (h * PER / 2 + q) * CTA, n2 = e >> LC, c = e & (COLS - 1);
        const uint32_t off = c * p.pitch + fft_pad(n2), bo = off * (uint32_t)sizeof(double2);
        const double2 t = radix4_row(ld_cluster(xb[0] + bo), ld_cluster(xb[1] + bo), ld_cluster(xb[2] + bo),
                                     ld_cluster(xb[3] + bo), r);
        y[q] = (r == 0 || n2 == 0) ? t : cmul(t, twN<N>(twn, twn + 64, n2 * r));
      }
      cluster.sync();  // every CTA has read half h of the others' tiles
#pragma unroll
      for (int q = 0; q < PER / 2; ++q) {
        const uint32_t e = threadIdx.x + (h * PER / 2 + q) * CTA, n2 = e >> LC, c = e & (COLS - 1);
        fsm[c * p.pitch + fft_pad(n2)] = y[q];
      }
    }
  }
  __syncthreads();

  // ---- M-point transforms of this CTA's residue class, k = r + 4 k2 ----
  const uint32_t s = threadIdx.x & (COLS - 1), tid = threadIdx.x >> LC;
  double2* Xs = fsm + (size_t)s * p.pitch;
  const uint64_t seq = col0 + s;
  FftPass q = p;
  q.kadd = r;
  FftIo io{nullptr, nullptr, col0, cin, cout, rout, nullptr, 0.0, twm, twm + 64, nullptr, nullptr};
  double2 a[16];
  FlatAcc fa;
  const bool col0_group = col0 == 0;  // the packed DC / Nyquist column is sequence 0 of group 0
  if constexpr (OUT == FFT_OUT_HALF_SPECTRUM) {
    fft_passes<LM, 0, FFT_IN_COMPLEX, FFT_OUT_HALF_SPECTRUM, true>(q, io, a, Xs, tid, seq, true, true, fa,
                                                                    no_prefetch);
    if (col0_group) {  // cluster-uniform: U[k] here, U[-k] in CTA (4 - r) & 3
      cluster.sync();
      const uint32_t rp = (kClusterRanks - r) & (kClusterRanks - 1);
      const double2* up = cluster.map_shared_rank(fsm, rp);  // sequence 0 of the partner
      for (uint32_t k2 = threadIdx.x; k2 < (uint32_t)M; k2 += CTA) {
        const uint32_t k2p = r == 0 ? (M - k2) & (M - 1) : M - 1 - k2;
        const double2 av = fsm[fft_pad(k2)], bz = up[fft_pad(k2p)];
        const double2 A = make_double2(__dmul_rn(__dadd_rn(av.x, bz.x), 0.5), __dmul_rn(__dsub_rn(av.y, bz.y), 0.5));
        const double2 Bv = make_double2(__dmul_rn(__dadd_rn(av.y, bz.y), 0.5), __dmul_rn(__dsub_rn(bz.x, av.x), 0.5));
        const double P0 = __dmul_rn(__dadd_rn(__dmul_rn(A.x, A.x), __dmul_rn(A.y, A.y)), p.scale);
        const double P1 = __dmul_rn(__dadd_rn(__dmul_rn(Bv.x, Bv.x), __dmul_rn(Bv.y, Bv.y)), p.scale);
        const uint64_t k = (uint64_t)r + kClusterRanks * (uint64_t)k2;
        const uint64_t row = ((k + p.H / 2) & (p.H - 1)) * p.W;
        rout[row + p.W / 2] = P0;  // column 0 -> centred column W/2
        rout[row] = P1;            // column W/2 -> centred column 0
        if (p.part) {
          if (k != 0) fa.add(P0);
          fa.add(P1);
        }
      }
      cluster.sync();  // the partner has read this CTA's column 0
    }
    if (p.part) flat_partial<CTA>(fa, p.part);
  } else {
    fft_passes<LM, 0, FFT_IN_COMPLEX, FFT_OUT_SMEM, true>(q, io, a, Xs, tid, seq, true, true, fa, no_prefetch);
    // |X|^2 in place; the packed column 0 -> (|A|^2, |B|^2) with U[-k] from the partner CTA
    {
      double2 w[PER];
      if (col0_group) cluster.sync();  // partners' transforms done before their column 0 is read
      const uint32_t rp = (kClusterRanks - r) & (kClusterRanks - 1);
      const double2* up = cluster.map_shared_rank(fsm, rp);
#pragma unroll
      for (int qq = 0; qq < PER; ++qq) {
        const uint32_t e = threadIdx.x + qq * CTA, k2 = e >> LC, c = e & (COLS - 1);
        const double2 av = fsm[c * p.pitch + fft_pad(k2)];
        if (col0_group && c == 0 && p.packed0) {
          const uint32_t k2p = r == 0 ? (M - k2) & (M - 1) : M - 1 - k2;
          const double2 bz = up[fft_pad(k2p)];
          const double2 A = make_double2(__dmul_rn(__dadd_rn(av.x, bz.x), 0.5), __dmul_rn(__dsub_rn(av.y, bz.y), 0.5));
          const double2 Bv = make_double2(__dmul_rn(__dadd_rn(av.y, bz.y), 0.5), __dmul_rn(__dsub_rn(bz.x, av.x), 0.5));
          w[qq] = make_double2(__dadd_rn(__dmul_rn(A.x, A.x), __dmul_rn(A.y, A.y)),
                               __dadd_rn(__dmul_rn(Bv.x, Bv.x), __dmul_rn(Bv.y, Bv.y)));
        } else {
          w[qq] = make_double2(__dadd_rn(__dmul_rn(av.x, av.x), __dmul_rn(av.y, av.y)), 0.0);
        }
      }
      if (col0_group) cluster.sync();  // the partner has read this CTA's column 0
      else __syncthreads();
#pragma unroll
      for (int qq = 0; qq < PER; ++qq) {
        const uint32_t e = threadIdx.x + qq * CTA, k2 = e >> LC, c = e & (COLS - 1);
        fsm[c * p.pitch + fft_pad(k2)] = w[qq];
      }
    }
    __syncthreads();
    // DIT: M-point transforms over k2, twiddle W_N^{r m1}, radix-4 across the cluster
    fft_passes<LM, 0, FFT_IN_COMPLEX, FFT_OUT_SMEM, true>(q, io, a, Xs, tid, seq, true, true, fa, no_prefetch);
#pragma unroll
    for (int qq = 0; qq < PER; ++qq) {
      const uint32_t e = threadIdx.x + qq * CTA, m1 = e >> LC, c = e & (COLS - 1);
      if (r != 0 && m1 != 0) {
        double2& v = fsm[c * p.pitch + fft_pad(m1)];
        v = cmul(v, twN<N>(twn, twn + 64, m1 * r));
      }
    }
    cluster.sync();
    uint32_t xb[kClusterRanks];
#pragma unroll
    for (int k = 0; k < kClusterRanks; ++k) xb[k] = cluster_base(fsm, k);
#pragma unroll
    for (int qq = 0; qq < PER; ++qq) {
      const uint32_t e = threadIdx.x + qq * CTA, m1 = e >> LC, c = e & (COLS - 1);
      const uint32_t bo = (c * p.pitch + fft_pad(m1)) * (uint32_t)sizeof(double2);
      cout[(uint64_t)(r * M + m1) * p.out_pitch + col0 + c] =
          radix4_row(ld_cluster(xb[0] + bo), ld_cluster(xb[1] + bo), ld_cluster(xb[2] + bo), ld_cluster(xb[3] + bo), r);
    }
    cluster.sync();  // nobody leaves while a partner still reads its tile
  }
}

}  // namespace lz
