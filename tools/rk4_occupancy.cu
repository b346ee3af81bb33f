// FP64-pipe utilisation of the cipher's integration loop versus resident warps per SM
// sub-partition (SMSP), for the canonical RK4 (43 DADD + 32 DMUL per step) and the NEXT-3
// FMA-formulated RK4 (7 DADD + 8 DMUL + 30 DFMA). The loop is lz::integrate<INTEG> of
// lorenz_device.cuh itself (the same inlined code the chain kernels run), without the
// per-character work around it, so this is the ceiling the chain kernels can reach at a given
// number of resident chains per SMSP.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 \
//          -o tools/rk4_occupancy tools/rk4_occupancy.cu
// Output: one JSON object on stdout.
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_1201_3114_b200/csrc/lorenz_device.cuh"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

// one lane = one trajectory; `reps` calls of integrate (C.n_it steps each), the state kept live
template <int INTEG>
__global__ void __launch_bounds__(1024, 1) occ_kernel(const lz::DevConst C, int reps, double* out, uint64_t lanes) {
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= lanes) return;
  double x = 1.0 + 1e-7 * (double)(g & 1023), y = 1.5, z = 20.0;
#pragma unroll 1
  for (int r = 0; r < reps; ++r) lz::integrate<INTEG>(x, y, z, C);
  out[g] = x + y + z;
}

template <int INTEG>
int run(const lz::DevConst& C, int reps, double* d, int sms, double peak, double ops_per_step, const char* name,
        bool first) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("%s\"%s\": [", first ? "" : ", ", name);
  // whole warps per SMSP (1 CTA of 128 w threads per SM), then the C3 and 100,000-block layouts of
  // the wave kernel (whole warps spread over the SMSPs unevenly)
  const double per_smsp[] = {1, 2, 3, 4, 5, 6, 8, 2048.0 / 592, 3125.0 / 592};
  for (int i = 0; i < 9; ++i) {
    uint64_t lanes;
    int cta, grid;
    if (i < 7) {
      cta = 128 * (int)per_smsp[i];
      grid = sms;
      lanes = (uint64_t)cta * grid;
    } else {
      cta = 128;
      lanes = (uint64_t)(per_smsp[i] * 592 * 32 + 0.5);
      grid = (int)((lanes + cta - 1) / cta);
    }
    occ_kernel<INTEG><<<grid, cta>>>(C, 1, d, lanes);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      occ_kernel<INTEG><<<grid, cta>>>(C, reps, d, lanes);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    const double ops = (double)lanes * reps * C.n_it * ops_per_step;
    printf("%s{\"warps_per_smsp\": %.3f, \"ms\": %.3f, \"pipe_frac\": %.4f}", i ? ", " : "", per_smsp[i], best,
           ops / (best * 1e-3) / peak);
  }
  printf("]");
  return 0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  const int sms = p.multiProcessorCount;
  const double peak = (double)sms * 64 * clk_khz * 1e3;  // FP64 lane-ops/s at the max SM clock
  lz::DevConst C{};
  volatile double three = 3.0, six = 6.0;
  C.sigma = 10.0;
  C.rho = 28.0;
  C.beta = 8.0 / three;
  C.h = 0.01;
  C.h2 = 0.005;
  C.h6 = 0.01 / six;
  C.n_it = 1000;
  double* d;
  CK(cudaMalloc(&d, sizeof(double) * 148 * 1024 * 2));
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_max_mhz\": %.0f, \"steps_per_lane\": %d, ", p.name, sms,
         clk_khz / 1e3, 40 * C.n_it);
  if (run<LORENZ_RK4>(C, 40, d, sms, peak, 75.0, "rk4", true)) return 1;
  if (run<LORENZ_RK4_FMA>(C, 40, d, sms, peak, 45.0, "rk4_fma", false)) return 1;
  if (run<LORENZ_EULER>(C, 40, d, sms, peak, 15.0, "euler", false)) return 1;
  printf("}\n");
  return 0;
}
