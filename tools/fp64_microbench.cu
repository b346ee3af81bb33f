// FP64-pipe microbenchmark for B200 (sm_100a): peak DADD/DMUL issue rate,
// dependent-op latency, and the number of resident warps needed to saturate
// the pipe with a 3-way-ILP dependent chain (the shape of the Lorenz RK4 loop).
// MEASURED_PEAKS.json carries no FP64 figure, so the roofline denominator for
// the cipher kernel (SURVEY.md §8d "Roofline") comes from this program.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o fp64_microbench fp64_microbench.cu
// Output: one JSON object on stdout.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}

// 8 independent accumulators per thread; half DADD, half DMUL.
template <int ITERS>
__global__ void __launch_bounds__(256) peak_kernel(double* out, double a, double m,
                                                   unsigned long long* clk, unsigned long long* ns) {
  double r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  uint64_t c0 = clock64(), t0 = gtimer();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      r[i] = __dadd_rn(r[i], a);
      r[i + 1] = __dmul_rn(r[i + 1], m);
    }
  }
  uint64_t c1 = clock64(), t1 = gtimer();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s = __dadd_rn(s, r[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) { *clk = c1 - c0; *ns = t1 - t0; }
}

// One dependent chain: latency in cycles of DADD (mode 0) or DMUL (mode 1).
__global__ void lat_kernel(double* out, double a, int n, int mode, unsigned long long* clk) {
  double x = out[0];
  uint64_t c0 = clock64();
  if (mode == 0) { for (int i = 0; i < n; ++i) x = __dadd_rn(x, a); }
  else           { for (int i = 0; i < n; ++i) x = __dmul_rn(x, a); }
  uint64_t c1 = clock64();
  out[1] = x;
  *clk = c1 - c0;
}

// 3-way ILP chain, depth ~6 per "step", 18 ops per step: throughput versus
// resident warps. Each thread: s = (x,y,z); step: x=x*a+y.. without FMA.
__global__ void ilp3_kernel(double* out, int steps, double a, double b, int active = 32) {
  if ((int)(threadIdx.x & 31) >= active) return;  // partially filled warps (half-warp issue test)
  double x = 1.0 + threadIdx.x * 1e-9, y = 2.0, z = 3.0;
  for (int i = 0; i < steps; ++i) {
    double tx = __dmul_rn(x, a), ty = __dmul_rn(y, a), tz = __dmul_rn(z, a);
    tx = __dadd_rn(tx, b); ty = __dadd_rn(ty, b); tz = __dadd_rn(tz, b);
    double ux = __dmul_rn(tx, a), uy = __dmul_rn(ty, a), uz = __dmul_rn(tz, a);
    ux = __dadd_rn(ux, b); uy = __dadd_rn(uy, b); uz = __dadd_rn(uz, b);
    x = __dadd_rn(__dmul_rn(ux, a), b); y = __dadd_rn(__dmul_rn(uy, a), b); z = __dadd_rn(__dmul_rn(uz, a), b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x + y + z;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  double* d; unsigned long long *clk, *ns;
  CK(cudaMalloc(&d, sizeof(double) * 148 * 64 * 2048));
  CK(cudaMalloc(&clk, 8)); CK(cudaMalloc(&ns, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);

  // ---- peak: 8 CTAs x 256 threads per SM (full 2048 threads) ----
  const int ITERS = 20000;
  int grid = sms * 8;
  peak_kernel<ITERS><<<grid, 256>>>(d, 1e-12, 1.0000001, clk, ns);
  CK(cudaDeviceSynchronize());
  float best = 1e30f; unsigned long long hc = 0, hn = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    peak_kernel<ITERS><<<grid, 256>>>(d, 1e-12, 1.0000001, clk, ns);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) { best = ms; cudaMemcpy(&hc, clk, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&hn, ns, 8, cudaMemcpyDeviceToHost); }
  }
  double ops = (double)grid * 256 * ITERS * 8;
  double rate = ops / (best * 1e-3);
  double mhz = (double)hc / (double)hn * 1e3;
  double per_clk_sm = rate / (sms * mhz * 1e6);

  // ---- latency ----
  unsigned long long lc[2];
  for (int m = 0; m < 2; ++m) {
    lat_kernel<<<1, 1>>>(d, 1.0000001, 4096, m, clk); CK(cudaDeviceSynchronize());
    lat_kernel<<<1, 1>>>(d, 1.0000001, 4096, m, clk); CK(cudaDeviceSynchronize());
    cudaMemcpy(&lc[m], clk, 8, cudaMemcpyDeviceToHost);
  }

  // ---- occupancy sweep for a 3-way ILP chain (18 ops/step) ----
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"peak_kernel_ms\": %.3f, \"fp64_lane_ops_per_s\": %.4e, "
         "\"sm_mhz_in_kernel\": %.1f, \"fp64_lane_ops_per_clk_per_sm\": %.2f, "
         "\"dadd_latency_cyc\": %.2f, \"dmul_latency_cyc\": %.2f, \"ilp3_sweep\": [",
         p.name, sms, best, rate, mhz, per_clk_sm, lc[0] / 4096.0, lc[1] / 4096.0);
  const int STEPS = 4000;
  int warps_list[] = {4, 8, 12, 16, 24, 32, 48, 64};
  for (int wi = 0; wi < 8; ++wi) {
    int wps = warps_list[wi];   // warps per SM
    int g = sms * wps / 4;      // CTAs of 128 threads
    ilp3_kernel<<<g, 128>>>(d, STEPS, 1.0000001, 1e-12); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    ilp3_kernel<<<g, 128>>>(d, STEPS, 1.0000001, 1e-12);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double o = (double)g * 128 * STEPS * 18;
    printf("%s{\"warps_per_sm\": %d, \"ms\": %.3f, \"lane_ops_per_s\": %.4e, \"frac_of_peak\": %.3f}",
           wi ? ", " : "", wps, ms, o / (ms * 1e-3), o / (ms * 1e-3) / rate);
  }
  printf("], \"active_lanes_sweep\": [");
  // same warps (16/SM), fewer active lanes: does a 16-lane warp cost one FP64 pipe cycle or two?
  int act_list[] = {32, 24, 17, 16, 8, 1};
  for (int ai = 0; ai < 6; ++ai) {
    int g = sms * 16 / 4;
    ilp3_kernel<<<g, 128>>>(d, STEPS, 1.0000001, 1e-12, act_list[ai]); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    ilp3_kernel<<<g, 128>>>(d, STEPS, 1.0000001, 1e-12, act_list[ai]);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%s{\"active_lanes\": %d, \"warps_per_sm\": 16, \"ms\": %.3f}", ai ? ", " : "", act_list[ai], ms);
  }
  printf("]}\n");
  return 0;
}
