// lorenz_seg.cu — host launch of the balanced chain kernel for one OP (LZ_SEG_OP: 0 encrypt,
// 1 decrypt, 2 verify), all integrators and CTA sizes. See seg_launch.h and DESIGN.md §4.
#include <cuda_runtime.h>

#include "../../include/lorenz.h"
#include "lorenz_device.cuh"
#include "seg_launch.h"

#ifndef LZ_SEG_OP
#error "compile once per OP with -DLZ_SEG_OP=0|1|2 (build.py does)"
#endif

namespace lz {
namespace {

template <int OP, int INTEG, int CTA>
cudaError_t launch_seg(const DevConst& C, const SegPlan& P, const DevKey& K, const DevKey* Kb,
                       const uint8_t* in, uint8_t* out, lorenz_result* res, uint8_t* tags, uint8_t* block_ok,
                       cudaStream_t st) {
  const size_t hdr = (4 * ((size_t)P.slots + 2) + 15) & ~(size_t)15;  // ticket + S + 1 flags
  const size_t bytes = hdr + ((size_t)P.slots + 1) * kSegWords * 32 * 8;
  uint8_t* scr = nullptr;
  cudaError_t e = lib_malloc_async(reinterpret_cast<void**>(&scr), bytes, st);
  if (e == cudaErrorMemoryAllocation) {  // no room for the hand-over scratch: take the wave kernel
    (void)cudaGetLastError();
    return cudaErrorNotReady;
  }
  if (e != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(scr, 0, hdr, st)) == cudaSuccess) {
    uint32_t* ticket = reinterpret_cast<uint32_t*>(scr);
    const unsigned grid = (unsigned)((P.slots + CTA / 32 - 1) / (CTA / 32));
    lorenz_chain_seg_kernel<OP, INTEG, CTA><<<grid, CTA, 0, st>>>(
        C, K, Kb, in, out, res, tags, block_ok, P, ticket, ticket + 1, reinterpret_cast<uint64_t*>(scr + hdr));
    e = cudaGetLastError();
  }
  const cudaError_t f = cudaFreeAsync(scr, st);
  return e != cudaSuccess ? e : f;
}

template <int OP, int INTEG>
cudaError_t launch_seg_cta(const DevConst& C, const SegPlan& P, int cta, const DevKey& K, const DevKey* Kb,
                           const uint8_t* in, uint8_t* out, lorenz_result* res, uint8_t* tags, uint8_t* block_ok,
                           cudaStream_t st) {
  return cta == 512   ? launch_seg<OP, INTEG, 512>(C, P, K, Kb, in, out, res, tags, block_ok, st)
         : cta == 384 ? launch_seg<OP, INTEG, 384>(C, P, K, Kb, in, out, res, tags, block_ok, st)
                      : launch_seg<OP, INTEG, 256>(C, P, K, Kb, in, out, res, tags, block_ok, st);
}

}  // namespace

template <int OP>
cudaError_t launch_seg_op(const DevConst& C, const SegPlan& P, int cta, uint32_t integrator, const DevKey& K,
                          const DevKey* Kb, const uint8_t* in, uint8_t* out, lorenz_result* res, uint8_t* tags,
                          uint8_t* block_ok, cudaStream_t st) {
  return integrator == LORENZ_EULER
             ? launch_seg_cta<OP, LORENZ_EULER>(C, P, cta, K, Kb, in, out, res, tags, block_ok, st)
         : integrator == LORENZ_RK4_FMA
             ? launch_seg_cta<OP, LORENZ_RK4_FMA>(C, P, cta, K, Kb, in, out, res, tags, block_ok, st)
             : launch_seg_cta<OP, LORENZ_RK4>(C, P, cta, K, Kb, in, out, res, tags, block_ok, st);
}

template cudaError_t launch_seg_op<LZ_SEG_OP>(const DevConst&, const SegPlan&, int, uint32_t, const DevKey&,
                                              const DevKey*, const uint8_t*, uint8_t*, lorenz_result*, uint8_t*,
                                              uint8_t*, cudaStream_t);

}  // namespace lz

#if defined(LZ_SEG_TRACE) && LZ_SEG_OP == 0
// Tuning builds only (tools/seg_trace.py, encrypt launches): copy the per-slot timeline (4096 x 8
// u64) out, then zero it (slots with no work record nothing, so rows of an earlier launch would
// otherwise survive).
extern "C" int lorenz_debug_seg_trace(unsigned long long* host) {
  if (cudaMemcpyFromSymbol(host, lz::g_seg_trace, sizeof lz::g_seg_trace) != cudaSuccess) return 1;
  static unsigned long long zeros[4096 * 8];
  return cudaMemcpyToSymbol(lz::g_seg_trace, zeros, sizeof zeros) == cudaSuccess ? 0 : 1;
}
#endif
