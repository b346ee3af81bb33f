// seg_launch.h — host entry of the balanced chain kernel (lorenz_device.cuh), defined in
// lorenz_seg.cu. That file is compiled once per OP (-DLZ_SEG_OP=0|1|2) so the three sets of
// kernel instantiations build in parallel (build.py).
#pragma once
#include <cuda_runtime.h>

#include "lorenz_device.cuh"

namespace lz {
// Stream-ordered allocation from the library's own per-device pool (lorenz.cu); free with
// cudaFreeAsync.
cudaError_t lib_malloc_async(void** p, size_t bytes, cudaStream_t st);

// Enqueue one balanced launch on `st`: a pool allocation for the hand-over scratch, a memset of
// its ticket and flags, the kernel (one CTA of `cta` threads per SM), the free. Returns
// cudaErrorNotReady (nothing enqueued) when the scratch cannot be allocated: take the wave kernel.
template <int OP>
cudaError_t launch_seg_op(const DevConst& C, const SegPlan& P, int cta, uint32_t integrator, const DevKey& K,
                          const DevKey* Kb, const uint8_t* in, uint8_t* out, lorenz_result* res, uint8_t* tags,
                          uint8_t* block_ok, cudaStream_t st);
}  // namespace lz
