// dist_kernels.cuh — device-side view of a cuppl_dist (fp32 parameters) and launchers.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/cuppl_gpu.h"

namespace cuppl {

struct DistArgs {
  int tag;
  int K;       // categorical size
  int ia, ib;  // uniform-discrete bounds [ia, ib)
  float p0, p1, p2;
  const uint64_t* table;
};

cudaError_t launch_dist_sample(const DistArgs& a, uint64_t key, uint32_t tag, uint64_t first_id,
                               uint64_t count, void* out, int sm_count, cudaStream_t stream);
cudaError_t launch_dist_score(const DistArgs& a, const void* x, uint64_t count, float* score,
                              int sm_count, cudaStream_t stream);
cudaError_t launch_philox_blocks(uint64_t key, uint64_t first_id, uint32_t block, uint32_t tag,
                                 uint64_t count, uint32_t* out, int sm_count, cudaStream_t stream);

}  // namespace cuppl
