// saw_walk.h -- declarations of the per-R K1 launchers (definitions: saw_walk.cuh,
// explicit instantiations: saw_walk_r*.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "saw_device.h"

namespace labs_b200 {
template <int R, int LPW>
cudaError_t launch_walk_fixed(const WalkParams& P, int grid, size_t smem, cudaStream_t st,
                              int* score_out, int* corr_out, bool count);
template <int R, int LPW>
int blocks_per_sm_fixed(const WalkParams& P, size_t smem);
}  // namespace labs_b200
