// saw_walk_mma_checked.cu -- explicit instantiations of the checked and counting K1t kernels of one q-tile (MODE 1, 2)
// (saw_walk_mma.cuh; split over translation units for a parallel build).
#include "saw_walk_mma.cuh"

namespace labs_b200 {
template __global__ void saw_walk_mma_kernel<1, 1, true, 0>(WalkParams, int*, int*);
template __global__ void saw_walk_mma_kernel<1, 1, false, 0>(WalkParams, int*, int*);
template __global__ void saw_walk_mma_kernel<1, 2, true, 0>(WalkParams, int*, int*);
template __global__ void saw_walk_mma_kernel<1, 2, false, 0>(WalkParams, int*, int*);
}  // namespace labs_b200
