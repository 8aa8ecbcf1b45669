// saw_walk_mma_plain.cu -- explicit instantiations of the plain K1t kernels of one q-tile (MODE 0; 8 / 10 / any k-steps)
// (saw_walk_mma.cuh; split over translation units for a parallel build).
#include "saw_walk_mma.cuh"

namespace labs_b200 {
template __global__ void saw_walk_mma_kernel<1, 0, true, 0>(WalkParams, int*, int*);
template __global__ void saw_walk_mma_kernel<1, 0, true, 8>(WalkParams, int*, int*);
template __global__ void saw_walk_mma_kernel<1, 0, true, 10>(WalkParams, int*, int*);
template __global__ void saw_walk_mma_kernel<1, 0, false, 0>(WalkParams, int*, int*);
template __global__ void saw_walk_mma_kernel<1, 0, false, 8>(WalkParams, int*, int*);
template __global__ void saw_walk_mma_kernel<1, 0, false, 10>(WalkParams, int*, int*);
}  // namespace labs_b200
