// saw_walk_mma_q2.cu -- explicit instantiations of the K1t kernels of two q-tiles
// (saw_walk_mma.cuh; split over translation units for a parallel build).
#include "saw_walk_mma.cuh"

namespace labs_b200 {
template __global__ void saw_walk_mma_kernel<2, 0, true, 0>(WalkParams, int*, int*);
template __global__ void saw_walk_mma_kernel<2, 0, false, 0>(WalkParams, int*, int*);
template __global__ void saw_walk_mma_kernel<2, 1, true, 0>(WalkParams, int*, int*);
template __global__ void saw_walk_mma_kernel<2, 1, false, 0>(WalkParams, int*, int*);
template __global__ void saw_walk_mma_kernel<2, 2, true, 0>(WalkParams, int*, int*);
template __global__ void saw_walk_mma_kernel<2, 2, false, 0>(WalkParams, int*, int*);
}  // namespace labs_b200
