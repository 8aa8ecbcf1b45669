// saw_walk_mma.cu -- launchers of K1t (tensor-core G, saw_walk_mma.cuh): 1 or 2 q-tiles.
// The kernels are instantiated in saw_walk_mma_{plain,checked,q2}.cu (parallel build).
#include "saw_walk_mma.cuh"

namespace labs_b200 {
extern template __global__ void saw_walk_mma_kernel<1, 0, true, 0>(WalkParams, int*, int*);
extern template __global__ void saw_walk_mma_kernel<1, 0, true, 8>(WalkParams, int*, int*);
extern template __global__ void saw_walk_mma_kernel<1, 0, true, 10>(WalkParams, int*, int*);
extern template __global__ void saw_walk_mma_kernel<1, 0, false, 0>(WalkParams, int*, int*);
extern template __global__ void saw_walk_mma_kernel<1, 0, false, 8>(WalkParams, int*, int*);
extern template __global__ void saw_walk_mma_kernel<1, 0, false, 10>(WalkParams, int*, int*);
extern template __global__ void saw_walk_mma_kernel<1, 1, true, 0>(WalkParams, int*, int*);
extern template __global__ void saw_walk_mma_kernel<1, 1, false, 0>(WalkParams, int*, int*);
extern template __global__ void saw_walk_mma_kernel<1, 2, true, 0>(WalkParams, int*, int*);
extern template __global__ void saw_walk_mma_kernel<1, 2, false, 0>(WalkParams, int*, int*);
extern template __global__ void saw_walk_mma_kernel<2, 0, true, 0>(WalkParams, int*, int*);
extern template __global__ void saw_walk_mma_kernel<2, 0, false, 0>(WalkParams, int*, int*);
extern template __global__ void saw_walk_mma_kernel<2, 1, true, 0>(WalkParams, int*, int*);
extern template __global__ void saw_walk_mma_kernel<2, 1, false, 0>(WalkParams, int*, int*);
extern template __global__ void saw_walk_mma_kernel<2, 2, true, 0>(WalkParams, int*, int*);
extern template __global__ void saw_walk_mma_kernel<2, 2, false, 0>(WalkParams, int*, int*);
template cudaError_t launch_walk_mma<1>(const WalkParams&, int, size_t, cudaStream_t, int*, int*, bool);
template cudaError_t launch_walk_mma<2>(const WalkParams&, int, size_t, cudaStream_t, int*, int*, bool);
template int blocks_per_sm_mma<1>(const WalkParams&, size_t);
template int blocks_per_sm_mma<2>(const WalkParams&, size_t);
}  // namespace labs_b200
