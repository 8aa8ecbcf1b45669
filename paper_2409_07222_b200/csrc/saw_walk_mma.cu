// saw_walk_mma.cu -- instantiations of K1t (tensor-core G, saw_walk_mma.cuh): 1 or 2 q-tiles.
#include "saw_walk_mma.cuh"

namespace labs_b200 {
template cudaError_t launch_walk_mma<1>(const WalkParams&, int, size_t, cudaStream_t, int*, int*, bool);
template cudaError_t launch_walk_mma<2>(const WalkParams&, int, size_t, cudaStream_t, int*, int*, bool);
template int blocks_per_sm_mma<1>(const WalkParams&, size_t);
template int blocks_per_sm_mma<2>(const WalkParams&, size_t);
}  // namespace labs_b200
