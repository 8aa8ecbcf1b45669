// saw_walk_r5_8.cu -- explicit instantiations of K1 (LPW = 32, 16 and 8) for R = 5..8 (parallel build).
#include "saw_walk.cuh"

namespace labs_b200 {
template cudaError_t launch_walk_fixed<5, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<5, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<5, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<5, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<6, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<6, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<6, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<6, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<7, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<7, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<7, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<7, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<8, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<8, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<8, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<8, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<5, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<5, 8>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<6, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<6, 8>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<7, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<7, 8>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<8, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<8, 8>(const WalkParams&, size_t);
}  // namespace labs_b200
