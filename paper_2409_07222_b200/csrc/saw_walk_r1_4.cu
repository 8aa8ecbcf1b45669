// saw_walk_r1_4.cu -- explicit instantiations of K1 (LPW = 32, 16 and 8) for R = 1..4 (parallel build).
#include "saw_walk.cuh"

namespace labs_b200 {
template cudaError_t launch_walk_fixed<1, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<1, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<1, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<1, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<2, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<2, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<2, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<2, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<3, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<3, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<3, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<3, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<4, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<4, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<4, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<4, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<1, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<1, 8>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<2, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<2, 8>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<3, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<3, 8>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<4, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<4, 8>(const WalkParams&, size_t);
}  // namespace labs_b200
