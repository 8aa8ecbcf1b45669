// saw_walk_r9_12.cu -- explicit instantiations of K1 (LPW = 32, 16 and 8) for R = 9..12 (parallel build).
#include "saw_walk.cuh"

namespace labs_b200 {
template cudaError_t launch_walk_fixed<9, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<9, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<9, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<9, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<10, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<10, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<10, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<10, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<11, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<11, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<11, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<11, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<12, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<12, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<12, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<12, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<9, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<9, 8>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<10, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<10, 8>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<11, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<11, 8>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<12, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<12, 8>(const WalkParams&, size_t);
}  // namespace labs_b200
