// saw_walk_r13_16.cu -- explicit instantiations of K1 (LPW = 32, 16 and 8) for R = 13..16 (parallel build).
#include "saw_walk.cuh"

namespace labs_b200 {
template cudaError_t launch_walk_fixed<13, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<13, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<13, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<13, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<14, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<14, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<14, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<14, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<15, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<15, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<15, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<15, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<16, 32>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<16, 32>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<16, 16>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<16, 16>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<13, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<13, 8>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<14, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<14, 8>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<15, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<15, 8>(const WalkParams&, size_t);
template cudaError_t launch_walk_fixed<16, 8>(const WalkParams&, int, size_t, cudaStream_t,
                                               int*, int*, bool);
template int blocks_per_sm_fixed<16, 8>(const WalkParams&, size_t);
}  // namespace labs_b200
