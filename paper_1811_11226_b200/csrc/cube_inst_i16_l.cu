// cube_inst_i16_l.cu -- instantiation unit of the warp kernel: int16_t images,
// the 104-volume parameter block (cube_kernel.cuh; one unit per pair so build.py
// compiles them in parallel).
#include "cube_kernel.cuh"

namespace w3d {
namespace cube {
template cudaError_t launch_typed_nv<int16_t, kMaxVolPerLaunch>(const WarpArgsT<kMaxVolPerLaunch>&, bool, cudaStream_t);
template cudaError_t read_stats_nv<int16_t, kMaxVolPerLaunch>(unsigned long long*);
}  // namespace cube
}  // namespace w3d
