// cube_inst_f32_l.cu -- instantiation unit of the warp kernel: float images,
// the 104-volume parameter block (cube_kernel.cuh; one unit per pair so build.py
// compiles them in parallel).
#include "cube_kernel.cuh"

namespace w3d {
namespace cube {
template cudaError_t launch_typed_nv<float, kMaxVolPerLaunch>(const WarpArgsT<kMaxVolPerLaunch>&, bool, cudaStream_t);
template cudaError_t read_stats_nv<float, kMaxVolPerLaunch>(unsigned long long*);
}  // namespace cube
}  // namespace w3d
