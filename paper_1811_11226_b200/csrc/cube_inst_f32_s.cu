// cube_inst_f32_s.cu -- instantiation unit of the warp kernel: float images,
// the <= 16-volume parameter block (cube_kernel.cuh; one unit per pair so build.py
// compiles them in parallel).
#include "cube_kernel.cuh"

namespace w3d {
namespace cube {
template cudaError_t launch_typed_nv<float, kSmallVol>(const WarpArgsT<kSmallVol>&, bool, cudaStream_t);
template cudaError_t read_stats_nv<float, kSmallVol>(unsigned long long*);
}  // namespace cube
}  // namespace w3d
