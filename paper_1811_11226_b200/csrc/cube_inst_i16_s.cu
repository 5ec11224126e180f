// cube_inst_i16_s.cu -- instantiation unit of the warp kernel: int16_t images,
// the <= 16-volume parameter block (cube_kernel.cuh; one unit per pair so build.py
// compiles them in parallel).
#include "cube_kernel.cuh"

namespace w3d {
namespace cube {
template cudaError_t launch_typed_nv<int16_t, kSmallVol>(const WarpArgsT<kSmallVol>&, bool, cudaStream_t);
template cudaError_t read_stats_nv<int16_t, kSmallVol>(unsigned long long*);
}  // namespace cube
}  // namespace w3d
