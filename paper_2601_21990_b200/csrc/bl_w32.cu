// bl_w32.cu — the W = 32 instantiations of the row / loop kernels and
// their launchers (one translation unit per width so the build runs in
// parallel).
#define BL_WLAUNCH_DEFINE
#include "bl_kernels.cuh"

namespace bl {
template struct WLaunch<32>;
}  // namespace bl
