// kernels_shared.cu -- instantiates the scan / batch kernels for StepShared
// (one translation unit per step policy so the library builds in parallel).
#include "kernels_impl.cuh"

namespace sfa {
SFA_DEFINE_STEP_LAUNCHERS(StepShared)
}  // namespace sfa
