// kernels_hot.cu -- instantiates the scan / batch kernels for StepHot
// (one translation unit per step policy so the library builds in parallel).
#include "kernels_impl.cuh"

namespace sfa {
SFA_DEFINE_STEP_LAUNCHERS(StepHot)
}  // namespace sfa
