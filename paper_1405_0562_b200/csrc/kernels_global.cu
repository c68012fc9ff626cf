// kernels_global.cu -- instantiates the scan / batch kernels for StepGlobal
// (one translation unit per step policy so the library builds in parallel).
#include "kernels_impl.cuh"

namespace sfa {
SFA_DEFINE_STEP_LAUNCHERS(StepGlobal)
}  // namespace sfa
