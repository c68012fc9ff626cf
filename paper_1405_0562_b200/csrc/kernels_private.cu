// kernels_private.cu -- instantiates the scan / batch kernels for StepPrivate
// (one translation unit per step policy so the library builds in parallel).
#include "kernels_impl.cuh"

namespace sfa {
SFA_DEFINE_STEP_LAUNCHERS(StepPrivate)
}  // namespace sfa
