// kernels_private_seg.cu -- instantiates the batch (SEG) scan kernels for StepPrivate
// (one translation unit per step policy and mode so the library builds in parallel).
#include "kernels_impl.cuh"

namespace sfa {
SFA_DEFINE_STEP_SEG_LAUNCHER(StepPrivate)
}  // namespace sfa
