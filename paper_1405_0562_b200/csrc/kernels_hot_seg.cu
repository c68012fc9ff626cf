// kernels_hot_seg.cu -- instantiates the batch (SEG) scan kernels for StepHot
// (one translation unit per step policy and mode so the library builds in parallel).
#include "kernels_impl.cuh"

namespace sfa {
SFA_DEFINE_STEP_SEG_LAUNCHER(StepHot)
}  // namespace sfa
