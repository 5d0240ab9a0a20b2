// step1d_p3_k2.cu — instantiation unit: 1D kernels for p=3, kind=MGRIT_KIND_FORWARD_EULER.
#define MGRIT_LAUNCH1D_IMPL
#include "step1d_kernels.cuh"
template struct mgrit::Launch1D<3, MGRIT_KIND_FORWARD_EULER>;
