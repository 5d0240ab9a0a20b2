// step1d_p1_k1.cu — instantiation unit: 1D kernels for p=1, kind=MGRIT_KIND_CORRECTED.
#define MGRIT_LAUNCH1D_IMPL
#include "step1d_kernels.cuh"
template struct mgrit::Launch1D<1, MGRIT_KIND_CORRECTED>;
