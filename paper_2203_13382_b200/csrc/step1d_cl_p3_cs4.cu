// step1d_cl_p3_cs4.cu — instantiation unit: cluster-split corrected 1D kernels, p=3, 4 CTAs per cluster.
#define MGRIT_LAUNCHCL_IMPL
#include <type_traits>

#include "step1d_cluster.cuh"
template struct mgrit::cl::LaunchCl<3, 4>;
