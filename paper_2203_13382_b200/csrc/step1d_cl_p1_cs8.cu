// step1d_cl_p1_cs8.cu — instantiation unit: cluster-split corrected 1D kernels, p=1, 8 CTAs per cluster.
#define MGRIT_LAUNCHCL_IMPL
#include <type_traits>

#include "step1d_cluster.cuh"
template struct mgrit::cl::LaunchCl<1, 8>;
