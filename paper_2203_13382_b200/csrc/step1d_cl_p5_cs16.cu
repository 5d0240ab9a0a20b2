// step1d_cl_p5_cs16.cu — instantiation unit: cluster-split corrected 1D kernels, p=5, 16 CTAs per cluster.
#define MGRIT_LAUNCHCL_IMPL
#include <type_traits>

#include "step1d_cluster.cuh"
template struct mgrit::cl::LaunchCl<5, 16>;
