// deg_p0.cu -- kernels and launchers of degree p = 0 (see dgswe_degree.cuh)
#include "dgswe_degree.cuh"

DGSWE_DEGREE_UNIT(0)
