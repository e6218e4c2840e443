// deg_p6.cu -- kernels and launchers of degree p = 6 (see dgswe_degree.cuh)
#include "dgswe_degree.cuh"

DGSWE_DEGREE_UNIT(6)
