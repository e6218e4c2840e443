// deg_p1.cu -- kernels and launchers of degree p = 1 (see dgswe_degree.cuh)
#include "dgswe_degree.cuh"

DGSWE_DEGREE_UNIT(1)
