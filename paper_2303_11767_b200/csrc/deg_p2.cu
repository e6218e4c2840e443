// deg_p2.cu -- kernels and launchers of degree p = 2 (see dgswe_degree.cuh)
#include "dgswe_degree.cuh"

DGSWE_DEGREE_UNIT(2)
