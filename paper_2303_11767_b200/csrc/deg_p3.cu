// deg_p3.cu -- kernels and launchers of degree p = 3 (see dgswe_degree.cuh)
#include "dgswe_degree.cuh"

DGSWE_DEGREE_UNIT(3)
