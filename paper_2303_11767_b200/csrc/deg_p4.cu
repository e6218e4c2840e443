// deg_p4.cu -- kernels and launchers of degree p = 4 (see dgswe_degree.cuh)
#include "dgswe_degree.cuh"

DGSWE_DEGREE_UNIT(4)
