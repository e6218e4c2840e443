// deg_p5.cu -- kernels and launchers of degree p = 5 (see dgswe_degree.cuh)
#include "dgswe_degree.cuh"

DGSWE_DEGREE_UNIT(5)
