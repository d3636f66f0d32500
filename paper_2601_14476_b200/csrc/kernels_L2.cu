// kernels_L2.cu -- the sweep kernels for count width L = 2 (degree < 2^2).
#include "kernels_L.cuh"

PBSA_INSTANTIATE_L(2)
