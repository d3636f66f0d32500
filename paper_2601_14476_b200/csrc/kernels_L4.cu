// kernels_L4.cu -- the sweep kernels for count width L = 4 (degree < 2^4).
#include "kernels_L.cuh"

PBSA_INSTANTIATE_L(4)
