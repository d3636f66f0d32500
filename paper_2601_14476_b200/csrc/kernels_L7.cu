// kernels_L7.cu -- the sweep kernels for count width L = 7 (degree < 2^7).
#include "kernels_L.cuh"

PBSA_INSTANTIATE_L(7)
