// kernels_L5.cu -- the sweep kernels for count width L = 5 (degree < 2^5).
#include "kernels_L.cuh"

PBSA_INSTANTIATE_L(5)
