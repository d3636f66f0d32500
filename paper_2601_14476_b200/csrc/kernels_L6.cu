// kernels_L6.cu -- the sweep kernels for count width L = 6 (degree < 2^6).
#include "kernels_L.cuh"

PBSA_INSTANTIATE_L(6)
