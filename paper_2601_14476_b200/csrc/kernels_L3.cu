// kernels_L3.cu -- the sweep kernels for count width L = 3 (degree < 2^3).
#include "kernels_L.cuh"

PBSA_INSTANTIATE_L(3)
