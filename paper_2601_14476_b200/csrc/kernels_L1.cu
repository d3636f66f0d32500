// kernels_L1.cu -- the sweep kernels for count width L = 1 (degree < 2^1).
#include "kernels_L.cuh"

PBSA_INSTANTIATE_L(1)
