// Kernel instantiation for moment order M=6 (see kernels_impl.cuh).
#include "kernels_impl.cuh"
MOMG_INSTANTIATE(6)
