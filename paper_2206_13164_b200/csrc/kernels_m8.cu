// Kernel instantiation for moment order M=8 (see kernels_impl.cuh).
#include "kernels_impl.cuh"
MOMG_INSTANTIATE(8)
