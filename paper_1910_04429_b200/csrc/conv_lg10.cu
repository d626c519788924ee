// Instantiates the conv kernels for 2^10-point row/column transforms.
#include "conv_kernels.cuh"
PAB_DEFINE_CONV(10)
