// Instantiates the conv kernels for 2^7-point row/column transforms.
#include "conv_kernels.cuh"
PAB_DEFINE_CONV(7)
