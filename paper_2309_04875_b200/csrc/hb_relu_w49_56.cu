// instantiates the ReLU kernels for window widths 49..56
#define HB_W_LO 49
#define HB_W_HI 56
#include "hb_relu_dispatch.cuh"
