// instantiates the ReLU kernels for window widths 2..8
#define HB_W_LO 2
#define HB_W_HI 8
#include "hb_relu_dispatch.cuh"
