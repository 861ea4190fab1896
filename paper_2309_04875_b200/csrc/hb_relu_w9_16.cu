// instantiates the ReLU kernels for window widths 9..16
#define HB_W_LO 9
#define HB_W_HI 16
#include "hb_relu_dispatch.cuh"
