// instantiates the ReLU kernels for window widths 57..64
#define HB_W_LO 57
#define HB_W_HI 64
#include "hb_relu_dispatch.cuh"
