// instantiates the ReLU kernels for window widths 25..32
#define HB_W_LO 25
#define HB_W_HI 32
#include "hb_relu_dispatch.cuh"
