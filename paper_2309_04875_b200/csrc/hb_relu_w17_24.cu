// instantiates the ReLU kernels for window widths 17..24
#define HB_W_LO 17
#define HB_W_HI 24
#include "hb_relu_dispatch.cuh"
