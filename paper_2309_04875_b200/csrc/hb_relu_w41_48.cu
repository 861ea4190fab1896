// instantiates the ReLU kernels for window widths 41..48
#define HB_W_LO 41
#define HB_W_HI 48
#include "hb_relu_dispatch.cuh"
