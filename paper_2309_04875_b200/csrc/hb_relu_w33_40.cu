// instantiates the ReLU kernels for window widths 33..40
#define HB_W_LO 33
#define HB_W_HI 40
#include "hb_relu_dispatch.cuh"
