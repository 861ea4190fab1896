// hb_ring_tc.cuh -- argument block of the fused tcgen05 ring conv (hb_ring_tc.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hb_common.cuh"

namespace hb {
namespace tc {

struct ConvArgs {
  const u64* x;
  int B, C, H, W, kh, kw, stride, pad, OH, OW;
  long long M, K;      // M = B*OH*OW rows, K = C*kh*kw
  int Kp;              // K padded to a multiple of KB
  int N, J;            // output channels, weight limbs
  const int8_t* wl;    // [N/N_T][Kp/KB][J][N_T x KB canonical]
  int party, frac;
  const u64* bias;     // [N] (party 0) or null
  u64* y;              // NCHW [B][N][OH*OW]
  int nstage;          // smem pipeline depth (set by hb_tc_conv)
  int dbg;             // profiling switches (HB_TC_DEBUG): 1 = no MMAs, 2 = no global gathers, 4 = timestamps
  long long* stamps;   // dbg & 4: per-CTA clock64 phase stamps [grid][8]
};

}  // namespace tc
}  // namespace hb

cudaError_t hb_tc_conv(const hb::tc::ConvArgs& A, int nt, cudaStream_t s);
