// hb_conv_tma.cuh -- argument block of the TMA-fed tcgen05 ring conv (hb_conv_tma.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hb_common.cuh"

namespace hb {
namespace tc {

struct TmaConvArgs {
  long long M;         // output rows = B*OH*OW
  int N, J;            // output channels, weight limbs
  int B, OH, OW, stride, pad, kw;
  int ncc, nkb;        // 64-channel chunks, K blocks = kh*kw*ncc (order: tap-major, chunk-minor)
  int tiles_n, tiles;  // N tiles, total tiles (m-major, n-minor)
  const int8_t* wl;    // [N tiles][nkb][J][NT rows x 64 B, SWIZZLE_64B]
  int party, frac;
  const u64* bias;     // [N] (party 0) or null
  const u64* res;      // NCHW [B][N][OH*OW] residual share added to y, or null
  u64* y;              // NCHW [B][N][OH*OW]
  int nstage;          // smem pipeline depth
  int dbg;             // HB_TC_DEBUG & 1: no MMAs, & 2: no loads, & 4: MMA-warp clock stamps
  long long* stamps;   // dbg & 4: per CTA [total, wait tmem-empty, wait full, issue, stages, units, -, -]
};

}  // namespace tc
}  // namespace hb

cudaError_t hb_limbs_nhwc_launch(const uint64_t* x, long long B, int C, long long HW, uint8_t* planes,
                                 cudaStream_t s);
cudaError_t hb_im2col_planes_launch(const uint64_t* x, int B, int C, int H, int W, int kh, int kw, int stride, int pad,
                                    uint8_t* planes, cudaStream_t s);
int hb_tma_conv_box(int B, int OH, int OW, int* bb, int* bh, int* bw);
cudaError_t hb_tma_conv(const uint8_t* planes, int B, int C, int H, int W, int kh, int kw, int stride, int pad,
                        const int8_t* wl, int N, int J, int nt, int party, int frac, const uint64_t* bias,
                        const uint64_t* res, uint64_t* y, cudaStream_t s);
