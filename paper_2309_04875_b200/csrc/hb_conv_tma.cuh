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
  int tiles_n, tiles;  // N tiles, total tiles (party-major, then m-major, n-minor)
  int tiles_pp;        // tiles per party (tiles = nparts * tiles_pp)
  const int8_t* wl;    // [N tiles][nkb][J][NT rows x 64 B, SWIZZLE_64B]
  int frac;
  int party[2];        // the party of sub-problem 0 / 1 (one launch may hold both parties' convs)
  const u64* bias;     // [N] (added by party 0) or null
  const u64* res[2];   // NCHW [B][N][OH*OW] residual share added to y, or null
  u64* y[2];           // NCHW [B][N][OH*OW]
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
// nparts = 1: one party's conv (planes[0], party[0], res[0], y[0]); nparts = 2: both parties' convs of
// one layer (same geometry and weights) in ONE launch -- half the launches, twice the tiles to
// balance over the persistent grid.
cudaError_t hb_tma_conv(int nparts, const uint8_t* const* planes, int B, int C, int H, int W, int kh, int kw,
                        int stride, int pad, const int8_t* wl, int N, int J, int nt, const int* party, int frac,
                        const uint64_t* bias, const uint64_t* const* res, uint64_t* const* y, cudaStream_t s);
