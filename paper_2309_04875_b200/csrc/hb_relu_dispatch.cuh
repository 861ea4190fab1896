// hb_relu_dispatch.cuh -- per-width launchers.  Each translation unit
// hb_relu_w<lo>_<hi>.cu defines HB_W_LO / HB_W_HI and includes this file, so
// the 63 window widths compile in parallel (make -j).
#pragma once
#include "hb_relu_impl.cuh"
#include "hb_relu_p2p.cuh"

namespace hb {

#ifndef HB_PAIR_TP
#define HB_PAIR_TP 32
#endif
constexpr int PAIR_TP = HB_PAIR_TP;  // threads per party per CTA (CTA = 2 * PAIR_TP)

template <int W>
size_t pair_smem_bytes() {
  return sizeof(u64) * 2 * 2 * PairGeo<W>::SEGW * PAIR_TP;
}

template <int W, bool R64>
cudaError_t launch_pair_impl(const PairArgs& A, cudaStream_t s) {
  constexpr int GS = Geo<W>::GS;
  const u64 ngroups = (A.count + GS - 1) / GS;
  const u64 blocks = (ngroups + PAIR_TP - 1) / PAIR_TP;
  const size_t smem = pair_smem_bytes<W>();
  static bool configured = false;  // benign race: idempotent attribute set
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(k_relu_pair<W, PAIR_TP, R64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  k_relu_pair<W, PAIR_TP, R64><<<(unsigned)blocks, 2 * PAIR_TP, smem, s>>>(A);
  return cudaGetLastError();
}

template <int W>
cudaError_t launch_pair(const PairArgs& A, cudaStream_t s) {
  return A.N == 64 ? launch_pair_impl<W, true>(A, s) : launch_pair_impl<W, false>(A, s);
}

template <int W>
cudaError_t launch_stage(const StageArgs& A, int L, cudaStream_t s) {
  const unsigned blocks = (unsigned)((A.ngroups + 255) / 256);
  if (blocks == 0) return cudaSuccess;
  const int r = A.round;
  if (r == 0) k_stage<W, RK_OTHER><<<blocks, 256, 0, s>>>(A);
  else if (r <= L) k_stage<W, RK_LEVEL><<<blocks, 256, 0, s>>>(A);
  else if (r == L + 1) k_stage<W, RK_B2A><<<blocks, 256, 0, s>>>(A);
  else if (r == L + 2) k_stage<W, RK_MULT><<<blocks, 256, 0, s>>>(A);
  else k_stage<W, RK_FINAL><<<blocks, 256, 0, s>>>(A);
  return cudaGetLastError();
}

}  // namespace hb

#if defined(HB_W_LO) && defined(HB_W_HI)
#define HB_CAT2(a, b, c) a##b##_##c
#define HB_CAT(a, b, c) HB_CAT2(a, b, c)

// Range dispatchers: return cudaErrorInvalidValue if W is outside this TU's range.
cudaError_t HB_CAT(hb_pair_dispatch_, HB_W_LO, HB_W_HI)(int W, const hb::PairArgs& A, cudaStream_t s) {
  switch (W) {
#define HB_CASE(w) \
  case w:          \
    if (w >= HB_W_LO && w <= HB_W_HI) return hb::launch_pair<(w >= HB_W_LO && w <= HB_W_HI) ? w : HB_W_LO>(A, s); \
    break;
#include "hb_widths.inc"
#undef HB_CASE
    default:
      break;
  }
  return cudaErrorInvalidValue;
}

cudaError_t HB_CAT(hb_stage_dispatch_, HB_W_LO, HB_W_HI)(int W, const hb::StageArgs& A, int L, cudaStream_t s) {
  switch (W) {
#define HB_CASE(w) \
  case w:          \
    if (w >= HB_W_LO && w <= HB_W_HI) return hb::launch_stage<(w >= HB_W_LO && w <= HB_W_HI) ? w : HB_W_LO>(A, L, s); \
    break;
#include "hb_widths.inc"
#undef HB_CASE
    default:
      break;
  }
  return cudaErrorInvalidValue;
}

cudaError_t HB_CAT(hb_p2p_dispatch_, HB_W_LO, HB_W_HI)(int W, const hb::P2PArgs& A, const hb::P2PArgs* B, int max_ctas,
                                                       int max_ctas1, int dual_sys, cudaStream_t s) {
  switch (W) {
#define HB_CASE(w) \
  case w:          \
    if (w >= HB_W_LO && w <= HB_W_HI) return hb::launch_p2p<(w >= HB_W_LO && w <= HB_W_HI) ? w : HB_W_LO>(A, B, max_ctas, max_ctas1, dual_sys, s); \
    break;
#include "hb_widths.inc"
#undef HB_CASE
    default:
      break;
  }
  return cudaErrorInvalidValue;
}

unsigned long long HB_CAT(hb_p2p_layout_, HB_W_LO, HB_W_HI)(int W, unsigned long long n, int drelu_only,
                                                           unsigned long long* ntiles) {
  switch (W) {
#define HB_CASE(w)                                                                                    \
  case w:                                                                                             \
    if (w >= HB_W_LO && w <= HB_W_HI) {                                                               \
      hb::u64 off[hb::P2P_MAXR], nt;                                                                  \
      const hb::u64 b = hb::p2p_layout<(w >= HB_W_LO && w <= HB_W_HI) ? w : HB_W_LO>(n, drelu_only, off, &nt); \
      *ntiles = nt;                                                                                   \
      return b;                                                                                       \
    }                                                                                                 \
    break;
#include "hb_widths.inc"
#undef HB_CASE
    default:
      break;
  }
  return 0;
}

size_t HB_CAT(hb_pair_smem_, HB_W_LO, HB_W_HI)(int W) {
  switch (W) {
#define HB_CASE(w) \
  case w:          \
    return (w >= HB_W_LO && w <= HB_W_HI) ? hb::pair_smem_bytes<(w >= HB_W_LO && w <= HB_W_HI) ? w : HB_W_LO>() : 0;
#include "hb_widths.inc"
#undef HB_CASE
    default:
      break;
  }
  return 0;
}
#endif
