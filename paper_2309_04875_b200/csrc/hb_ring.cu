// hb_ring.cu -- ring-exact linear / conv / avgpool on Z/2^64 shares (ringmpc nn.py:198-259).
//
// (X @ W^T) mod 2^64 with X a uint64 share and W a small signed fixed-point
// weight is computed on int8 tensor cores by byte-limb decomposition:
//
//   X = sum_i x_i 256^i,  x_i in [0, 255]          (8 limbs; shares are full-width)
//   W = sum_j w_j 256^j,  w_j in [-128, 127]       (J balanced limbs, J = 3 for |W| < 2^23)
//   X W^T mod 2^64 = sum_{i + j <= 7} 256^(i+j) (x_i w_j^T)
//
// Each limb product is an exact int32 GEMM (|sum| <= K * 255 * 128 < 2^31 for
// K <= 65793).  The tensor cores take signed int8, so the A operand carries
// x_i - 128 and the epilogue adds back 128 * colsum(w_j).  All limb products come
// from ONE int8 GEMM: A = [x_0-128; ...; x_7-128] stacked along M (8M x Kp) and
// B = [w_0 | ... | w_{J-1}] stacked along N (Kp x JN).
//
//   k_limbs_im2col   share (NCHW or [B,K]) -> A, fused im2col + limb split
//   k_ring_combine   int32 limb products -> uint64 shares, fused with the local
//                    truncation (nn.py:198-211), the party-0 bias (nn.py:224) and
//                    the NCHW output layout (nn.py:242-243)
//   k_avgpool        window sum, * encode(1/kk), truncation (nn.py:246-259)
#include <cstdint>
#include <cuda_runtime.h>

#include "hb_common.cuh"

namespace hb {

// One thread per (m, k) patch entry: writes the 8 limbs (minus 128) into the
// 8 limb planes A[i][m][k].  Columns k in [K, Kp) pad K to the GEMM's multiple
// of 16; B's padded rows are zero, so whatever A holds there contributes 0.
__global__ void k_limbs_im2col(const u64* __restrict__ x, int Bn, int C, int H, int Wd, int kh, int kw, int stride,
                               int pad, int OH, int OW, long long K, long long Kp, long long M,
                               int8_t* __restrict__ A) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= M * Kp) return;
  const long long m = idx / Kp, k = idx - m * Kp;
  u64 v = 0;
  if (k < K) {
    const int c = (int)(k / (kh * kw));
    const int t = (int)(k - (long long)c * kh * kw);
    const int ki = t / kw, kj = t - ki * kw;
    const long long b = m / ((long long)OH * OW);
    const int r = (int)(m - b * OH * OW);
    const int oh = r / OW, ow = r - oh * OW;
    const int ih = oh * stride + ki - pad, iw = ow * stride + kj - pad;
    if (ih >= 0 && ih < H && iw >= 0 && iw < Wd) v = x[((b * C + c) * H + ih) * (long long)Wd + iw];
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) A[(long long)i * M * Kp + idx] = (int8_t)((int)((v >> (8 * i)) & 0xff) - 128);
}

// out[m, n] = trunc( sum_{i+j<=7} (P[i*M+m, j*Np+n] + 128 colsum[j][n]) << 8(i+j) ) + [p0] bias[n]
// (Np >= N: each weight-limb block is padded to the GEMM's multiple of 8 columns)
// layout 0: out[m*N + n];  layout 1 (conv): m = b*S + s -> out[(b*N + n)*S + s]
__global__ void k_ring_combine(const int32_t* __restrict__ P, long long M, long long N, long long Np, int J,
                               const int32_t* __restrict__ colsum, int party, int frac, const u64* __restrict__ bias,
                               int layout, long long S, u64* __restrict__ out) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= M * N) return;
  const long long m = idx / N, n = idx - m * N;
  const long long ld = (long long)J * Np;
  u64 acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    for (int j = 0; j < J && i + j <= 7; ++j) {
      const long long p = (long long)P[((long long)i * M + m) * ld + (long long)j * Np + n] + 128ll * colsum[j * Np + n];
      acc += (u64)p << (8 * (i + j));
    }
  }
  // SecureML local truncation (nn.py:206-210): p0 shifts, p1 negates-shifts-negates
  u64 y = party == 0 ? (acc >> frac) : (0ull - ((0ull - acc) >> frac));
  if (party == 0 && bias) y += bias[n];
  if (layout == 0) {
    out[idx] = y;
  } else {
    const long long b = m / S, s = m - b * S;
    out[(b * N + n) * S + s] = y;
  }
}

__global__ void k_avgpool(const u64* __restrict__ x, long long BC, int H, int Wd, int kh, int kw, int stride, int OH,
                          int OW, u64 inv, int party, int frac, u64* __restrict__ out) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= BC * OH * OW) return;
  const long long bc = idx / ((long long)OH * OW);
  const int r = (int)(idx - bc * OH * OW);
  const int oh = r / OW, ow = r - oh * OW;
  u64 s = 0;
  for (int i = 0; i < kh; ++i)
    for (int j = 0; j < kw; ++j) s += x[(bc * H + oh * stride + i) * (long long)Wd + ow * stride + j];
  s *= inv;
  out[idx] = party == 0 ? (s >> frac) : (0ull - ((0ull - s) >> frac));
}

// NHWC variant: x [B, H, W, C] -> out [B, OH, OW, C]
__global__ void k_avgpool_nhwc(const u64* __restrict__ x, long long Bn, int H, int Wd, int C, int kh, int kw,
                               int stride, int OH, int OW, u64 inv, int party, int frac, u64* __restrict__ out) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Bn * OH * OW * C) return;
  const int c = (int)(idx % C);
  const long long pix = idx / C;
  const int ow = (int)(pix % OW);
  const long long t = pix / OW;
  const int oh = (int)(t % OH);
  const long long b = t / OH;
  u64 s = 0;
  for (int i = 0; i < kh; ++i)
    for (int j = 0; j < kw; ++j) s += x[((b * H + oh * stride + i) * (long long)Wd + ow * stride + j) * C + c];
  s *= inv;
  out[idx] = party == 0 ? (s >> frac) : (0ull - ((0ull - s) >> frac));
}

// out = share + other share (mod 2^64): the residual add of ResNet blocks (sharing.py:118-122)
__global__ void k_add(const u64* __restrict__ a, const u64* __restrict__ b, long long n, u64* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] + b[i];
}

inline unsigned nblk(long long n) { return (unsigned)((n + 255) / 256); }

}  // namespace hb

cudaError_t hb_ring_limbs_im2col(const hb::u64* x, int B, int C, int H, int W, int kh, int kw, int stride, int pad,
                                 long long Kp, int8_t* A, cudaStream_t s) {
  const int OH = (H + 2 * pad - kh) / stride + 1, OW = (W + 2 * pad - kw) / stride + 1;
  const long long M = (long long)B * OH * OW, K = (long long)C * kh * kw;
  if (M * Kp) hb::k_limbs_im2col<<<hb::nblk(M * Kp), 256, 0, s>>>(x, B, C, H, W, kh, kw, stride, pad, OH, OW, K, Kp, M, A);
  return cudaGetLastError();
}

cudaError_t hb_ring_combine(const int32_t* P, long long M, long long N, long long Np, int J, const int32_t* colsum,
                            int party, int frac, const hb::u64* bias, int layout, long long S, hb::u64* out,
                            cudaStream_t s) {
  if (M * N)
    hb::k_ring_combine<<<hb::nblk(M * N), 256, 0, s>>>(P, M, N, Np, J, colsum, party, frac, bias, layout, S, out);
  return cudaGetLastError();
}

cudaError_t hb_ring_avgpool(const hb::u64* x, long long BC, int H, int W, int kh, int kw, int stride, hb::u64 inv,
                            int party, int frac, hb::u64* out, cudaStream_t s) {
  const int OH = (H - kh) / stride + 1, OW = (W - kw) / stride + 1;
  if (BC * OH * OW)
    hb::k_avgpool<<<hb::nblk(BC * OH * OW), 256, 0, s>>>(x, BC, H, W, kh, kw, stride, OH, OW, inv, party, frac, out);
  return cudaGetLastError();
}

cudaError_t hb_ring_avgpool_nhwc(const hb::u64* x, long long B, int H, int W, int C, int kh, int kw, int stride,
                                 hb::u64 inv, int party, int frac, hb::u64* out, cudaStream_t s) {
  const int OH = (H - kh) / stride + 1, OW = (W - kw) / stride + 1;
  const long long n = B * OH * OW * C;
  if (n) hb::k_avgpool_nhwc<<<hb::nblk(n), 256, 0, s>>>(x, B, H, W, C, kh, kw, stride, OH, OW, inv, party, frac, out);
  return cudaGetLastError();
}

cudaError_t hb_ring_add(const hb::u64* a, const hb::u64* b, long long n, hb::u64* out, cudaStream_t s) {
  if (n) hb::k_add<<<hb::nblk(n), 256, 0, s>>>(a, b, n, out);
  return cudaGetLastError();
}
