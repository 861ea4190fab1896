// hb_ring_tc.cu -- fused ring-exact conv / linear on tcgen05 tensor cores (sm_100a).
//
// y = trunc( (patches(x) W^T) mod 2^64 ) + [p0] b  for a uint64 share x (nn.py:198-243).
//
// x_i (8 unsigned byte limbs of the share) times w_j (J signed byte limbs of the
// encoded weight) are exact u8 x s8 -> s32 MMAs (tcgen05.mma kind::i8).  Products
// with the same shift s = i + j are ACCUMULATED IN THE SAME TMEM REGION, so the
// CTA keeps just 8 accumulators (one per byte shift) of N_T columns each:
//     acc_s = sum_{i+j=s} x_i w_j^T   (|acc_s| <= 3 K 255 128 < 2^31 for K <= 21900)
//     y     = sum_s acc_s 2^(8s) mod 2^64
// so nothing but x, the weight limbs and y ever touches HBM (the cuBLASLt path
// writes 8*J int32 partial products per output).
//
// CTA: 128 threads, output tile 128 rows (M = batch*OH*OW) x N_T columns.
//   mainloop, per K block of 64:  all threads gather the im2col patch values of
//   the tile (u64), split them into 8 limb planes and store them in shared memory
//   in the UMMA K-major SWIZZLE_64B layout (64-byte rows, 16-byte chunks XOR-swizzled); the
//   weight-limb tile is copied as-is (host pre-lays it out).  One elected thread
//   issues the MMAs and tcgen05.commit's a per-stage mbarrier; two stages, so the
//   gather of block k+1 overlaps the tensor-core work of block k.
//   epilogue: each thread owns one accumulator row (TMEM lane), tcgen05.ld's its
//   8 x N_T values, folds the shifts mod 2^64, truncates (party-dependent), adds
//   the party-0 bias and stores NCHW (consecutive threads = consecutive pixels).
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "hb_common.cuh"
#include "hb_ring_tc.cuh"
#include "hb_tc_ptx.cuh"

namespace hb {
namespace tc {

// SWIZZLE_64B K-major offset of (row r, K byte c) inside one [rows x 64 B] tile
__device__ __forceinline__ int canon(int r, int c) { return r * 64 + ((((c >> 4) ^ (r >> 1)) & 3) << 4) + (c & 15); }

constexpr int NPROD = 512;        // producer threads: 4 per accumulator row
constexpr int TPB = NPROD + 32;   // + one MMA-issuer warp
constexpr int MAX_STAGE = 3;

// Warp-specialised: warps 0..15 gather/split/store (and run the epilogue), warp 16
// issues the MMAs.  Stages are handed over with full/empty mbarriers, so producer
// warps run up to NSTAGE blocks ahead of the tensor cores and of each other.
template <int NT>
__global__ void __launch_bounds__(TPB, 1) k_conv_tc(const ConvArgs A) {
  constexpr int NACC_COL = 8 * NT;  // 8 shift accumulators x NT columns
  constexpr int TMEM_COLS = NACC_COL < 32 ? 32 : NACC_COL;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int J = A.J;
  const int stage_bytes = 8 * PLANE + J * NT * KB;  // [8 limb planes][J weight tiles]
  __shared__ uint64_t bar_full[MAX_STAGE], bar_empty[MAX_STAGE];
  const int NSTAGE = A.nstage;
  __shared__ uint64_t bar_done;
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, warp = tid >> 5;
  const long long m0 = (long long)blockIdx.x * BM;
  const int ntile = blockIdx.y;
  const int nkb = A.Kp / KB;
  const int n16 = J * NT * KB / 16;  // int4 per weight tile (<= 2 per producer thread)

  const bool stamp = (A.dbg & 4) && A.stamps;
  long long* my_st = stamp ? A.stamps + ((long long)blockIdx.y * gridDim.x + blockIdx.x) * 8 : nullptr;
  if (stamp && tid == 0) my_st[0] = clock64();
  if (warp == 0) tmem_alloc<TMEM_COLS>(&tmem_base_s);
  if (tid == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&bar_full[i], NPROD / 32);  // one arrival per producer warp
      mbar_init(&bar_empty[i], 1);
    }
    mbar_init(&bar_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  if (stamp && tid == 0) my_st[1] = clock64();

  if (warp == NPROD / 32) {
    // ================= MMA issuer
    for (int kb = 0; kb < nkb; ++kb) {
      const int st = kb % NSTAGE;
      mbar_wait(&bar_full[st], (kb / NSTAGE) & 1);
      tc_fence_after();
      if ((tid & 31) == 0 && !(A.dbg & 1)) {
        const uint8_t* sA = smem + st * stage_bytes;
        const uint32_t aBase = smem_u32(sA), bBase = smem_u32(sA + 8 * PLANE);
#pragma unroll
        for (int ks = 0; ks < KB / 32; ++ks) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            for (int j = 0; j < J; ++j) {
              const int sh = i + j;
              if (sh > 7) continue;
              const int first_i = sh - (J - 1) > 0 ? sh - (J - 1) : 0;
              const uint32_t acc = (kb == 0 && ks == 0 && i == first_i) ? 0u : 1u;
              const uint64_t da = sdesc(aBase + i * PLANE + ks * 32);
              const uint64_t db = sdesc(bBase + j * NT * KB + ks * 32);
              mma_i8(tmem + sh * NT, da, db, idesc_i8(NT), acc);
            }
          }
        }
      }
      if ((tid & 31) == 0) {
        mma_commit(&bar_empty[st]);
        if (kb == nkb - 1) mma_commit(&bar_done);
      }
      __syncwarp();
    }
  } else {
    // ================= producers: thread (r, q) owns row r, K bytes [16q, 16q + 16) of each block.
    // r & 7 = tid & 7: each 8-thread phase of a 128-bit smem store covers 8 rows of one 512-byte
    // swizzle atom, whose XOR spreads them over all 32 banks; consecutive threads = consecutive pixels.
    const int r = ((tid >> 5) << 3) | (tid & 7), q = (tid >> 3) & 3;
    const long long m = m0 + r;
    const bool row_ok = m < A.M;
    const long long S = (long long)A.OH * A.OW;
    int b = 0, oh = 0, ow = 0;
    if (row_ok) {
      b = (int)(m / S);
      const int rem = (int)(m - (long long)b * S);
      oh = rem / A.OW;
      ow = rem - oh * A.OW;
    }
    const int khw = A.kh * A.kw;
    const int ih0 = oh * A.stride - A.pad, iw0 = ow * A.stride - A.pad;
    const long long HW = (long long)A.H * A.W;
    const u64* xb = A.x + (long long)b * A.C * HW;
    const int4* wsrc = reinterpret_cast<const int4*>(A.wl) + (long long)ntile * nkb * n16;
    const int off = canon(r, q * 16);

    // 16 patch values (k = c*khw + ki*kw + kj) of block kb for this thread
    auto gather = [&](int kb, u64 (&v)[16]) {
      const int k0 = kb * KB + q * 16;
      int c = k0 / khw;
      const int t0 = k0 - c * khw;
      int ki = t0 / A.kw, kj = t0 - ki * A.kw;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int ih = ih0 + ki, iw = iw0 + kj;
        const bool ok = !(A.dbg & 2) && row_ok && (k0 + e < A.K) && (unsigned)ih < (unsigned)A.H &&
                        (unsigned)iw < (unsigned)A.W;
        v[e] = ok ? (u64)__ldg(reinterpret_cast<const unsigned long long*>(xb + c * HW + (long long)ih * A.W + iw))
                  : 0ull;
        if (++kj == A.kw) {
          kj = 0;
          if (++ki == A.kh) {
            ki = 0;
            ++c;
          }
        }
      }
    };

    u64 v[16];
    gather(0, v);
    for (int kb = 0; kb < nkb; ++kb) {
      const int st = kb % NSTAGE;
      uint8_t* sA = smem + st * stage_bytes;
      uint8_t* sB = sA + 8 * PLANE;
      // software pipeline: the next block's gathers are in flight while this block is split
      u64 nv[16];
      if (kb + 1 < nkb) gather(kb + 1, nv);
      int4 wv[2];
#pragma unroll
      for (int u = 0; u < 2; ++u)
        wv[u] = (tid + u * NPROD < n16) ? __ldg(wsrc + (long long)kb * n16 + tid + u * NPROD) : make_int4(0, 0, 0, 0);
      if (kb >= NSTAGE) mbar_wait(&bar_empty[st], ((kb / NSTAGE) - 1) & 1);  // MMAs of block kb-NSTAGE done
      // split into 8 limb planes: 4x4 byte transposes (limb i of 16 values = 16 bytes)
      uint32_t lo[4][4], hi[4][4];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        bytes_t4((uint32_t)v[4 * g], (uint32_t)v[4 * g + 1], (uint32_t)v[4 * g + 2], (uint32_t)v[4 * g + 3], lo[g]);
        bytes_t4((uint32_t)(v[4 * g] >> 32), (uint32_t)(v[4 * g + 1] >> 32), (uint32_t)(v[4 * g + 2] >> 32),
                 (uint32_t)(v[4 * g + 3] >> 32), hi[g]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        *reinterpret_cast<uint4*>(sA + i * PLANE + off) = make_uint4(lo[0][i], lo[1][i], lo[2][i], lo[3][i]);
        *reinterpret_cast<uint4*>(sA + (4 + i) * PLANE + off) = make_uint4(hi[0][i], hi[1][i], hi[2][i], hi[3][i]);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (tid + u * NPROD < n16) reinterpret_cast<int4*>(sB)[tid + u * NPROD] = wv[u];
      fence_async_smem();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&bar_full[st]);
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = nv[e];
    }

    if (stamp && tid == 0) my_st[2] = clock64();
    // ================= epilogue: warp w reads TMEM lane quarter w%4, column group w/4
    mbar_wait(&bar_done, 0);
    tc_fence_after();
    if (stamp && tid == 0) my_st[3] = clock64();
    constexpr int CPG = NT / 4 < 8 ? 8 : NT / 4;  // columns per warp group
    constexpr int NGRP = NT / CPG;
    const int quarter = warp & 3, cgrp = warp >> 2;
    if (cgrp < NGRP) {
      const int er = quarter * 32 + (tid & 31);  // this thread's accumulator row
      const long long em = m0 + er;
      const bool eok = em < A.M;
      const int eb = eok ? (int)(em / S) : 0;
      const long long esp = eok ? em - (long long)eb * S : 0;
      const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
#pragma unroll 1
      for (int c0 = cgrp * CPG; c0 < (cgrp + 1) * CPG; c0 += 8) {
        u64 acc[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = 0;
        uint32_t vv[8][8];
#pragma unroll
        for (int sh = 0; sh < 8; ++sh) tmem_ld8(lane_base + sh * NT + c0, vv[sh]);
        tmem_wait_ld();
#pragma unroll
        for (int sh = 0; sh < 8; ++sh)
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[k] += (u64)(long long)(int32_t)vv[sh][k] << (8 * sh);
        if (eok) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int n = ntile * NT + c0 + k;
            if (n < A.N) {
              u64 yv = A.party == 0 ? (acc[k] >> A.frac) : (0ull - ((0ull - acc[k]) >> A.frac));
              if (A.party == 0 && A.bias) yv += A.bias[n];
              A.y[((long long)eb * A.N + n) * S + esp] = yv;
            }
          }
        }
      }
    }
  }
  if (stamp && tid == 0) my_st[4] = clock64();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<TMEM_COLS>(tmem);
  if (stamp && tid == 0) {
    my_st[5] = clock64();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    my_st[6] = smid;
  }
}

}  // namespace tc
}  // namespace hb

long long* hb_tc_last_stamps = nullptr;
size_t hb_tc_last_stamps_n = 0;

cudaError_t hb_tc_conv(const hb::tc::ConvArgs& A, int nt, cudaStream_t s) {
  using namespace hb::tc;
  const int stage_bytes = 8 * PLANE + A.J * nt * KB;
  ConvArgs B = A;
  static const int dbg = [] {
    const char* e = getenv("HB_TC_DEBUG");
    return e ? atoi(e) : 0;
  }();
  B.dbg = dbg;
  B.stamps = nullptr;
  if (dbg & 4) {
    static long long* buf = nullptr;
    static size_t cap = 0;
    const size_t need = (size_t)((A.M + BM - 1) / BM) * ((A.N + nt - 1) / nt) * 8;
    if (need > cap) {
      if (buf) cudaFree(buf);
      cudaMalloc(&buf, need * sizeof(long long));
      cap = need;
    }
    B.stamps = buf;
    hb_tc_last_stamps = buf;
    hb_tc_last_stamps_n = need;
  }
  B.nstage = (size_t)MAX_STAGE * stage_bytes + 2048 <= 227 * 1024 ? MAX_STAGE : 2;
  const size_t smem = B.nstage * (size_t)stage_bytes;
  dim3 grid((unsigned)((A.M + BM - 1) / BM), (unsigned)((A.N + nt - 1) / nt));
  cudaError_t e;
  switch (nt) {
#define HB_NT(NT_)                                                                                      \
  case NT_:                                                                                             \
    e = cudaFuncSetAttribute(k_conv_tc<NT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
    if (e != cudaSuccess) return e;                                                                     \
    k_conv_tc<NT_><<<grid, TPB, smem, s>>>(B);                                                          \
    break;
    HB_NT(16)
    HB_NT(32)
    HB_NT(64)
#undef HB_NT
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// debug export: copy the last launch's phase stamps to host (HB_TC_DEBUG & 4)
extern "C" int hb_debug_conv_stamps(long long* host, long long cap) {
  if (!hb_tc_last_stamps) return 0;
  const size_t n = hb_tc_last_stamps_n < (size_t)cap ? hb_tc_last_stamps_n : (size_t)cap;
  cudaDeviceSynchronize();
  cudaMemcpy(host, hb_tc_last_stamps, n * sizeof(long long), cudaMemcpyDeviceToHost);
  return (int)n;
}
