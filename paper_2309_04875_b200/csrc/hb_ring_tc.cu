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
//   in the UMMA canonical K-major no-swizzle layout (8x16B core matrices); the
//   weight-limb tile is copied as-is (host pre-lays it out).  One elected thread
//   issues the MMAs and tcgen05.commit's a per-stage mbarrier; two stages, so the
//   gather of block k+1 overlaps the tensor-core work of block k.
//   epilogue: each thread owns one accumulator row (TMEM lane), tcgen05.ld's its
//   8 x N_T values, folds the shifts mod 2^64, truncates (party-dependent), adds
//   the party-0 bias and stores NCHW (consecutive threads = consecutive pixels).
#include <cstdint>
#include <cuda_runtime.h>

#include "hb_common.cuh"
#include "hb_ring_tc.cuh"

namespace hb {
namespace tc {

constexpr int BM = 128;   // rows per CTA = TMEM lanes
constexpr int KB = 64;    // K bytes per stage (2 MMAs of K = 32)
constexpr int PLANE = BM * KB;  // bytes per limb plane per stage (8 KB)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE (canonical layout
// ((8,m),(T,2)):((1T,SBO),(1,LBO)) in 16-byte units; cute mma_traits_sm100.hpp)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);  // version 1 (sm100)
}

// instruction descriptor: D s32, A u8, B s8, both K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

template <int NCOL>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst)), "n"(NCOL));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}

template <int NCOL>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(NCOL));
}

// 8 consecutive 32-bit TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// canonical K-major offset of (row r, K byte c) inside one [rows x 64 B] tile
__device__ __forceinline__ int canon(int r, int c) { return (r >> 3) * 512 + (c >> 4) * 128 + (r & 7) * 16 + (c & 15); }


// 4x4 byte transpose: out[i] = byte i of (w0, w1, w2, w3), packed little-endian
__device__ __forceinline__ void bytes_t4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&o)[4]) {
  const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w2, w3, 0x5140);
  const uint32_t t2 = __byte_perm(w0, w1, 0x7362), t3 = __byte_perm(w2, w3, 0x7362);
  o[0] = __byte_perm(t0, t1, 0x5410);
  o[1] = __byte_perm(t0, t1, 0x7632);
  o[2] = __byte_perm(t2, t3, 0x5410);
  o[3] = __byte_perm(t2, t3, 0x7632);
}

constexpr int TPB = 512;  // 4 threads per accumulator row

template <int NT>
__global__ void __launch_bounds__(TPB, 1) k_conv_tc(const ConvArgs A) {
  constexpr int NACC_COL = 8 * NT;  // 8 shift accumulators x NT columns
  constexpr int TMEM_COLS = NACC_COL < 32 ? 32 : NACC_COL;
  extern __shared__ __align__(1024) uint8_t smem[];
  // stage s: [8 limb planes (PLANE each)][J weight tiles (NT*KB each)]
  const int J = A.J;
  const int stage_bytes = 8 * PLANE + J * NT * KB;
  __shared__ uint64_t bar_empty[2];
  __shared__ uint64_t bar_done;
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, warp = tid >> 5;
  const long long m0 = (long long)blockIdx.x * BM;
  const int ntile = blockIdx.y;
  const int nkb = A.Kp / KB;

  if (warp == 0) tmem_alloc<TMEM_COLS>(&tmem_base_s);
  if (tid == 0) {
    mbar_init(&bar_empty[0], 1);
    mbar_init(&bar_empty[1], 1);
    mbar_init(&bar_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  // gather role: row r = tid / 4 of the tile, K bytes [16q, 16q + 16) of each stage
  const int r = tid >> 2, q = tid & 3;
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

  uint32_t phase[2] = {0, 0};
  for (int kb = 0; kb < nkb; ++kb) {
    const int st = kb & 1;
    uint8_t* sA = smem + st * stage_bytes;
    uint8_t* sB = sA + 8 * PLANE;
    // ---- gather 16 patch values (all loads issued before any use); k = c*khw + ki*kw + kj
    u64 v[16];
    {
      const int k0 = kb * KB + q * 16;
      int c = k0 / khw;
      const int t0 = k0 - c * khw;
      int ki = t0 / A.kw, kj = t0 - ki * A.kw;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int ih = ih0 + ki, iw = iw0 + kj;
        const bool ok = row_ok && (k0 + e < A.K) && (unsigned)ih < (unsigned)A.H && (unsigned)iw < (unsigned)A.W;
        v[e] = ok ? (u64)__ldg(reinterpret_cast<const unsigned long long*>(xb + c * HW + (long long)ih * A.W + iw)) : 0ull;
        if (++kj == A.kw) {
          kj = 0;
          if (++ki == A.kh) {
            ki = 0;
            ++c;
          }
        }
      }
    }
    // weight-limb tile loads go out together with the patch loads (<= 2 int4 per thread)
    const int n16 = J * NT * KB / 16;
    int4 wv[2];
    {
      const int4* src = reinterpret_cast<const int4*>(A.wl + ((long long)ntile * nkb + kb) * J * NT * KB);
#pragma unroll
      for (int u = 0; u < 2; ++u) wv[u] = (tid + u * TPB < n16) ? __ldg(src + tid + u * TPB) : make_int4(0, 0, 0, 0);
    }
    if (kb >= 2) {  // the MMAs that read this stage (block kb-2) must be done
      mbar_wait(&bar_empty[st], phase[st]);
      phase[st] ^= 1;
    }
    // ---- split into 8 limb planes: 4x4 byte transposes (limb i of 16 values = 16 bytes)
    {
      uint32_t lo[4][4], hi[4][4];  // [group of 4 values][limb]
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        bytes_t4((uint32_t)v[4 * g], (uint32_t)v[4 * g + 1], (uint32_t)v[4 * g + 2], (uint32_t)v[4 * g + 3], lo[g]);
        bytes_t4((uint32_t)(v[4 * g] >> 32), (uint32_t)(v[4 * g + 1] >> 32), (uint32_t)(v[4 * g + 2] >> 32),
                 (uint32_t)(v[4 * g + 3] >> 32), hi[g]);
      }
      const int off = canon(r, q * 16);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        *reinterpret_cast<uint4*>(sA + i * PLANE + off) = make_uint4(lo[0][i], lo[1][i], lo[2][i], lo[3][i]);
        *reinterpret_cast<uint4*>(sA + (4 + i) * PLANE + off) = make_uint4(hi[0][i], hi[1][i], hi[2][i], hi[3][i]);
      }
    }
    // ---- B: this thread's share of the pre-laid-out weight-limb tile (loaded above)
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (tid + u * TPB < n16) reinterpret_cast<int4*>(sB)[tid + u * TPB] = wv[u];
    fence_async_smem();
    __syncthreads();
    // ---- MMA issue (one thread): 2 K-steps x all limb pairs with i + j <= 7
    if (tid == 0) {
      tc_fence_after();
      const uint32_t aBase = smem_u32(sA), bBase = smem_u32(sB);
#pragma unroll
      for (int ks = 0; ks < KB / 32; ++ks) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          for (int j = 0; j < J; ++j) {
            const int s = i + j;
            if (s > 7) continue;
            const int first_i = s - (J - 1) > 0 ? s - (J - 1) : 0;
            const uint32_t acc = (kb == 0 && ks == 0 && i == first_i) ? 0u : 1u;
            const uint64_t da = sdesc(aBase + i * PLANE + ks * 256, 128, 512);
            const uint64_t db = sdesc(bBase + j * NT * KB + ks * 256, 128, 512);
            mma_i8(tmem + s * NT, da, db, idesc_i8(NT), acc);
          }
        }
      }
      mma_commit(&bar_empty[st]);
      if (kb == nkb - 1) mma_commit(&bar_done);
    }
  }

  // ---- epilogue: warp w reads TMEM lanes 32*(w%4).. (its row quarter) and a column group
  mbar_wait(&bar_done, 0);
  tc_fence_after();
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
      for (int s = 0; s < 8; ++s) tmem_ld8(lane_base + s * NT + c0, vv[s]);
      tmem_wait_ld();
#pragma unroll
      for (int s = 0; s < 8; ++s)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += (u64)(long long)(int32_t)vv[s][k] << (8 * s);
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
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<TMEM_COLS>(tmem);
}

}  // namespace tc
}  // namespace hb

cudaError_t hb_tc_conv(const hb::tc::ConvArgs& A, int nt, cudaStream_t s) {
  using namespace hb::tc;
  const int stage_bytes = 8 * PLANE + A.J * nt * KB;
  const size_t smem = 2 * (size_t)stage_bytes;
  dim3 grid((unsigned)((A.M + BM - 1) / BM), (unsigned)((A.N + nt - 1) / nt));
  cudaError_t e;
  switch (nt) {
#define HB_NT(NT_)                                                                                      \
  case NT_:                                                                                             \
    e = cudaFuncSetAttribute(k_conv_tc<NT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
    if (e != cudaSuccess) return e;                                                                     \
    k_conv_tc<NT_><<<grid, TPB, smem, s>>>(A);                                                          \
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
