// Timing harness for a pair ReLU that also writes the next conv's byte-limb planes
// ([limb][C/64][B][H][W][64], k_limbs_nhwc's layout) -- CTA orders and tile shapes against
// k_relu_pair (+ k_limbs_nhwc), on synthetic shares / triples (speed does not depend on the values).
// Measured on B200, ResNet18 layer1 b512 (2^25 elements): k_relu_pair 0.927 ms + 2 x k_limbs_nhwc
// 0.079 ms = 1.085 ms vs 1.109 ms for the best fused variant (4 channel runs per thread, planes
// only) -- the element-to-CTA remap costs what the separate pass costs, so the product keeps it.  Build (W = 8):
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
//        tools/micro/planes_bench.cu -o tools/micro/planes_bench
//   ./tools/micro/planes_bench [B] [C] [HW] [reps]
#include <cstdio>
#include <cstdlib>

#include "../../paper_2309_04875_b200/csrc/hb_relu_impl.cuh"

using namespace hb;

struct PlaneArgs {
  uint8_t* planes[2];
  u64 B;
  int C, HW, PR;
  int write_y;
};

HB_DEV void bytes_t4x(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&o)[4]) {
  const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w2, w3, 0x5140);
  const uint32_t t2 = __byte_perm(w0, w1, 0x7362), t3 = __byte_perm(w2, w3, 0x7362);
  o[0] = __byte_perm(t0, t1, 0x5410);
  o[1] = __byte_perm(t0, t1, 0x7632);
  o[2] = __byte_perm(t2, t3, 0x5410);
  o[3] = __byte_perm(t2, t3, 0x7632);
}

#ifndef HB_MICRO_TP
#define HB_MICRO_TP 64
#endif
#ifndef HB_MICRO_W
#define HB_MICRO_W 8
#endif
constexpr int W = HB_MICRO_W, TP = HB_MICRO_TP;

__global__ void k_fill(u64* p, u64 n, u64 seed) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    u64 z = (i + seed) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    p[i] = z ^ (z >> 31);
  }
}

static u64* dalloc(u64 words, u64 seed) {
  u64* p;
  if (cudaMalloc(&p, words * 8) != cudaSuccess) exit(1);
  k_fill<<<1184, 256>>>(p, words, seed);
  return p;
}

// ORDER 0: channel group fastest; 1: pixel run fastest (within the image); 2: CTAs in groups of G
// runs x all channel groups (run-major blocks)
template <int ORDER, bool STORE>
__global__ void __launch_bounds__(2 * TP, 1) k_var(const PairArgs A, const PlaneArgs P) {
  constexpr int GS = Geo<W>::GS;
  extern __shared__ u64 wire[];
  const int party = threadIdx.x >= TP ? 1 : 0;
  const int t = threadIdx.x - party * TP;
  const int PR = P.PR, tpr = PR / GS, cpc = TP * GS / PR, ngrp = P.C / cpc;
  const u64 cta = blockIdx.x;
  const int rpi = P.HW / PR;
  const u64 nrun = P.B * (u64)rpi;
  int cg;
  u64 run;
  if (ORDER == 0) {
    cg = (int)(cta % (u64)ngrp);
    run = cta / (u64)ngrp;
  } else if (ORDER == 1) {
    run = cta % nrun;
    cg = (int)(cta / nrun);
  } else {
    const u64 G = 16, blk = cta / (G * ngrp), in = cta % (G * ngrp);
    run = blk * G + in % G;
    cg = (int)(in / G);
  }
  const u64 b = run / (u64)rpi;
  const int p0 = (int)(run % (u64)rpi) * PR;
  const int ci = t / tpr, pj = (t % tpr) * GS;
  const int c = cg * cpc + ci;
  const u64 e0 = (b * (u64)P.C + (u64)c) * (u64)P.HW + (u64)(p0 + pj);
  u64 yv[GS];
  pair_group<W, TP, true>(A, party, t, e0, GS, wire, yv);
  if (P.write_y) store_u64s<GS>(A.io[party].y + e0, GS, yv);
  if (!STORE) return;
  __syncthreads();
  u64* stage = wire + (u64)party * PR * cpc;
#pragma unroll
  for (int j = 0; j < GS; ++j) stage[(pj + j) * cpc + ci] = yv[j];
  __syncthreads();
  const int oct = cpc / 8;
  const u64 plane = P.B * (u64)P.HW * (u64)P.C;
  const int cb = cg * cpc;
  uint8_t* base = P.planes[party] + (u64)(cb / 64) * (P.B * (u64)P.HW * 64) + (b * (u64)P.HW + (u64)p0) * 64 + (cb % 64);
  for (int it = t; it < PR * oct; it += TP) {
    const int q = it / oct, o = it - q * oct;
    const u64* v = stage + q * cpc + o * 8;
    uint32_t lo03[4], lo47[4], hi03[4], hi47[4];
    bytes_t4x((uint32_t)v[0], (uint32_t)v[1], (uint32_t)v[2], (uint32_t)v[3], lo03);
    bytes_t4x((uint32_t)v[4], (uint32_t)v[5], (uint32_t)v[6], (uint32_t)v[7], lo47);
    bytes_t4x((uint32_t)(v[0] >> 32), (uint32_t)(v[1] >> 32), (uint32_t)(v[2] >> 32), (uint32_t)(v[3] >> 32), hi03);
    bytes_t4x((uint32_t)(v[4] >> 32), (uint32_t)(v[5] >> 32), (uint32_t)(v[6] >> 32), (uint32_t)(v[7] >> 32), hi47);
    uint8_t* dst = base + (u64)q * 64 + o * 8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      *reinterpret_cast<uint2*>(dst + i * plane) = make_uint2(lo03[i], lo47[i]);
      *reinterpret_cast<uint2*>(dst + (4 + i) * plane) = make_uint2(hi03[i], hi47[i]);
    }
  }
}

// ITERS channel-runs per thread: CTA = (ITERS * TP * GS / PR) channels x PR pixels, so the plane
// stores cover whole 32 / 64-byte channel rows (cpc = 32 / 64)
template <int ITERS>
__global__ void __launch_bounds__(2 * TP, 1) k_it(const PairArgs A, const PlaneArgs P) {
  constexpr int GS = Geo<W>::GS;
  extern __shared__ u64 smem_all[];
  const int party = threadIdx.x >= TP ? 1 : 0;
  const int t = threadIdx.x - party * TP;
  const int PR = P.PR, tpr = PR / GS, cpi = TP / tpr, cpc = ITERS * cpi, ngrp = P.C / cpc;
  u64* wire = smem_all;
  u64* stage = smem_all + 2 * 2 * PairGeo<W>::SEGW * TP + (u64)party * PR * cpc;
  const u64 cta = blockIdx.x;
  const int rpi = P.HW / PR;
  const int cg = (int)(cta % (u64)ngrp);
  const u64 run = cta / (u64)ngrp;
  const u64 b = run / (u64)rpi;
  const int p0 = (int)(run % (u64)rpi) * PR;
  const int pj = (t % tpr) * GS;
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
    const int ci = it * cpi + t / tpr;
    const int c = cg * cpc + ci;
    const u64 e0 = (b * (u64)P.C + (u64)c) * (u64)P.HW + (u64)(p0 + pj);
    u64 yv[GS];
    if (it) __syncthreads();
    pair_group<W, TP, true>(A, party, t, e0, GS, wire, yv);
    if (P.write_y) store_u64s<GS>(A.io[party].y + e0, GS, yv);
#pragma unroll
    for (int j = 0; j < GS; ++j) stage[(pj + j) * cpc + ci] = yv[j];
  }
  __syncthreads();
  const int oct = cpc / 8;
  const u64 plane = P.B * (u64)P.HW * (u64)P.C;
  const int cb = cg * cpc;
  uint8_t* base = P.planes[party] + (u64)(cb / 64) * (P.B * (u64)P.HW * 64) + (b * (u64)P.HW + (u64)p0) * 64 + (cb % 64);
  for (int it = t; it < PR * oct; it += TP) {
    const int q = it / oct, o = it - q * oct;
    const u64* v = stage + q * cpc + o * 8;
    uint32_t lo03[4], lo47[4], hi03[4], hi47[4];
    bytes_t4x((uint32_t)v[0], (uint32_t)v[1], (uint32_t)v[2], (uint32_t)v[3], lo03);
    bytes_t4x((uint32_t)v[4], (uint32_t)v[5], (uint32_t)v[6], (uint32_t)v[7], lo47);
    bytes_t4x((uint32_t)(v[0] >> 32), (uint32_t)(v[1] >> 32), (uint32_t)(v[2] >> 32), (uint32_t)(v[3] >> 32), hi03);
    bytes_t4x((uint32_t)(v[4] >> 32), (uint32_t)(v[5] >> 32), (uint32_t)(v[6] >> 32), (uint32_t)(v[7] >> 32), hi47);
    uint8_t* dst = base + (u64)q * 64 + o * 8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      *reinterpret_cast<uint2*>(dst + i * plane) = make_uint2(lo03[i], lo47[i]);
      *reinterpret_cast<uint2*>(dst + (4 + i) * plane) = make_uint2(hi03[i], hi47[i]);
    }
  }
}

int main(int argc, char** argv) {
  const u64 B = argc > 1 ? atoll(argv[1]) : 512;
  const int C = argc > 2 ? atoi(argv[2]) : 64;
  const int HW = argc > 3 ? atoi(argv[3]) : 1024;
  const int reps = argc > 4 ? atoi(argv[4]) : 10;
  const u64 n = B * C * HW;
  constexpr int GS = Geo<W>::GS, L = constexpr_levels(W);
  const u64 nb = n * (1 + 2 * L), nbw = (nb * W + 63) / 64;
  PairArgs A;
  for (int p = 0; p < 2; ++p) {
    PartyIO& io = A.io[p];
    io.x = dalloc(n, 1 + p);
    io.y = dalloc(n, 3 + p);
    io.ba = dalloc(nbw, 5 + p);
    io.bb = dalloc(nbw, 7 + p);
    io.bc = dalloc(nbw, 9 + p);
    io.bcur = 0;
    io.bnw = nbw;
    io.aa = dalloc(2 * n, 11 + p);
    io.ab = dalloc(2 * n, 13 + p);
    io.ac = dalloc(2 * n, 15 + p);
    io.acur = 0;
  }
  A.n = n;
  A.first = 0;
  A.count = n;
  A.N = 64;
  A.m = 14;
  A.drelu_only = 0;
  PlaneArgs P;
  cudaMalloc(&P.planes[0], 8 * n);
  cudaMalloc(&P.planes[1], 8 * n);
  P.B = B;
  P.C = C;
  P.HW = HW;
  const size_t smem = sizeof(u64) * 2 * 2 * PairGeo<W>::SEGW * TP;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = 2.0 * n * (8 + 8 + 3.0 * (1 + 2 * L) * W / 8 + 48);
  auto timeit = [&](const char* name, auto launch, double extra) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%-34s %8.3f ms  %7.1f GB/s (alg %.0f B/elem/party)  err=%s\n", name, ms, (bytes + extra) / ms / 1e6,
           (bytes + extra) / 2 / n, cudaGetErrorString(cudaGetLastError()));
  };
  timeit("k_relu_pair", [&] { k_relu_pair<W, TP, true><<<(unsigned)(n / GS / TP), 2 * TP, smem>>>(A); }, 0);
  for (int pr : {32, 16}) {
    P.PR = pr;
    for (int wy : {1, 0}) {
      P.write_y = wy;
      const double ex = 2.0 * n * (8.0 - (wy ? 0 : 8));
      char nm[96];
#define RUN_IT(IT)                                                                                       \
  {                                                                                                      \
    const int cpc = IT * TP * GS / pr;                                                                   \
    if (cpc <= 64 && HW % pr == 0) {                                                                     \
      const unsigned blocks = (unsigned)(B * (HW / pr) * (C / cpc));                                     \
      const size_t sm = smem + 2 * (size_t)pr * cpc * 8;                                                 \
      cudaFuncSetAttribute(k_it<IT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);              \
      snprintf(nm, sizeof nm, "iters=%d PR=%d cpc=%d y=%d", IT, pr, cpc, wy);                           \
      timeit(nm, [&] { k_it<IT><<<blocks, 2 * TP, sm>>>(A, P); }, ex);                                   \
    }                                                                                                    \
  }
      RUN_IT(1) RUN_IT(2) RUN_IT(4) RUN_IT(8)
    }
  }
  if (argc > 5) return 0;
  for (int pr : {32, 16, 8, 4}) {
    P.PR = pr;
    const int cpc = TP * GS / pr;
    if (cpc > 64 || HW % pr) continue;
    const unsigned blocks = (unsigned)(B * (HW / pr) * (C / cpc));
    for (int wy : {1, 0}) {
      P.write_y = wy;
      char nm[96];
      const double ex = 2.0 * n * (8.0 - (wy ? 0 : 8));
      snprintf(nm, sizeof nm, "planes o0 PR=%d y=%d", pr, wy);
      timeit(nm, [&] { k_var<0, true><<<blocks, 2 * TP, smem>>>(A, P); }, ex);
      snprintf(nm, sizeof nm, "planes o1 PR=%d y=%d", pr, wy);
      timeit(nm, [&] { k_var<1, true><<<blocks, 2 * TP, smem>>>(A, P); }, ex);
      snprintf(nm, sizeof nm, "planes o2 PR=%d y=%d", pr, wy);
      timeit(nm, [&] { k_var<2, true><<<blocks, 2 * TP, smem>>>(A, P); }, ex);
      if (wy) {
        snprintf(nm, sizeof nm, "no-store o0 PR=%d", pr);
        timeit(nm, [&] { k_var<0, false><<<blocks, 2 * TP, smem>>>(A, P); }, 0);
        snprintf(nm, sizeof nm, "no-store o1 PR=%d", pr);
        timeit(nm, [&] { k_var<1, false><<<blocks, 2 * TP, smem>>>(A, P); }, 0);
      }
    }
  }
  return 0;
}
