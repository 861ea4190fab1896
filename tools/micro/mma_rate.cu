// tcgen05.mma kind::i8 issue-rate microbenchmark (1 CTA per SM, 148 CTAs): cycles per MMA for
// different N and accumulator-overlap patterns.  Operands are whatever is in shared memory.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2309_04875_b200/csrc/hb_tc_ptx.cuh"
using namespace hb::tc;

// pattern 0: all MMAs write cols [0, N) (plain K loop); 1: stacked shift pattern (limb i -> cols i*64, N = 2*64);
// 2: 8 independent regions (MMA i -> cols i*64, N = 64); 3: stacked pattern with N=64 (i,j) pairs
template <int PAT, int N>
__global__ void __launch_bounds__(128, 1) k_mma(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bars[4];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1); asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    const uint64_t da = sdesc_k<64>(a), db = sdesc_k<64>(b);
    t0 = clock64();
    int nmma = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (PAT == 0) {
          mma_i8(tmem, da + (i * 512), db, idesc_i8(N), 1u);
        } else if (PAT == 1) {
          mma_i8(tmem + i * 64, da + (i * 512), db, idesc_i8(i == 7 ? 64 : 128), 1u);
        } else if (PAT == 2) {
          mma_i8(tmem + i * 64, da + (i * 512), db, idesc_i8(64), 1u);
        } else if (PAT >= 4) {
          mma_i8(tmem + i * 64, da + (i * 512), db, idesc_i8(i == 7 ? 64 : 128), 1u);
        } else {
          mma_i8(tmem + i * 64, da + (i * 512), db, idesc_i8(64), 1u);
          if (i < 7) mma_i8(tmem + (i + 1) * 64, da + (i * 512), db + 256, idesc_i8(64), 1u);
        }
      }
      nmma += 8;
      if (PAT >= 4) {  // kernel-like stage handoff: commit per group, wait for the group 3 back
        if (PAT == 5) tc_fence_after();
        mma_commit(&bars[it & 3]);
        if (it >= 3) mbar_wait(&bars[(it - 3) & 3], ((it - 3) >> 2) & 1);
        if (PAT == 5) tc_fence_after();
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int PAT, int N>
void run(const char* name, double macs_per_iter) {
  long long* d; cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k_mma<PAT, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 2000;
  k_mma<PAT, N><<<148, 128, 200 * 1024>>>(10, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_mma<PAT, N><<<148, 128, 200 * 1024>>>(iters, d);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("%-40s %8.1f clk per 8-MMA group  -> %6.0f MAC/clk/SM (peak 8192)  %.2f int8 POPS (wall)  %s\n", name,
         avg / iters, macs_per_iter / (avg / iters), 2.0 * 148 * iters * macs_per_iter / (ms * 1e-3) / 1e15,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0, 64>("same D, N=64 x8", 8.0 * 128 * 64 * 32);
  run<0, 128>("same D, N=128 x8", 8.0 * 128 * 128 * 32);
  run<0, 256>("same D, N=256 x8", 8.0 * 128 * 256 * 32);
  run<1, 128>("stacked shifts (7xN=128 + N=64)", (7.0 * 128 + 64) * 128 * 32);
  run<2, 64>("8 disjoint regions N=64", 8.0 * 128 * 64 * 32);
  run<3, 64>("(i,j) pairs N=64 (15 MMAs)", 15.0 * 128 * 64 * 32);
  run<4, 128>("stacked + commit/wait per group", (7.0 * 128 + 64) * 128 * 32);
  run<5, 128>("stacked + commit/wait + fences", (7.0 * 128 + 64) * 128 * 32);
  return 0;
}
