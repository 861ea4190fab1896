// Latency of a system-scope release (MEMBAR.SYS) vs gpu scope, idle and under background HBM load.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k_probe(unsigned long long* buf, unsigned long long* out, int iters, int scope, int nstores) {
  // one warp: each lane stores nstores words, then lane 0 releases a flag; time the release
  unsigned long long acc = 0;
  for (int i = 0; i < iters; ++i) {
    for (int k = 0; k < nstores; ++k) buf[((size_t)blockIdx.x * 4096 + (i * nstores + k) % 4096) * 32 % (1 << 20) + threadIdx.x] = i;
    __syncwarp();
    if (threadIdx.x == 0) {
      unsigned long long t0 = gt();
      if (scope == 0) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(buf + (1 << 20) + blockIdx.x * 8), "l"((unsigned long long)i) : "memory");
      else asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(buf + (1 << 20) + blockIdx.x * 8), "l"((unsigned long long)i) : "memory");
      acc += gt() - t0;
    }
    __syncwarp();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc / iters;
}
__global__ void k_load(const uint4* src, uint4* dst, size_t n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) dst[i] = src[i];
}
int main() {
  unsigned long long *buf, *out;
  cudaMalloc(&buf, 64 << 20);
  cudaMalloc(&out, 4096 * 8);
  size_t nb = 1ull << 30;
  uint4 *src, *dst;
  cudaMalloc(&src, nb);
  cudaMalloc(&dst, nb);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  for (int scope = 0; scope < 2; ++scope)
    for (int nb_ : {1, 16, 148, 592, 1184}) {
      k_probe<<<nb_, 32, 0, s1>>>(buf, out, 200, scope, 1);
      cudaDeviceSynchronize();
      unsigned long long h[4096];
      cudaMemcpy(h, out, 8 * nb_, cudaMemcpyDeviceToHost);
      double m = 0;
      for (int i = 0; i < nb_; ++i) m += h[i];
      printf("scope=%s concurrent warps=%d : release %.0f ns (mean)\n", scope ? "gpu" : "sys", nb_, m / nb_);
    }
  return 0;
}
