// Standalone timing harness of the NVLink party kernel (both parties in one launch on one GPU, the
// k_relu_p2p_dual harness) on synthetic shares / triples: the kernel's speed does not depend on the
// values, so this isolates its synchronisation design from the Python stack.  Build (one width):
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
//        -DHB_MICRO_W=8 tools/micro/p2p_bench.cu -o tools/micro/p2p_bench -lcuda
//   ./tools/micro/p2p_bench [logn] [reps] [max_ctas]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2309_04875_b200/csrc/hb_relu_p2p.cuh"

#ifndef HB_MICRO_W
#define HB_MICRO_W 8
#endif
using namespace hb;

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
  if (cudaMalloc(&p, words * 8) != cudaSuccess) {
    fprintf(stderr, "cudaMalloc %llu failed\n", (unsigned long long)words * 8);
    exit(1);
  }
  k_fill<<<1184, 256>>>(p, words, seed);
  return p;
}

int main(int argc, char** argv) {
  constexpr int W = HB_MICRO_W;
  const int logn = argc > 1 ? atoi(argv[1]) : 24;
  const int reps = argc > 2 ? atoi(argv[2]) : 20;
  const int max_ctas = argc > 3 ? atoi(argv[3]) : 0;
  const int sys = argc > 4 ? atoi(argv[4]) : 1;
  const u64 n = 1ull << logn;
  const int L = constexpr_levels(W), R = L + 3;
  const u64 nb = n * (1 + 2 * L), nbw = (nb * W + 63) / 64;
  P2PArgs A[2] = {};
  u64 off[P2P_MAXR], ntiles = 0;
  const u64 rbytes = p2p_layout<W>(n, 0, off, &ntiles);
  int* err;
  cudaMalloc(&err, 4);
  cudaMemset(err, 0, 4);
  uint8_t* recv[2];
  unsigned long long* flags[2];
  for (int p = 0; p < 2; ++p) {
    cudaMalloc(&recv[p], rbytes);
    cudaMalloc(&flags[p], ntiles * 8);
    cudaMemset(recv[p], 0, rbytes);
    cudaMemset(flags[p], 0, ntiles * 8);
  }
  for (int p = 0; p < 2; ++p) {
    PartyIO& io = A[p].io;
    io.x = dalloc(n, 1 + p);
    io.y = dalloc(n, 3 + p);
    io.ba = dalloc(nbw, 10 + p);
    io.bb = dalloc(nbw, 20 + p);
    io.bc = dalloc(nbw, 30 + p);
    io.bcur = 0;
    io.bnw = nbw;
    io.aa = dalloc(2 * n, 40 + p);
    io.ab = dalloc(2 * n, 50 + p);
    io.ac = dalloc(2 * n, 60 + p);
    io.acur = 0;
    A[p].n = n;
    A[p].N = 64;
    A[p].m = 14;
    A[p].party = p;
    A[p].drelu_only = 0;
    A[p].recv = recv[p];
    A[p].my_flag = flags[p];
    A[p].peer_recv = recv[p ^ 1];
    A[p].peer_flag = flags[p ^ 1];
    A[p].timeout_ns = 20ull * 1000000000ull;
    A[p].err = err;
    A[p].wire_bytes = nullptr;
  }
  unsigned long long* stamps = nullptr;
  const size_t nst = 2 * 4 * 32 * P2P_MAXR * 5;
  cudaMalloc(&stamps, nst * 8);
  cudaMemset(stamps, 0, nst * 8);
  for (int p = 0; p < 2; ++p) A[p].stamps = nullptr;
  cudaDeviceSynchronize();
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  u64 seq = 0;
  auto launch = [&]() {
    A[0].seq0 = A[1].seq0 = seq;
    seq += R;
    cudaError_t e = launch_p2p<W>(A[0], &A[1], max_ctas, 0, sys, s);
    if (e != cudaSuccess) {
      fprintf(stderr, "launch: %s\n", cudaGetErrorString(e));
      exit(1);
    }
  };
  for (int i = 0; i < 3; ++i) launch();
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  // one more launch with phase stamps (CTAs 0..3 of each party, first 32 tiles)
  for (int p = 0; p < 2; ++p) A[p].stamps = stamps;
  launch();
  cudaStreamSynchronize(s);
  std::vector<unsigned long long> hs(nst);
  cudaMemcpy(hs.data(), stamps, nst * 8, cudaMemcpyDeviceToHost);
  // per round: [0] enter exchange, [1] after bar 1, [2] after release, [3] flag seen + acquire, [4] after bar 2
  double ph[P2P_MAXR][5] = {}, cnt[P2P_MAXR] = {};
  for (int sl = 0; sl < 8; ++sl)
    for (int i = 2; i < 30; ++i) {
      const unsigned long long* q = hs.data() + (sl * 32 + i) * (P2P_MAXR * 5);
      if (!q[0] || !q[(R - 1) * 5 + 4]) continue;
      for (int r = 0; r < R; ++r) {
        const unsigned long long* z = q + r * 5;
        const unsigned long long prev = r ? q[(r - 1) * 5 + 4] : 0;
        if (r) ph[r][0] += (double)(z[0] - prev);
        for (int k = 1; k < 5; ++k) ph[r][k] += (double)(z[k] - z[k - 1]);
        cnt[r] += 1;
      }
    }
  printf("phase ns per round (mean over sampled tiles): compute->enter | bar1 | release | wait-peer | bar2\n");
  for (int r = 0; r < R; ++r)
    printf("  r%d: %7.0f %7.0f %7.0f %7.0f %7.0f\n", r, ph[r][0] / cnt[r], ph[r][1] / cnt[r], ph[r][2] / cnt[r],
           ph[r][3] / cnt[r], ph[r][4] / cnt[r]);
  int herr = 0;
  cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost);
  const double per = ms / reps;
  const double wire = (2.0 * W + 4.0 * L * W) / 8 + 32;
  const double H = 16 + 3.0 * (1 + 2 * L) * W / 8 + 48 + 2 * wire;
  const double eps = n / (per * 1e-3);
  printf("{\"sys\": %d, \"W\": %d, \"logn\": %d, \"ms\": %.4f, \"elems_per_s\": %.4g, \"hbm_GBps\": %.1f, \"H\": %.1f, "
         "\"err\": %d, \"status\": \"%s\"}\n",
         sys, W, logn, per, eps, 2 * H * eps / 1e9, H, herr, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
