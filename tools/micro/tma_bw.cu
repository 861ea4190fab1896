// TMA load throughput microbenchmark: 148 CTAs each stream boxes of a 3-D uint8 tensor into a
// smem ring (no consumer work).  Reports bytes/clk/SM and TB/s vs inner box bytes and box rows.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2309_04875_b200/csrc/hb_tc_ptx.cuh"
using namespace hb::tc;

__global__ void k_tma(const __grid_constant__ CUtensorMap tmap, int iters, int box_bytes, int nst, int rows_per_box,
                      int nrowblocks, int inner_blocks) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int it = 0; it < iters; ++it) {
    const int st = it % nst;
    if (it >= nst) mbar_wait(&bar[st], ((it / nst) - 1) & 1);
    mbar_expect_tx(&bar[st], box_bytes);
    const int blk = (blockIdx.x * 7919 + it * 104729) % (nrowblocks * inner_blocks);
    const int c0 = (blk % inner_blocks), r0 = (blk / inner_blocks) * rows_per_box;
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            smem_u32(smem + st * box_bytes)),
        "l"(&tmap), "r"(0), "r"(r0), "r"(c0), "r"(smem_u32(&bar[st]))
        : "memory");
  }
  for (int it = iters - nst; it < iters; ++it) mbar_wait(&bar[it % nst], (it / nst) & 1);
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  const size_t total = 1ull << 30;  // 1 GiB tensor (L2 misses) or small (L2 hits)
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int l2res : {1, 0}) {
    for (int inner : {32, 64, 128}) {
      for (int rows : {128, 256}) {
        // tensor (inner, R rows, C blocks) with row pitch = inner * C blocks
        const int box_bytes = inner * rows;  // one "limb" box
        const size_t span = l2res ? (32ull << 20) : total;  // 32 MB working set stays in L2
        const int cblocks = 8;
        const size_t R = span / ((size_t)inner * cblocks);
        CUtensorMap tmap;
        cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)R, (cuuint64_t)cblocks};
        cuuint64_t strides[2] = {(cuuint64_t)inner * cblocks, (cuuint64_t)inner};
        // dim1 stride = inner*cblocks (row pitch), dim2 stride = inner (block within row)
        cuuint32_t box[3] = {(cuuint32_t)inner, (cuuint32_t)rows, 1};
        cuuint32_t es[3] = {1, 1, 1};
        CUtensorMapSwizzle sw = inner == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : inner == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
        CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, buf, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
        const int nst = (200 * 1024) / box_bytes > 8 ? 8 : (200 * 1024) / box_bytes;
        const int smem = nst * box_bytes + 1024;
        cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int iters = 4000;
        const int nrowblocks = (int)(R / rows);
        k_tma<<<148, 32, smem>>>(tmap, 100, box_bytes, nst, rows, nrowblocks, cblocks);
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        k_tma<<<148, 32, smem>>>(tmap, iters, box_bytes, nst, rows, nrowblocks, cblocks);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double bytes = 148.0 * iters * box_bytes;
        printf("%s inner %3d rows %3d stages %d: %.2f TB/s  %.1f B/clk/SM (at %d MHz)  err=%s\n", l2res ? "L2 " : "HBM", inner, rows, nst,
               bytes / ms / 1e9, bytes / 148 / (ms * 1e-3 * clk * 1e3), clk / 1000, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
