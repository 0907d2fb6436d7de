// tma_probe2.cu -- 4-D u16 tensor map over frames with reordered dimensions
// {8 columns (contiguous), rows (stride pitch), 8-column chunks (stride 16 B), frames}: one
// box {8, R, C, 1} lands in shared memory as [chunk][row][16 B] (the UMMA core-matrix
// layout), zero filled outside.  Checks the bytes against the host copy.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o dbg_so/tma_probe2 tools/tma_probe2.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
constexpr int R = 26, C = 8;

__global__ void probe(const __grid_constant__ CUtensorMap tm, uint16_t *out, int x, int y, int z) {
  __shared__ __align__(1024) uint16_t buf[8 * R * C];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(8 * R * C * 2)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4, %5}], [%6];" ::"r"(su32(buf)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(y), "r"(x), "r"(z), "r"(su32(&bar))
        : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
          su32(&bar))
      : "memory");
  for (int i = threadIdx.x; i < 8 * R * C; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int cols = 512, rows = 512, frames = 3;
  uint16_t *d, *o;
  cudaMalloc(&d, (size_t)cols * rows * frames * 2);
  cudaMalloc(&o, 8 * R * C * 2);
  uint16_t *h = (uint16_t *)malloc((size_t)cols * rows * frames * 2);
  for (int i = 0; i < cols * rows * frames; ++i) h[i] = (uint16_t)(i * 2654435761u >> 20);
  cudaMemcpy(d, h, (size_t)cols * rows * frames * 2, cudaMemcpyHostToDevice);
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
  CUtensorMap tm;
  const cuuint64_t dims[4] = {8, (cuuint64_t)rows, (cuuint64_t)(cols / 8), (cuuint64_t)frames};
  const cuuint64_t strides[3] = {(cuuint64_t)cols * 2, 16, (cuuint64_t)cols * rows * 2};
  const cuuint32_t box[4] = {8, R, C, 1}, es[4] = {1, 1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  if (r != CUDA_SUCCESS) return 1;
  uint16_t ho[8 * R * C];
  const int xs[5] = {0, -2, 60, 3, 10}, ys[5] = {0, -5, 500, 7, 100};
  for (int c = 0; c < 5; ++c) {
    const int x = xs[c], y = ys[c], z = 1;
    probe<<<1, 128>>>(tm, o, x, y, z);
    cudaError_t ke = cudaDeviceSynchronize();
    if (ke != cudaSuccess) {
      printf("case %d: %s\n", c, cudaGetErrorString(ke));
      return 1;
    }
    cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int ch = 0; ch < C; ++ch)
      for (int rr = 0; rr < R; ++rr)
        for (int e = 0; e < 8; ++e) {
          const int gy = y + rr, gx = (x + ch) * 8 + e;
          const uint16_t want = (gy >= 0 && gy < rows && x + ch >= 0 && x + ch < cols / 8)
                                    ? h[(size_t)z * rows * cols + (size_t)gy * cols + gx]
                                    : 0;
          bad += ho[(ch * R + rr) * 8 + e] != want;
        }
    printf("case %d (chunk x=%d, row y=%d): %d mismatches\n", c, x, y, bad);
  }
  return 0;
}
