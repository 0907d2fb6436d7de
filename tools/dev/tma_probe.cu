// tma_probe.cu -- standalone check of 3-D u16 TMA tensor loads (zero fill) on this box.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void probe(const __grid_constant__ CUtensorMap tm, const CUtensorMap *gtm, uint16_t *out, int x, int y,
                      int z) {
  __shared__ __align__(1024) uint16_t buf[18 * 128];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t tmp = MODE == 0 ? reinterpret_cast<uint64_t>(&tm) : reinterpret_cast<uint64_t>(gtm);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(18 * 128 * 2)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4}], [%5];" ::"r"(su32(buf)),
        "l"(tmp), "r"(x), "r"(y), "r"(z), "r"(su32(&bar))
        : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
          su32(&bar))
      : "memory");
  for (int i = threadIdx.x; i < 18 * 128; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int cols = 512, rows = 512, frames = 4;
  uint16_t *d, *o;
  cudaMalloc(&d, (size_t)cols * rows * frames * 2);
  cudaMalloc(&o, 18 * 128 * 2);
  uint16_t *h = (uint16_t *)malloc((size_t)cols * rows * frames * 2);
  for (int i = 0; i < cols * rows * frames; ++i) h[i] = (uint16_t)(i % 4093 + 1);
  cudaMemcpy(d, h, (size_t)cols * rows * frames * 2, cudaMemcpyHostToDevice);
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  printf("entry point: %d q=%d fp=%p\n", (int)e, (int)q, fp);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
  CUtensorMap tm;
  const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)frames};
  const cuuint64_t strides[2] = {(cuuint64_t)cols * 2, (cuuint64_t)cols * rows * 2};
  const cuuint32_t box[3] = {128, 18, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  CUtensorMap *gtm;
  cudaMalloc(&gtm, sizeof(CUtensorMap));
  cudaMemcpy(gtm, &tm, sizeof(tm), cudaMemcpyHostToDevice);
  uint16_t ho[18 * 128];
  for (int mode = 0; mode < 2; ++mode) {
    const int xs[7] = {0, 0, -8, 3, 8, -5, 450}, ys[7] = {0, -3, 0, 0, 500, 0, 500};
    for (int c = 0; c < 7; ++c) {
      const int x = xs[c], y = ys[c], z = 1;
      if (mode == 0) probe<0><<<1, 128>>>(tm, gtm, o, x, y, z);
      else probe<1><<<1, 128>>>(tm, gtm, o, x, y, z);
      cudaError_t ke = cudaDeviceSynchronize();
      if (ke != cudaSuccess) {
        printf("mode %d case %d (x=%d y=%d): %s\n", mode, c, x, y, cudaGetErrorString(ke));
        return 1;
      }
      cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int r2 = 0; r2 < 18; ++r2)
        for (int c2 = 0; c2 < 128; ++c2) {
          const int gy = y + r2, gx = x + c2;
          const uint16_t want = (gy >= 0 && gy < rows && gx >= 0 && gx < cols)
                                    ? h[(size_t)z * rows * cols + (size_t)gy * cols + gx]
                                    : 0;
          bad += ho[r2 * 128 + c2] != want;
        }
      printf("mode %d case %d (x=%d y=%d): %d mismatches\n", mode, c, x, y, bad);
    }
  }
  return 0;
}
