// mma_probe.cu -- issue-rate microbenchmark for tcgen05.mma kind::i8 (M=128, K=32)
// with no-swizzle K-major shared-memory operands, as the coarse search uses them.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_1506_06039_b200/csrc \
//      -o dbg_so/mma_probe tools/mma_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "kernels_tc.cuh"

using namespace moco;

// mode 0: plain MMAs; 1: + commit every 4; 2: + commit every 4 and wait for the commit
// 7 groups back; 3: + a try_wait on an already-completed barrier every 4 MMAs
__global__ void probe(int N, int mode, int reps, unsigned long long *out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 200 * 1024);
  uint64_t *cb = bar + 1;   // [8] commit targets
  uint64_t *done = bar + 9;
  uint32_t *holder = reinterpret_cast<uint32_t *>(bar + 10);
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = i * 2654435761u;
  if (threadIdx.x < 32) tmem_alloc(holder, 512);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(done, 1);
    for (int i = 0; i < 8; ++i) mbar_init(&cb[i], 1);
    fence_mbar_init();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(done);   // phase 0 of `done` completes now
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = *holder;
  if (threadIdx.x < 32) {
    const uint32_t idesc = idesc_i8(128, N);
    const uint64_t bd = umma_desc(smem_u32(sm + 160 * 1024), 128, 256);
    const uint64_t ad = umma_desc(smem_u32(sm), 20480, 128);
    const uint32_t alo0 = (uint32_t)ad, ahi = (uint32_t)(ad >> 32), blo = (uint32_t)bd, bhi = (uint32_t)(bd >> 32);
    const uint32_t t0c = taddr, t1c = taddr + (uint32_t)N;
    __syncwarp();
    const unsigned long long t0 = clock64();
    uint32_t alo = alo0;
    for (int g = 0; g < reps / 4; ++g) {
      if (mode == 3) mbar_wait(done, 0);
      const uint32_t acc = g ? 1u : 0u;
      mma_i8_x2_elect(t0c, t1c, alo, alo + 128, ahi, blo, bhi, idesc, acc);
      mma_i8_x2_elect(t0c, t1c, alo + 8, alo + 136, ahi, blo + 256, bhi, idesc, acc);
      alo = alo0 + ((alo - alo0 + 16) & 1023);
      if (mode >= 1 && (mode != 4 || (g & 1))) {   // mode 4: commit every 8 MMAs (2 groups)
        const int c = mode == 4 ? g >> 1 : g;
        mma_commit_elect(&cb[c & 7]);
        __syncwarp();
        if ((mode == 2 || mode == 4) && c >= 7) mbar_wait(&cb[(c - 7) & 7], ((c - 7) >> 3) & 1);
        if (mode == 4) {
          mbar_wait(done, 0);
          tc_fence_after();
        }
      }
    }
    mma_commit_elect(bar);
    mbar_wait(bar, 0);
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(taddr, 512);
}

int main() {
  unsigned long long *d, h[148];
  cudaMalloc(&d, sizeof(h));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 201 * 1024);
  const int reps = 4096;
  const int Ns[4] = {64, 128, 192, 256};
  for (int mode = 0; mode < 5; ++mode)
    for (int ni = 1; ni < 4; ++ni) {
      const int N = Ns[ni], grid = 148;
      probe<<<grid, 128, 201 * 1024>>>(N, mode, reps, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(h, d, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("N %3d mode %d: %.1f cyc/MMA (floor %d)\n", N, mode, mx / reps, 128 * N / 256);
      fflush(stdout);
    }
  return 0;
}
