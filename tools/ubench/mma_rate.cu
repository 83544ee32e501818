// Microbenchmark: back-to-back tcgen05.mma.kind::i8 issue rate from shared
// memory (no TMA, no epilogue) -- the per-SM ceiling the pair GEMM's
// "tensor pipe active" fraction is measured against.  Development tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I../../paper_2506_11277_b200/csrc mma_rate.cu -o mma_rate
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include "ozgpu_ptx.cuh"

using namespace ozgpu;

template <int N>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, int nk, unsigned long long* cycles,
                                                   int fill) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;              // 128 x 128 bytes per k-block, nk blocks
  uint8_t* sB = smem + nk * 16384; // N x 128 bytes per k-block
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < nk * (16384 + N * 128); i += blockDim.x)
    smem[i] = fill ? static_cast<uint8_t>((i * 2654435761u) >> 24) : 0;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc(&holder, 256 >= N ? 256 : 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  if (warp == 0) {
    constexpr uint32_t idesc = idesc_i8<128, N>();
    const uint64_t ad0 = sdesc_sw128(smem_addr(sA));
    const uint64_t bd0 = sdesc_sw128(smem_addr(sB));
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
        for (int kb = 0; kb < nk; ++kb) {
          const uint64_t ad = ad0 + static_cast<uint64_t>(kb * (16384 >> 4));
          const uint64_t bd = bd0 + static_cast<uint64_t>(kb * ((N * 128) >> 4));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) tc_mma_i8(tmem, ad + 2 * kk, bd + 2 * kk, idesc, (it | kb | kk) != 0);
        }
      }
      __syncwarp();
    }
    if (elect_one()) tc_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256 >= N ? 256 : 512);
  }
}

template <int N>
void run(int iters, int nk, int fill) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = nk * (16384 + N * 128) + 1024;
  cudaFuncSetAttribute(mma_loop<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mma_loop<N><<<148, 128, smem>>>(10, nk, d, fill);
  cudaEventRecord(e0);
  mma_loop<N><<<148, 128, smem>>>(iters, nk, d, fill);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < 148; ++i) mean += h[i];
  mean /= 148;
  const double mmas = static_cast<double>(iters) * nk * 4;
  const double ideal = 128.0 * N / 256.0;  // cycles per 128xNx32 MMA at 8192 int8 MAC/clk/SM
  const double ops = 2.0 * 128 * N * 32 * mmas * 148;
  printf("N=%d nk=%d fill=%d: %.1f cycles/MMA (ideal %.0f, %.1f%%), %.0f TOPS, %.3f ms, err=%s\n", N, nk,
         fill, mean / mmas, ideal, 100.0 * ideal / (mean / mmas), ops / (ms * 1e-3) / 1e12, ms,
         cudaGetErrorString(err));
  cudaFree(d);
}

int main(int argc, char** argv) {
  if (argc > 1) {  // long run: power-capped steady state
    const int iters = atoi(argv[1]);
    run<256>(iters, 4, 1);
    run<256>(iters, 4, 0);
    return 0;
  }
  run<256>(2000, 4, 0);
  run<256>(2000, 4, 1);
  run<128>(2000, 4, 1);
  run<256>(2000, 2, 1);
  run<256>(20000, 4, 1);
  return 0;
}
