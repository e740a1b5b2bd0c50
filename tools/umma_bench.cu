// Dev microbenchmark: back-to-back tcgen05.mma issue rate on this B200 (no TMA, operands resident
// in shared memory), M=128, N in {64, 128, 256}, kind::tf32 (K=8) and kind::f16 bf16 (K=16), one
// accumulator, one CTA per SM. Prints SM cycles per MMA and the implied dense TFLOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_18207_b200/csrc \
//        -o /tmp/umma tools/umma_bench.cu -lcuda && /tmp/umma
#include <cstdio>
#include "sm100.cuh"

using namespace prohd::sm100;

template <int KIND, int N>
__global__ void __launch_bounds__(128, 1) umma_kernel(int iters, long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* A = smem;               // 128 rows x 128 B
  uint8_t* B = smem + 128 * 128;   // N rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (128 + N) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) tmem_alloc<256>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = KIND == 0 ? idesc_tf32(128, N) : idesc_bf16(128, N);
    const uint32_t a = smem_u32(A), b = smem_u32(B);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t da = smem_desc_k_sw128(a + kk * 32), db = smem_desc_k_sw128(b + kk * 32);
        if (KIND == 0)
          mma_tf32(d, da, db, idesc, 1u);
        else
          mma_bf16(d, da, db, idesc, 1u);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<256>(d);
  }
}

template <int KIND, int N>
void run(const char* name) {
  long long* dc;
  cudaMalloc(&dc, 148 * sizeof(long long));
  const int iters = 4096;
  const size_t smem = 1024 + (128 + N) * 128;
  cudaFuncSetAttribute(umma_kernel<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  umma_kernel<KIND, N><<<148, 128, smem>>>(16, dc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  umma_kernel<KIND, N><<<148, 128, smem>>>(iters, dc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long hc[148];
  cudaMemcpy(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < 148; ++i) mean += hc[i];
  mean /= 148;
  const double nmma = 4.0 * iters;
  const double k = KIND == 0 ? 8 : 16;
  const double flops = 2.0 * 128 * N * k * nmma * 148;
  printf("%-5s N=%3d: %.1f SM cycles per MMA, %.1f dense TFLOP/s (%.3f ms) %s\n", name, N, mean / nmma,
         flops / (ms / 1e3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(dc);
}

int main() {
  run<0, 64>("tf32");
  run<0, 128>("tf32");
  run<0, 256>("tf32");
  run<1, 64>("bf16");
  run<1, 128>("bf16");
  run<1, 256>("bf16");
  return 0;
}
