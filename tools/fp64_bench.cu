// Dev microbenchmark: fp64 vector throughput/latency on this B200 (DFMA, DADD, sqrt, div).
#include <cstdio>
__global__ void thr(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void lat(double* out, int iters, long long* cyc) {
  double a = threadIdx.x * 1e-3 + 1.0, q = 1.5;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) a = fma(a, 1.0000001, 1e-9);
  long long t1 = clock64();
  for (int it = 0; it < iters; ++it) q = sqrt(q + 1.0);
  long long t2 = clock64();
  for (int it = 0; it < iters; ++it) q = 1.0 / (q + 1.0);
  long long t3 = clock64();
  double f = a;
  for (int it = 0; it < iters; ++it) f = __shfl_xor_sync(0xffffffffu, f, 1) + 1.0;
  long long t4 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
  out[threadIdx.x] = a + q + f;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 148 * 1024 * 8 * 4); cudaMallocManaged(&c, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w : {1, 4, 8, 32}) {
    int it = 20000;
    thr<<<148, 32 * w>>>(o, 10);
    cudaEventRecord(e0); thr<<<148, 32 * w>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA throughput, %2d warps/SM: %.2f TFLOP/s\n", w, 148.0 * 32 * w * it * 8 * 2 / ms / 1e9);
  }
  lat<<<1, 32>>>(o, 1000, c); cudaDeviceSynchronize();
  printf("latency per op (cycles): DFMA %.1f  sqrt %.1f  div %.1f  shfl64+dadd %.1f\n", c[0] / 1000.0,
         c[1] / 1000.0, c[2] / 1000.0, c[3] / 1000.0);
  return 0;
}
