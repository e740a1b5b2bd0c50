// Dev microbenchmark: fp64 tensor (DMMA) throughput on this B200, register-only loops.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma tools/dmma_peak.cu && /tmp/dmma
#include <cstdio>
__global__ void k(double* out, int iters) {
  double a[8], b[4], c[4][4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001 + i;
  for (int i = 0; i < 4; ++i) b[i] = threadIdx.x * 0.002 + i;
  for (int j = 0; j < 4; ++j) for (int i = 0; i < 4; ++i) c[j][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
      : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int j = 0; j < 4; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k4(double* out, int iters) {
  double a[4], b[4], c[4][4][2];
  for (int i = 0; i < 4; ++i) { a[i] = threadIdx.x * 0.001 + i; b[i] = threadIdx.x * 0.002 + i; }
  for (int j = 0; j < 4; ++j) for (int i = 0; i < 4; ++i) c[j][i][0] = c[j][i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[j][i][0]), "+d"(c[j][i][1]) : "d"(a[i]), "d"(b[j]));
  }
  double s = 0; for (int j = 0; j < 4; ++j) for (int i = 0; i < 4; ++i) s += c[j][i][0] + c[j][i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* o; cudaMalloc(&o, 148 * 8 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 1; w <= 16; w *= 2) {
    int it = 4096;
    k<<<148 * 4, 32 * w>>>(o, 16); k4<<<148*4, 32*w>>>(o, 16);
    cudaEventRecord(e0); k<<<148 * 4, 32 * w>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 148.0 * 4 * w * it * 4 * (16.0 * 8 * 16 * 2);
    printf("m16n8k16 warps/CTA=%d (4 CTA/SM): %.2f TFLOP/s\n", w, fl / ms / 1e9);
    cudaEventRecord(e0); k4<<<148 * 4, 32 * w>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 148.0 * 4 * w * it * 16 * (8.0 * 8 * 4 * 2);
    printf("m8n8k4   warps/CTA=%d (4 CTA/SM): %.2f TFLOP/s\n", w, fl / ms / 1e9);
  }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
