// Dev microbenchmark: cost of cluster-wide barriers (cg::cluster_group::sync) and of
// __syncthreads for the eigen-solver design. nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
template <int CL>
__global__ void __cluster_dims__(CL, 1, 1) kcl(int iters, double* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double x;
  if (threadIdx.x == 0) x = 0;
  cl.sync();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) *cl.map_shared_rank(&x, (cl.block_rank() + 1) % CL) += 1.0;
    cl.sync();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = x;
}
__global__ void kbs(int iters, double* out) {
  __shared__ double x;
  if (threadIdx.x == 0) x = 0;
  __syncthreads();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) x += 1.0;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = x;
}
int main() {
  double* o;
  cudaMalloc(&o, 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int it = 10000;
  float ms;
  for (int t : {256, 1024}) {
    kcl<8><<<8, t>>>(10, o);
    cudaEventRecord(a); kcl<8><<<8, t>>>(it, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("cluster8 sync, %d thr: %.3f us\n", t, ms * 1e3 / it);
    kcl<2><<<2, t>>>(10, o);
    cudaEventRecord(a); kcl<2><<<2, t>>>(it, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("cluster2 sync, %d thr: %.3f us\n", t, ms * 1e3 / it);
    kbs<<<1, t>>>(10, o);
    cudaEventRecord(a); kbs<<<1, t>>>(it, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("syncthreads, %d thr: %.3f us\n", t, ms * 1e3 / it);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
