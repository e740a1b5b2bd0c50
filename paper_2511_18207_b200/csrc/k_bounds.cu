// k_bounds.cu — f2 bound reporting: delta(u) and H_U on the device.
//
// PAPER.md Eq. (2): delta(u) = max_{p in A u B} ||p - (p^T u) u||, and the
// multi-direction bound Eq. (4): H_U <= H <= H_U + 2 min_u delta(u), with
// H_U = max_{u in U} H_u(A,B), H_u the 1-D Hausdorff distance of the projections
// (P:378-386). delta is reported in both frames: through the
// origin (literal) and centred at the union mean mu (the bound holds for any centre).
//
//   bounds_kernel   one warp per point: ||x||^2, x.mu and pi_l = x.u_l (fp32), per-block
//                   maxima of the two delta^2 terms per direction, each inflated by an
//                   upper bound of its fp32 rounding error so the reported delta is never
//                   below the true one; writes the fp32 projections (order-preserving keys)
//   radix sort      keys only, 4 LSD passes of 8 bits, one segment per direction: per-tile
//                   digit histograms, one-block-per-direction exclusive scan, stable scatter
//                   (warp match_any ranking, tile slots in index order)
//   hu_kernel       h_u(X, Y) = max_x min_y |pi(x) - pi(y)| by binary search of pi(x) in
//                   the sorted pi(Y) (fp64 differences of the fp32 values)
#include "internal.cuh"
#include "prohd_kernels.cuh"

#include <cfloat>

namespace prohd {
namespace {

__device__ __forceinline__ unsigned okey(float f) {
  unsigned u = __float_as_uint(f == 0.0f ? 0.0f : f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float okey_inv(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// per direction: out2[l*2+0] = max delta^2 through the origin, out2[l*2+1] = centred (fp64 bits)
__global__ void __launch_bounds__(256) bounds_kernel(const float* __restrict__ X, int64_t n, int D,
                                                     const float* __restrict__ U32, int L,
                                                     const double* __restrict__ mu, unsigned* __restrict__ keys,
                                                     unsigned long long* out2) {
  extern __shared__ float sm[];  // [L][D] directions, then mu (fp32)
  __shared__ unsigned long long bmax[64];
  __shared__ float umu[32];  // mu . u_l
  float* su = sm;
  float* smu = sm + L * D;
  for (int i = threadIdx.x; i < L * D; i += blockDim.x) su[i] = U32[i];
  for (int i = threadIdx.x; i < D; i += blockDim.x) smu[i] = static_cast<float>(mu[i]);
  for (int i = threadIdx.x; i < 2 * L; i += blockDim.x) bmax[i] = 0ull;
  __syncthreads();
  if (threadIdx.x < L) {
    float acc = 0.0f;
    for (int c = 0; c < D; ++c) acc = fmaf(smu[c], su[threadIdx.x * D + c], acc);
    umu[threadIdx.x] = acc;
  }
  __syncthreads();
  double mun2 = 0.0;
  for (int i = 0; i < D; ++i) mun2 += static_cast<double>(mu[i]) * mu[i];
  const double mun = sqrt(mun2);
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const double g = (4.0 * D + 16.0) * 0x1p-24;  // fp32 rounding-error factor (see header)
  for (int64_t r = warp; r < n; r += nwarps) {
    const float* x = X + r * D;
    float nx = 0.0f, xm = 0.0f;
    for (int c = lane; c < D; c += 32) {
      const float v = __ldg(x + c);
      nx = fmaf(v, v, nx);
      xm = fmaf(v, smu[c], xm);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      nx += __shfl_xor_sync(0xffffffffu, nx, o);
      xm += __shfl_xor_sync(0xffffffffu, xm, o);
    }
    const double xn = sqrt(static_cast<double>(nx));
    for (int l = 0; l < L; ++l) {
      float p = 0.0f;
      for (int c = lane; c < D; c += 32) p = fmaf(__ldg(x + c), su[l * D + c], p);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
      const float um = umu[l];
      if (lane == 0) {
        keys[static_cast<int64_t>(l) * n + r] = okey(p);
        const double pd = p;
        const double d0 = static_cast<double>(nx) - pd * pd + g * static_cast<double>(nx);
        const double pc = pd - static_cast<double>(um);
        const double xc2 = static_cast<double>(nx) - 2.0 * static_cast<double>(xm) + mun2;
        const double d1 = xc2 - pc * pc + g * (xn + mun) * (xn + mun);
        atomicMax(&bmax[2 * l], __double_as_longlong(fmax(d0, 0.0)));
        atomicMax(&bmax[2 * l + 1], __double_as_longlong(fmax(d1, 0.0)));
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * L; i += blockDim.x) atomicMax(&out2[i], bmax[i]);
}

// ------------------------------------------------------------------ radix sort (keys only)
constexpr int kRT = 256;          // threads per tile block
constexpr int kRI = 4;            // keys per thread
constexpr int kTile = kRT * kRI;  // 1024 keys per tile

__global__ void __launch_bounds__(kRT) rs_hist_kernel(const unsigned* __restrict__ in, int64_t n, int shift,
                                                      unsigned* __restrict__ counts, int nblk) {
  __shared__ unsigned h[256];
  const int l = blockIdx.y;
  const unsigned* seg = in + static_cast<int64_t>(l) * n;
  h[threadIdx.x] = 0u;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
  for (int it = 0; it < kRI; ++it) {
    const int64_t i = base + it * kRT + threadIdx.x;
    if (i < n) atomicAdd(&h[(seg[i] >> shift) & 0xFFu], 1u);
  }
  __syncthreads();
  counts[(static_cast<int64_t>(l) * 256 + threadIdx.x) * nblk + blockIdx.x] = h[threadIdx.x];
}

// exclusive scan of the digit-major [256][nblk] counts of one direction, in place
__global__ void __launch_bounds__(1024) rs_scan_kernel(unsigned* counts, int nblk) {
  __shared__ unsigned part[1024];
  unsigned* c = counts + static_cast<int64_t>(blockIdx.x) * 256 * nblk;
  const int64_t tot = static_cast<int64_t>(256) * nblk;
  const int64_t per = (tot + 1023) / 1024;
  const int64_t b0 = threadIdx.x * per, b1 = min(tot, b0 + per);
  unsigned s = 0;
  for (int64_t i = b0; i < b1; ++i) s += c[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const unsigned v = threadIdx.x >= static_cast<unsigned>(o) ? part[threadIdx.x - o] : 0u;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  unsigned run = part[threadIdx.x] - s;
  for (int64_t i = b0; i < b1; ++i) {
    const unsigned v = c[i];
    c[i] = run;
    run += v;
  }
}

__global__ void __launch_bounds__(kRT) rs_scatter_kernel(const unsigned* __restrict__ in, unsigned* __restrict__ out,
                                                         int64_t n, int shift, const unsigned* __restrict__ offs,
                                                         int nblk) {
  __shared__ unsigned slot[kRI * (kRT / 32)][256];
  const int l = blockIdx.y;
  const unsigned* seg = in + static_cast<int64_t>(l) * n;
  unsigned* oseg = out + static_cast<int64_t>(l) * n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kRI * (kRT / 32) * 256; i += kRT) (&slot[0][0])[i] = 0u;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
  unsigned key[kRI], rnk[kRI];
  int dig[kRI];
  for (int it = 0; it < kRI; ++it) {
    const int64_t i = base + it * kRT + threadIdx.x;
    const bool ok = i < n;
    key[it] = ok ? seg[i] : 0u;
    dig[it] = ok ? static_cast<int>((key[it] >> shift) & 0xFFu) : 256;  // 256: no key
    const unsigned peers = __match_any_sync(0xffffffffu, dig[it]);
    rnk[it] = __popc(peers & ((1u << lane) - 1u));
    if (ok && rnk[it] == 0) slot[it * (kRT / 32) + warp][dig[it]] = __popc(peers);
  }
  __syncthreads();
  {  // exclusive prefix over the slots (index order) for digit d = threadIdx.x
    unsigned run = 0;
    for (int s = 0; s < kRI * (kRT / 32); ++s) {
      const unsigned v = slot[s][threadIdx.x];
      slot[s][threadIdx.x] = run;
      run += v;
    }
  }
  __syncthreads();
  for (int it = 0; it < kRI; ++it) {
    if (dig[it] == 256) continue;
    const unsigned pos = offs[(static_cast<int64_t>(l) * 256 + dig[it]) * nblk + blockIdx.x] +
                         slot[it * (kRT / 32) + warp][dig[it]] + rnk[it];
    oseg[pos] = key[it];
  }
}

// h_u(X, Y) per direction: keysX [L][nX] (any order), sortedY [L][nY] ascending keys
__global__ void __launch_bounds__(256) hu_kernel(const unsigned* __restrict__ keysX, int64_t nX,
                                                 const unsigned* __restrict__ sortedY, int64_t nY,
                                                 unsigned long long* out) {
  __shared__ unsigned long long bm;
  const int l = blockIdx.y;
  if (threadIdx.x == 0) bm = 0ull;
  __syncthreads();
  const unsigned* ys = sortedY + static_cast<int64_t>(l) * nY;
  double best = 0.0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nX;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned k = keysX[static_cast<int64_t>(l) * nX + i];
    int64_t lo = 0, hi = nY;  // first position with ys[pos] >= k
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ys[mid] < k)
        lo = mid + 1;
      else
        hi = mid;
    }
    const double x = okey_inv(k);
    double d = DBL_MAX;
    if (lo < nY) d = fmin(d, fabs(static_cast<double>(okey_inv(ys[lo])) - x));
    if (lo > 0) d = fmin(d, fabs(x - static_cast<double>(okey_inv(ys[lo - 1]))));
    best = fmax(best, d);
  }
  atomicMax(&bm, __double_as_longlong(best));
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&out[l], bm);
}

// deterministic fp64 column sums of A and B (mean of the union): per-block partials + fixed reduce
__global__ void __launch_bounds__(256) colsum_kernel(const float* __restrict__ X, int64_t n, int D, int nparts,
                                                     double* __restrict__ part) {
  const int64_t per = (n + nparts - 1) / nparts;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * per, r1 = min(n, r0 + per);
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    double s = 0.0;
    for (int64_t r = r0; r < r1; ++r) s += static_cast<double>(__ldg(X + r * D + c));
    part[static_cast<int64_t>(blockIdx.x) * D + c] = s;
  }
}

__global__ void colmean_kernel(const double* __restrict__ part, int nparts, int D, int64_t N, double* mu) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < D; c += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < nparts; ++p) s += part[static_cast<int64_t>(p) * D + c];
    mu[c] = s / static_cast<double>(N);
  }
}

}  // namespace

cudaError_t launch_union_mean(const float* A, int64_t nA, const float* B, int64_t nB, int D, double* part,
                              double* mu, cudaStream_t st) {
  count_launch();
  colsum_kernel<<<kMeanParts, 256, 0, st>>>(A, nA, D, kMeanParts, part);
  count_launch();
  colsum_kernel<<<kMeanParts, 256, 0, st>>>(B, nB, D, kMeanParts, part + static_cast<int64_t>(kMeanParts) * D);
  count_launch();
  colmean_kernel<<<(D + 255) / 256, 256, 0, st>>>(part, 2 * kMeanParts, D, nA + nB, mu);
  return cudaGetLastError();
}

BoundsPlan plan_bounds(int64_t nA, int64_t nB, int L) {
  BoundsPlan p;
  const int64_t n = nA > nB ? nA : nB;
  p.nblk = static_cast<int>((n + kTile - 1) / kTile);
  p.keys_words = static_cast<int64_t>(L) * n;
  p.count_words = static_cast<int64_t>(L) * 256 * p.nblk;
  return p;
}

static cudaError_t radix_sort_segments(unsigned* keys, unsigned* tmp, int64_t n, int L, unsigned* counts,
                                       cudaStream_t st) {
  const int nblk = static_cast<int>((n + kTile - 1) / kTile);
  unsigned* a = keys;
  unsigned* b = tmp;
  for (int pass = 0; pass < 4; ++pass) {
    count_launch();
    rs_hist_kernel<<<dim3(nblk, L), kRT, 0, st>>>(a, n, 8 * pass, counts, nblk);
    count_launch();
    rs_scan_kernel<<<L, 1024, 0, st>>>(counts, nblk);
    count_launch();
    rs_scatter_kernel<<<dim3(nblk, L), kRT, 0, st>>>(a, b, n, 8 * pass, counts, nblk);
    unsigned* t = a;
    a = b;
    b = t;
  }
  return cudaGetLastError();  // 4 passes: the sorted keys are back in `keys`
}

cudaError_t launch_bounds(const float* A, int64_t nA, const float* B, int64_t nB, int D, const float* U32, int L,
                          const double* mu, const BoundsBufs& b, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(b.delta2, 0, sizeof(unsigned long long) * 2 * L, st);
  if (e != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(b.hu, 0, sizeof(unsigned long long) * 2 * L, st)) != cudaSuccess) return e;
  const size_t smem = sizeof(float) * (L * D + D);
  if ((e = cudaFuncSetAttribute(bounds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem))) != cudaSuccess)
    return e;
  const float* X[2] = {A, B};
  const int64_t n[2] = {nA, nB};
  unsigned* keys[2] = {b.keysA, b.keysB};
  for (int s = 0; s < 2; ++s) {
    int64_t blocks = (n[s] + 7) / 8;
    if (blocks > 148 * 8) blocks = 148 * 8;
    count_launch();
    bounds_kernel<<<static_cast<int>(blocks), 256, smem, st>>>(X[s], n[s], D, U32, L, mu, keys[s], b.delta2);
  }
  // sorted copies: B's keys sorted (for h_u(A,B)), A's keys sorted (for h_u(B,A))
  if ((e = cudaMemcpyAsync(b.sortB, b.keysB, sizeof(unsigned) * L * nB, cudaMemcpyDeviceToDevice, st)) !=
      cudaSuccess)
    return e;
  if ((e = cudaMemcpyAsync(b.sortA, b.keysA, sizeof(unsigned) * L * nA, cudaMemcpyDeviceToDevice, st)) !=
      cudaSuccess)
    return e;
  if ((e = radix_sort_segments(b.sortB, b.tmp, nB, L, b.counts, st)) != cudaSuccess) return e;
  if ((e = radix_sort_segments(b.sortA, b.tmp, nA, L, b.counts, st)) != cudaSuccess) return e;
  count_launch();
  hu_kernel<<<dim3(148, L), 256, 0, st>>>(b.keysA, nA, b.sortB, nB, b.hu);
  count_launch();
  hu_kernel<<<dim3(148, L), 256, 0, st>>>(b.keysB, nB, b.sortA, nA, b.hu + L);
  return cudaGetLastError();
}

}  // namespace prohd
