// k_prep.cu — K0 operand preparation, K7 row-max key and fp64 witness search.
//
// K0 (SURVEY.md §2f, §8(a) "Centering"): per point, y = x - c (fp64, c the pair's
// common centre), hi = rn_tf32(fp32(y)) (rounded to nearest, ties to even, to 11
// significant bits with the low 13 mantissa bits zero, so the tensor core reads hi
// exactly whatever its fp32->tf32 conversion mode, and |lo| <= 2^-11 |y|),
// lo = fp32(y - hi) (exact in fp32), and ||y||^2 accumulated in fp64 then rounded to fp32 (without
// a centre: y = x and lo = x - hi exactly). K6 takes a.b = hi_a.hi_b (TF32 MMA) +
// [hi_a lo_a].[lo_b hi_b] (one bf16 MMA over interleaved pairs), so K0 writes hi (fp32) and
// the bf16 pairs in both orders: pr[f] = (bf16(hi_f), bf16(lo_f)) for the row role and
// pc[f] = (bf16(lo_f), bf16(hi_f)) for the column role (element 2f at the lower address).
// One warp per row; HBM-bound.
//
// K7: the directed maximum over row minima packed as
//   key = (float_bits(d2) << 32) | (0xFFFFFFFF - row)
// (d2 >= 0, so the float's bit pattern orders like its value; the complement
// makes the LOWEST row win ties), then the witness column is recomputed in fp64
// direct form sum_k (a_k - b_k)^2 over all of B (lowest index on exact ties),
// matching the oracle's definition (Eq. (1)).
#include "internal.cuh"

#include <cuda_bf16.h>

#include <cfloat>
#include <cmath>

namespace prohd {

// Round to nearest TF32 (ties to even) by integer carry into bit 13; a value that would
// round past FLT_MAX (to the inf pattern) keeps its truncation instead, so a finite x
// always gives a finite hi. NaN/inf pass through truncated (they are flagged by the norm).
__device__ __forceinline__ float tf32_rn(float x) {
  const uint32_t b = __float_as_uint(x);
  const uint32_t r = (b + 0xFFFu + ((b >> 13) & 1u)) & 0xFFFFE000u;
  const bool keep = ((b & 0x7F800000u) == 0x7F800000u) || ((r & 0x7F800000u) == 0x7F800000u);
  return __uint_as_float(keep ? (b & 0xFFFFE000u) : r);
}

__device__ __forceinline__ uint32_t bf16_pair(float first, float second) {
  const uint32_t a = __bfloat16_as_ushort(__float2bfloat16_rn(first));
  const uint32_t b = __bfloat16_as_ushort(__float2bfloat16_rn(second));
  return a | (b << 16);
}

template <bool kGather, bool kCentre, bool kSplit3>
__global__ void __launch_bounds__(256) prep_kernel(const float* __restrict__ X, const int64_t* __restrict__ idx,
                                                   int64_t n, int D, int Dp, int64_t n_pad,
                                                   const double* __restrict__ centre, float* __restrict__ hi,
                                                   uint32_t* __restrict__ pr, uint32_t* __restrict__ pc,
                                                   float* __restrict__ norms, int* bad) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_pad; r += nwarps) {
    if (r >= n) {
      if (lane == 0) norms[r] = __int_as_float(0x7f800000);
      continue;
    }
    const int64_t src = kGather ? idx[r] : r;
    const float* x = X + src * static_cast<int64_t>(D);
    float* h = hi + r * static_cast<int64_t>(Dp);
    uint32_t* qr = pr + r * static_cast<int64_t>(Dp);
    uint32_t* qc = pc + r * static_cast<int64_t>(Dp);
    double s = 0.0;
    for (int c = lane; c < Dp; c += 32) {
      const float v = c < D ? __ldg(x + c) : 0.0f;
      if (kCentre) {
        const double y = c < D ? static_cast<double>(v) - __ldg(centre + c) : 0.0;
        const float vh = tf32_rn(static_cast<float>(y));
        const float vl = static_cast<float>(y - static_cast<double>(vh));
        h[c] = vh;
        qr[c] = kSplit3 ? __float_as_uint(vl) : bf16_pair(vh, vl);
        qc[c] = kSplit3 ? __float_as_uint(vl) : bf16_pair(vl, vh);
        s = fma(y, y, s);
      } else {
        const float vh = tf32_rn(v);
        const float vl = v - vh;
        h[c] = vh;
        qr[c] = kSplit3 ? __float_as_uint(vl) : bf16_pair(vh, vl);
        qc[c] = kSplit3 ? __float_as_uint(vl) : bf16_pair(vl, vh);
        s = fma(static_cast<double>(v), static_cast<double>(v), s);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const float f = static_cast<float>(s);
      norms[r] = f;
      if (!isfinite(s) || !isfinite(f)) atomicExch(bad, 1);
    }
  }
}

static int grid_for_rows(int64_t rows) {
  int64_t blocks = (rows + 7) / 8;  // 8 warps per block, one row per warp
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  return static_cast<int>(blocks);
}

cudaError_t launch_prep(const float* X, int64_t n, int D, int Dp, int64_t n_pad, const double* centre, float* hi,
                        uint32_t* pr, uint32_t* pc, float* norms, int* bad, cudaStream_t st) {
  count_launch();
  const int g = grid_for_rows(n_pad);
  const bool s3 = k6_split3();
  if (centre && s3)
    prep_kernel<false, true, true><<<g, 256, 0, st>>>(X, nullptr, n, D, Dp, n_pad, centre, hi, pr, pc, norms, bad);
  else if (centre)
    prep_kernel<false, true, false><<<g, 256, 0, st>>>(X, nullptr, n, D, Dp, n_pad, centre, hi, pr, pc, norms, bad);
  else if (s3)
    prep_kernel<false, false, true><<<g, 256, 0, st>>>(X, nullptr, n, D, Dp, n_pad, nullptr, hi, pr, pc, norms, bad);
  else
    prep_kernel<false, false, false><<<g, 256, 0, st>>>(X, nullptr, n, D, Dp, n_pad, nullptr, hi, pr, pc, norms, bad);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- K7a row-max key
__device__ __forceinline__ unsigned long long shfl_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

__global__ void __launch_bounds__(256) rowmax_key_kernel(const float* __restrict__ rowmin, int64_t n,
                                                         int64_t row_offset, unsigned long long* key) {
  __shared__ unsigned long long sm[8];
  unsigned long long best = 0ull;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float d2 = fmaxf(rowmin[i], 0.0f);
    const unsigned long long k = (static_cast<unsigned long long>(__float_as_uint(d2)) << 32) |
                                 static_cast<unsigned long long>(0xFFFFFFFFu - static_cast<uint32_t>(i + row_offset));
    best = k > best ? k : best;
  }
  best = shfl_max_u64(best);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0ull;
    best = shfl_max_u64(best);
    if (threadIdx.x == 0) atomicMax(key, best);
  }
}

cudaError_t launch_rowmax_key(const float* rowmin, int64_t n, int64_t row_offset, unsigned long long* key,
                              cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(key, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 4) blocks = 148 * 4;
  if (blocks < 1) blocks = 1;
  count_launch();
  rowmax_key_kernel<<<static_cast<int>(blocks), 256, 0, st>>>(rowmin, n, row_offset, key);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- K7b fp64 NN of one point
struct DJ {
  double d;
  long long j;
};
__device__ __forceinline__ DJ dj_min(DJ a, DJ b) {
  if (b.d < a.d || (b.d == a.d && b.j < a.j)) return b;
  return a;
}
__device__ __forceinline__ DJ shfl_dj_min(DJ v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    DJ w;
    w.d = __shfl_xor_sync(0xffffffffu, v.d, o);
    w.j = __shfl_xor_sync(0xffffffffu, v.j, o);
    v = dj_min(v, w);
  }
  return v;
}

// One warp per candidate row j: lanes stride the coordinates, fixed-order tree
// reduction (deterministic). `a_ptr` may be decoded from a row-max key.
__global__ void __launch_bounds__(256) nn64_kernel(const float* __restrict__ X, int64_t x_offset, int64_t nX,
                                                   const unsigned long long* key, const float* __restrict__ a_direct,
                                                   const float* __restrict__ B, int64_t nB, int D,
                                                   double* blk_d, long long* blk_j) {
  __shared__ DJ sm[8];
  const float* a = a_direct;
  if (key != nullptr) {
    const long long row = static_cast<long long>(0xFFFFFFFFu - static_cast<uint32_t>(*key & 0xFFFFFFFFull)) - x_offset;
    const long long r = row < 0 ? 0 : (row >= nX ? nX - 1 : row);
    a = X + r * static_cast<int64_t>(D);
  }
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  DJ best{__longlong_as_double(0x7ff0000000000000ll), 0x7fffffffffffffffll};
  for (int64_t j = warp; j < nB; j += nwarps) {
    const float* b = B + j * static_cast<int64_t>(D);
    double s = 0.0;
    for (int c = lane; c < D; c += 32) {
      const double t = static_cast<double>(__ldg(a + c)) - static_cast<double>(__ldg(b + c));
      s = fma(t, t, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    best = dj_min(best, DJ{s, static_cast<long long>(j)});
  }
  if (lane == 0) sm[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    DJ v = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x]
                                           : DJ{__longlong_as_double(0x7ff0000000000000ll), 0x7fffffffffffffffll};
    v = shfl_dj_min(v);
    if (threadIdx.x == 0) {
      blk_d[blockIdx.x] = v.d;
      blk_j[blockIdx.x] = v.j;
    }
  }
}

__global__ void __launch_bounds__(256) nn64_final_kernel(const double* blk_d, const long long* blk_j, int nblocks,
                                                         double* out_d, long long* out_j) {
  __shared__ DJ sm[8];
  DJ best{__longlong_as_double(0x7ff0000000000000ll), 0x7fffffffffffffffll};
  for (int i = threadIdx.x; i < nblocks; i += blockDim.x) best = dj_min(best, DJ{blk_d[i], blk_j[i]});
  best = shfl_dj_min(best);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    DJ v = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x]
                                           : DJ{__longlong_as_double(0x7ff0000000000000ll), 0x7fffffffffffffffll};
    v = shfl_dj_min(v);
    if (threadIdx.x == 0) {
      *out_d = v.d;
      *out_j = v.j;
    }
  }
}

cudaError_t launch_nn64(const float* a, const float* B, int64_t nB, int D, double* blk_d, long long* blk_j,
                        int nblocks, double* out_d, long long* out_j, cudaStream_t st) {
  count_launch();
  nn64_kernel<<<nblocks, 256, 0, st>>>(nullptr, 0, 0, nullptr, a, B, nB, D, blk_d, blk_j);
  count_launch();
  nn64_final_kernel<<<1, 256, 0, st>>>(blk_d, blk_j, nblocks, out_d, out_j);
  return cudaGetLastError();
}

cudaError_t launch_nn64_from_key(const float* X, int64_t x_offset, int64_t nX, const unsigned long long* key,
                                 const float* B, int64_t nB, int D, double* blk_d, long long* blk_j, int nblocks,
                                 double* out_d, long long* out_j, cudaStream_t st) {
  count_launch();
  nn64_kernel<<<nblocks, 256, 0, st>>>(X, x_offset, nX, key, nullptr, B, nB, D, blk_d, blk_j);
  count_launch();
  nn64_final_kernel<<<1, 256, 0, st>>>(blk_d, blk_j, nblocks, out_d, out_j);
  return cudaGetLastError();
}

}  // namespace prohd
