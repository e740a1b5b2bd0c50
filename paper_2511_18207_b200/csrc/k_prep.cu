// k_prep.cu — K0 operand preparation, K7 row-max key and fp64 witness search.
//
// K0 (SURVEY.md §2f, §8(a) "Centering"): the distance kernel K6 forms
// a.b with the three-term split a.b ~= hi_a.hi_b + hi_a.lo_b + lo_a.hi_b (lo.lo dropped) on
// two operand arrays per set, H (hi) and L (lo). Per point y = x - c (fp64, c the pair's
// common centre; y = x without one). Two formats:
//   F16 (default): y is scaled by a power of two s (exact), hi = fp16_rn(s y), lo =
//        fp16_rn(s y - hi); 11 + 11 significant bits like 3xTF32, at the fp16 tensor rate and
//        half the operand bytes. s keeps |s y| <= 2^14 (no overflow): one scale per SET (the
//        set's max |y| -> (2^13, 2^14]) when the pair's dynamic range allows it, else one per
//        ROW (prep_mode below). scale[i] = s of row i.
//   TF32 (option k6_split3, the literal north-star form): hi = rn_tf32(fp32(y)) (low 13
//        mantissa bits zero, read exactly by the tensor core), lo = fp32(y - hi), s = 1.
// ||y||^2 is accumulated in fp64 and stored in fp32 (padded rows: +inf, so K6 needs no column
// masks). Rows are zero-padded to the array stride. A stats pass (warp per row) records each
// set's max |y| and min ||y||^2 (PrepStats) before the write pass, whose scale depends on both
// sets of the pair. One warp per row; HBM-bound.
//
// K7: the directed maximum over row minima packed as
//   key = (float_bits(d2) << 32) | (0xFFFFFFFF - row)
// (d2 >= 0, so the float's bit pattern orders like its value; the complement
// makes the LOWEST row win ties), then the witness column is recomputed in fp64
// direct form sum_k (a_k - b_k)^2 over all of B (lowest index on exact ties),
// matching the oracle's definition (Eq. (1)).
#include "internal.cuh"

#include <cuda_fp16.h>

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

template <bool kGather, bool kCentre>
__device__ __forceinline__ double coord(const float* __restrict__ x, const double* __restrict__ centre, int c, int D) {
  if (c >= D) return 0.0;
  const double v = static_cast<double>(__ldg(x + c));
  return kCentre ? v - __ldg(centre + c) : v;
}

// stats pass: norms (fp32, +inf padding), the set's max |y| and min ||y||^2 (float bits, atomics)
template <bool kGather, bool kCentre>
__global__ void __launch_bounds__(256) prep_stats_kernel(const float* __restrict__ X, const long long* __restrict__ idx,
                                                         int64_t n, int D, int64_t n_pad,
                                                         const double* __restrict__ centre, float* __restrict__ norms,
                                                         PrepStats* st, int* bad) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  __shared__ unsigned smax[8], smin[8];
  unsigned wmax = 0u, wmin = 0x7F800000u;
  for (int64_t r = warp; r < n_pad; r += nwarps) {
    if (r >= n) {
      if (lane == 0) norms[r] = __int_as_float(0x7f800000);
      continue;
    }
    const int64_t src = kGather ? idx[r] : r;
    const float* x = X + src * static_cast<int64_t>(D);
    double s = 0.0, mx = 0.0;
    for (int c = lane; c < D; c += 32) {
      const double y = coord<kGather, kCentre>(x, centre, c, D);
      s = fma(y, y, s);
      mx = fmax(mx, fabs(y));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const float f = static_cast<float>(s);
    const float fm = static_cast<float>(mx);
    if (lane == 0) norms[r] = f;
    if (!isfinite(s) || !isfinite(f) || !isfinite(fm)) {
      if (lane == 0) atomicExch(bad, 1);
    } else {
      wmax = max(wmax, __float_as_uint(fm));
      wmin = min(wmin, __float_as_uint(f));
    }
  }
  if (lane == 0) {
    smax[threadIdx.x >> 5] = wmax;
    smin[threadIdx.x >> 5] = wmin;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned bm = 0u, bn = 0x7F800000u;
    for (int i = 0; i < 8; ++i) {
      bm = max(bm, smax[i]);
      bn = min(bn, smin[i]);
    }
    if (bm != 0u) atomicMax(&st->maxabs, bm);
    if (bn != 0x7F800000u) atomicMin(&st->minnorm2, bn);
  }
}

// write pass: H, L and the per-row scale (F16) or fp32 hi / lo (TF32)
template <bool kGather, bool kCentre, bool kF16>
__global__ void __launch_bounds__(256) prep_write_kernel(const float* __restrict__ X,
                                                         const long long* __restrict__ idx, int64_t n, int D,
                                                         int Dh, int64_t n_pad, const double* __restrict__ centre,
                                                         const PrepStats* self, const PrepStats* other,
                                                         void* __restrict__ Hv, void* __restrict__ Lv,
                                                         float* __restrict__ scale) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const bool perrow = kF16 && prep_mode_perrow(self, other, D);
  const float sset = kF16 ? prep_scale_for(__uint_as_float(self->maxabs)) : 1.0f;
  for (int64_t r = warp; r < n_pad; r += nwarps) {
    if (r >= n) {
      if (lane == 0) scale[r] = sset;
      continue;
    }
    const int64_t src = kGather ? idx[r] : r;
    const float* x = X + src * static_cast<int64_t>(D);
    float sc = sset;
    if (perrow) {
      double mx = 0.0;
      for (int c = lane; c < D; c += 32) mx = fmax(mx, fabs(coord<kGather, kCentre>(x, centre, c, D)));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      sc = prep_scale_for(static_cast<float>(mx));
    }
    if (lane == 0) scale[r] = sc;
    if constexpr (kF16) {
      __half* h = reinterpret_cast<__half*>(Hv) + r * static_cast<int64_t>(Dh);
      __half* l = reinterpret_cast<__half*>(Lv) + r * static_cast<int64_t>(Dh);
      const double s64 = static_cast<double>(sc);
      for (int c = lane; c < Dh; c += 32) {
        const double y = coord<kGather, kCentre>(x, centre, c, D) * s64;  // exact: power-of-two scale
        const __half vh = __double2half(y);
        h[c] = vh;
        l[c] = __double2half(y - static_cast<double>(__half2float(vh)));
      }
    } else {
      float* h = reinterpret_cast<float*>(Hv) + r * static_cast<int64_t>(Dh);
      float* l = reinterpret_cast<float*>(Lv) + r * static_cast<int64_t>(Dh);
      for (int c = lane; c < Dh; c += 32) {
        const double y = coord<kGather, kCentre>(x, centre, c, D);
        const float vh = tf32_rn(static_cast<float>(y));
        h[c] = vh;
        l[c] = static_cast<float>(y - static_cast<double>(vh));
      }
    }
  }
}

static int grid_for_rows(int64_t rows) {
  int64_t blocks = (rows + 7) / 8;  // 8 warps per block, one row per warp
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  return static_cast<int>(blocks);
}

cudaError_t launch_prep_stats(const float* X, const long long* idx, int64_t n, int D, int64_t n_pad,
                              const double* centre, float* norms, PrepStats* st, int* bad, cudaStream_t st_) {
  count_launch();
  const int g = grid_for_rows(n_pad);
#define PS(G, C) prep_stats_kernel<G, C><<<g, 256, 0, st_>>>(X, idx, n, D, n_pad, centre, norms, st, bad)
  if (idx && centre) PS(true, true);
  else if (idx) PS(true, false);
  else if (centre) PS(false, true);
  else PS(false, false);
#undef PS
  return cudaGetLastError();
}

cudaError_t launch_prep_write(const float* X, const long long* idx, int64_t n, int D, int64_t n_pad,
                              const double* centre, const PrepStats* self, const PrepStats* other, bool f16, void* H,
                              void* L, float* scale, cudaStream_t st) {
  count_launch();
  const int g = grid_for_rows(n_pad);
  const int Dh = f16 ? k6_stride_f16(D) : k6_stride_f32(D);
#define PW(G, C, F) \
  prep_write_kernel<G, C, F><<<g, 256, 0, st>>>(X, idx, n, D, Dh, n_pad, centre, self, other, H, L, scale)
  if (f16) {
    if (idx && centre) PW(true, true, true);
    else if (idx) PW(true, false, true);
    else if (centre) PW(false, true, true);
    else PW(false, false, true);
  } else {
    if (idx && centre) PW(true, true, false);
    else if (idx) PW(true, false, false);
    else if (centre) PW(false, true, false);
    else PW(false, false, false);
  }
#undef PW
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
