// k_select.cu — K3 projection, K4 top/bottom-m selection, K5 union + gather.
//
// PAPER.md Alg. 1 lines 3-9 and Alg. 2 lines 4-11: for
// each set X and direction u_l, project every point (pi = x^T u), keep
// the m smallest and m largest projections, and take the union of all kept
// indices ("keep the unique indices").
//
// Selection semantics are the oracle's: the order is
// that of the fp64 projections of the fp32 points onto the fp64 directions, with
// ties broken by lower index: bottom = (pi asc, idx asc), top = (pi desc, idx asc).
//
// GPU scheme:
//   K3  pi32 = x . u32 in fp32 (one warp per point; HBM-bound) and max ||x||^2.
//   K4  radix select (11/11/10-bit digits, 3 histogram rounds over
//       order-preserving uint32 keys; the bottom tail uses the complemented key)
//       gives T, the m-th best fp32 projection per (direction, tail).
//       Every point with pi32 within the guard band 2*eps of T (or better) is a
//       candidate, eps = (D + 8) 2^-24 max||x|| bounding |pi32 - pi64|, so the
//       true fp64 top-m is always inside the band. Candidates are re-ranked by
//       their fp64 projection (fp64 dot with the fp64 direction) and the total
//       order above; rank < m is kept, at position `rank` of the list.
//   K5  kept indices are OR-ed into an n-bit bitmap; one CTA compacts it into
//       the sorted unique union; the rows are gathered for the subset HD.
#include "internal.cuh"
#include "prohd_kernels.cuh"

#include <cfloat>
#include <cmath>
#include <cstdlib>

namespace prohd {
namespace {

__device__ __forceinline__ unsigned order_key(float f) {
  unsigned u = __float_as_uint(f == 0.0f ? 0.0f : f);  // canonicalise -0 -> +0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_to_float(unsigned k) {
  const unsigned u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(u);
}

// ------------------------------------------------------------------ K3
constexpr int kProjGroup = 8;

__global__ void __launch_bounds__(256) project_kernel(const float* __restrict__ X, int64_t n, int D,
                                                      const float* __restrict__ U32, int L,
                                                      float* __restrict__ P32, unsigned* maxnorm2) {
  extern __shared__ float su[];  // [L][D]
  for (int i = threadIdx.x; i < L * D; i += blockDim.x) su[i] = U32[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  float wmax = 0.0f;
  for (int64_t r = warp; r < n; r += nwarps) {
    const float* x = X + r * D;
    float nrm = 0.0f;
    for (int g0 = 0; g0 < L; g0 += kProjGroup) {
      float acc[kProjGroup];
#pragma unroll
      for (int j = 0; j < kProjGroup; ++j) acc[j] = 0.0f;
      for (int c = lane; c < D; c += 32) {
        const float v = __ldg(x + c);
        if (g0 == 0) nrm = fmaf(v, v, nrm);
#pragma unroll
        for (int j = 0; j < kProjGroup; ++j)
          if (g0 + j < L) acc[j] = fmaf(v, su[(g0 + j) * D + c], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < kProjGroup; ++j) {
        float s = acc[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == j && g0 + j < L) P32[static_cast<int64_t>(g0 + j) * n + r] = s;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    // non-finite input must poison the max (fmaxf would drop a NaN)
    wmax = (isfinite(nrm) && isfinite(wmax)) ? fmaxf(wmax, nrm) : __int_as_float(0x7fffffff);
  }
  if (lane == 0) atomicMax(maxnorm2, __float_as_uint(wmax));  // non-negative floats order as uints
}

// K3 fast path (D % 4 == 0, L <= 32): one thread per point, the CTA's 256 points
// staged through shared memory in 64-feature chunks with cp.async double
// buffering; the direction rows are read as 16-byte broadcasts. FFMA-bound at
// ~17 x D FMAs per point, close to the HBM time of reading the points once.
constexpr int kPP = 256;  // points per CTA tile (= threads)
constexpr int kFC = 32;   // features per chunk
constexpr int kXS = 36;   // smem row stride (floats): 16-B aligned, 8 rows cover all banks

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int n = valid ? 16 : 0;  // src-size 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int LMAX, bool kExact>
__global__ void __launch_bounds__(kPP, 2) project_tile_kernel(const float* __restrict__ X, int64_t n, int D,
                                                              const float* __restrict__ U32, int L,
                                                              float* __restrict__ P32, unsigned* maxnorm2) {
  extern __shared__ float smp[];
  float* su = smp;                      // [L][D]
  float* xs = smp + ((L * D + 3) & ~3);  // [2][kPP][kXS]
  for (int i = threadIdx.x; i < L * D; i += blockDim.x) su[i] = U32[i];
  const int tid = threadIdx.x;
  const int nch = (D + kFC - 1) / kFC;
  float wmax = 0.0f;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * kPP; base < n;
       base += static_cast<int64_t>(gridDim.x) * kPP) {
    // issue chunk 0
    auto issue = [&](int c, int buf) {
      float* dst = xs + buf * kPP * kXS;
      const int f0 = c * kFC;
      // kPP rows x (kFC/4) 16-byte pieces, coalesced along the row
      for (int q = tid; q < kPP * (kFC / 4); q += kPP) {
        const int r = q / (kFC / 4), v = q % (kFC / 4);
        const int64_t p = base + r;
        const int f = f0 + 4 * v;
        const bool ok = p < n && f < D;
        cp_async16(dst + r * kXS + 4 * v, ok ? X + p * D + f : X, ok);
      }
      cp_async_commit();
    };
    float acc[LMAX];
#pragma unroll
    for (int l = 0; l < LMAX; ++l) acc[l] = 0.0f;
    float nrm = 0.0f;
    __syncthreads();  // previous tile's readers are done with both buffers
    issue(0, 0);
    for (int c = 0; c < nch; ++c) {
      if (c + 1 < nch) {
        issue(c + 1, (c + 1) & 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const float* xr = xs + (c & 1) * kPP * kXS + tid * kXS;
      const int f0 = c * kFC;
      const int fe = min(kFC, D - f0);
      for (int f = 0; f < fe; f += 4) {
        const float4 x4 = *reinterpret_cast<const float4*>(xr + f);
        nrm = fmaf(x4.x, x4.x, nrm);
        nrm = fmaf(x4.y, x4.y, nrm);
        nrm = fmaf(x4.z, x4.z, nrm);
        nrm = fmaf(x4.w, x4.w, nrm);
#pragma unroll
        for (int l = 0; l < LMAX; ++l) {
          if (kExact || l < L) {
            const float4 u4 = *reinterpret_cast<const float4*>(su + l * D + f0 + f);
            float a = acc[l];
            a = fmaf(x4.x, u4.x, a);
            a = fmaf(x4.y, u4.y, a);
            a = fmaf(x4.z, u4.z, a);
            a = fmaf(x4.w, u4.w, a);
            acc[l] = a;
          }
        }
      }
      __syncthreads();  // buffer (c & 1) may be refilled by the next issue
    }
    const int64_t p = base + tid;
    if (p < n) {
#pragma unroll
      for (int l = 0; l < LMAX; ++l)
        if (kExact || l < L) P32[static_cast<int64_t>(l) * n + p] = acc[l];
      wmax = (isfinite(nrm) && isfinite(wmax)) ? fmaxf(wmax, nrm) : __int_as_float(0x7fffffff);
    }
  }
  // block max of wmax -> one atomic
  __shared__ unsigned bm;
  if (tid == 0) bm = 0u;
  __syncthreads();
  atomicMax(&bm, __float_as_uint(wmax));
  __syncthreads();
  if (tid == 0) atomicMax(maxnorm2, bm);
}

// ------------------------------------------------------------------ K4 radix select
__device__ __forceinline__ void round_params(int round, int& shift, unsigned& binmask) {
  if (round == 0) {
    shift = 21;
    binmask = 0x7FFu;
  } else if (round == 1) {
    shift = 10;
    binmask = 0x7FFu;
  } else {
    shift = 0;
    binmask = 0x3FFu;
  }
}

__global__ void __launch_bounds__(256) radix_hist_kernel(const float* __restrict__ P32, int64_t n, int L,
                                                         const int* n_dirs, int round,
                                                         const unsigned* __restrict__ state, unsigned* hist) {
  __shared__ unsigned sh[2][kRadixBins];
  const int l = blockIdx.y;
  if (l >= *n_dirs) return;
  for (int i = threadIdx.x; i < 2 * kRadixBins; i += blockDim.x) (&sh[0][0])[i] = 0u;
  __syncthreads();
  int shift;
  unsigned binmask;
  round_params(round, shift, binmask);
  const unsigned pre0 = state[(l * 2 + 0) * 4 + 0], msk0 = state[(l * 2 + 0) * 4 + 1];
  const unsigned pre1 = state[(l * 2 + 1) * 4 + 0], msk1 = state[(l * 2 + 1) * 4 + 1];
  const float* p = P32 + static_cast<int64_t>(l) * n;
  auto add = [&](float x) {
    const unsigned kt = order_key(x);
    const unsigned kb = ~kt;
    if ((kt & msk0) == pre0) atomicAdd(&sh[0][(kt >> shift) & binmask], 1u);
    if ((kb & msk1) == pre1) atomicAdd(&sh[1][(kb >> shift) & binmask], 1u);
  };
  // 16-B loads over the aligned middle of the row, scalar head and tail
  const int64_t head = min(n, static_cast<int64_t>(((16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15) / 4));
  const int64_t nv = (n - head) / 4;
  const float4* p4 = reinterpret_cast<const float4*>(p + head);
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  if (tid < head) add(__ldg(p + tid));
  for (int64_t q = tid; q < nv; q += stride) {
    const float4 v = __ldg(p4 + q);
    add(v.x);
    add(v.y);
    add(v.z);
    add(v.w);
  }
  for (int64_t i = head + 4 * nv + tid; i < n; i += stride) add(__ldg(p + i));
  __syncthreads();
  unsigned* g = hist + (static_cast<int64_t>(round) * L + l) * 2 * kRadixBins;
  for (int i = threadIdx.x; i < 2 * kRadixBins; i += blockDim.x) {
    const unsigned v = (&sh[0][0])[i];
    if (v) atomicAdd(g + i, v);
  }
}

// One CTA per (direction, tail): find the bin b (scanning from the top) where the
// running count reaches the remaining rank `rem`, i.e. the first b >= 1 in descending
// order with cum(> b) + h[b] >= rem (else b = 0), as a block-wide suffix scan: thread i
// owns descending positions [i * per, (i + 1) * per), bin = binmask - position.
constexpr int kScanT = 256;
__global__ void __launch_bounds__(kScanT) radix_scan_kernel(const unsigned* __restrict__ hist, int L,
                                                           const int* n_dirs, int round, unsigned* state) {
  const int id = blockIdx.x;
  const int l = id >> 1, t = id & 1;
  if (l >= *n_dirs) return;
  int shift;
  unsigned binmask;
  round_params(round, shift, binmask);
  const int nbins = static_cast<int>(binmask) + 1;
  const int per = nbins / kScanT;  // 8 or 4
  const unsigned* h = hist + ((static_cast<int64_t>(round) * L + l) * 2 + t) * kRadixBins;
  unsigned* s = state + (l * 2 + t) * 4;
  const unsigned rem = s[2];
  __shared__ unsigned wsum[kScanT / 32];
  __shared__ int first;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  unsigned v[8];
  unsigned tot = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    v[j] = j < per ? h[binmask - (tid * per + j)] : 0u;
    tot += v[j];
  }
  // exclusive scan of the thread totals in descending-bin order
  unsigned inc = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (tid == 0) first = 0x7FFFFFFF;
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  unsigned excl = inc - tot;
  for (int i = 0; i < w; ++i) excl += wsum[i];
  unsigned cum = excl;
  int hit = 0x7FFFFFFF;
  unsigned cum_hit = 0, cum_ge1 = 0;
  for (int j = 0; j < per; ++j) {
    const int d = tid * per + j;
    const int bin = static_cast<int>(binmask) - d;
    if (bin >= 1 && hit == 0x7FFFFFFF && cum + v[j] >= rem) {
      hit = d;
      cum_hit = cum;
    }
    cum += v[j];
    if (bin == 1) cum_ge1 = cum;  // sum of all bins >= 1
  }
  if (hit != 0x7FFFFFFF) atomicMin(&first, hit);
  __syncthreads();
  const int f = first;
  if (f != 0x7FFFFFFF) {
    if (hit == f) {
      s[0] |= static_cast<unsigned>(static_cast<int>(binmask) - f) << shift;
      s[1] |= binmask << shift;
      s[2] = rem - cum_hit;
    }
  } else if (tid == (nbins - 2) / per) {  // owner of bin 1: fall back to bin 0
    s[1] |= binmask << shift;
    s[2] = rem - cum_ge1;
  }
}

__global__ void __launch_bounds__(256) collect_kernel(const float* __restrict__ P32, int64_t n, int D, int L,
                                                      const int* n_dirs, const unsigned* __restrict__ state,
                                                      const unsigned* maxnorm2, int* cand, unsigned* ccount,
                                                      int64_t cap, int* overflow, int all, double eps_coef) {
  const int l = blockIdx.y;
  if (l >= *n_dirs) return;
  // eps_coef * max||x|| bounds |pi32 - pi64| for the K3 variant that ran (1.0625: margin for
  // the fp32 norm and sqrt)
  const double eps = eps_coef * sqrt(static_cast<double>(__uint_as_float(*maxnorm2))) * 1.0625;
  const double Ttop = static_cast<double>(key_to_float(state[(l * 2 + 0) * 4 + 0]));
  const double Tbot = static_cast<double>(key_to_float(~state[(l * 2 + 1) * 4 + 0]));
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const double lo_top = all ? -inf : Ttop - 2.0 * eps;  // top candidates: pi >= lo_top
  const double hi_bot = all ? inf : Tbot + 2.0 * eps;   // bottom candidates: pi <= hi_bot
  const float* p = P32 + static_cast<int64_t>(l) * n;
  const int lane = threadIdx.x & 31;
  // every lane takes 4 consecutive points per step (16-B loads where the row is aligned); the
  // warp reserves its candidates of each tail with one atomicAdd and an exclusive lane scan
  const int64_t head = min(n, static_cast<int64_t>(((16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15) / 4));
  const int64_t nq = head + (n - head + 3) / 4;  // head singletons, then groups of 4
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < nq;
       base += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t q = base + threadIdx.x;
    float v[4];
    int64_t i0 = 0;
    int nvalid = 0;
    if (q < head) {
      i0 = q;
      nvalid = 1;
      v[0] = __ldg(p + q);
    } else if (q < nq) {
      i0 = head + 4 * (q - head);
      nvalid = n - i0 < 4 ? static_cast<int>(n - i0) : 4;
      if (nvalid == 4) {
        const float4 w = __ldg(reinterpret_cast<const float4*>(p + i0));
        v[0] = w.x;
        v[1] = w.y;
        v[2] = w.z;
        v[3] = w.w;
      } else {
        for (int j = 0; j < nvalid; ++j) v[j] = __ldg(p + i0 + j);
      }
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      unsigned mask = 0u;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double x = static_cast<double>(v[j]);
        const bool c = j < nvalid && (t == 0 ? x >= lo_top : x <= hi_bot);
        mask |= c ? 1u << j : 0u;
      }
      const unsigned cnt = __popc(mask);
      unsigned incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
      if (total == 0u) continue;
      unsigned pos0 = 0;
      if (lane == 31) pos0 = atomicAdd(&ccount[l * 2 + t], total);
      pos0 = __shfl_sync(0xffffffffu, pos0, 31);
      unsigned pos = pos0 + incl - cnt;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (mask & (1u << j)) {
          if (pos < cap)
            cand[(static_cast<int64_t>(l) * 2 + t) * cap + pos] = static_cast<int>(i0 + j);
          else
            *overflow = 1;
          ++pos;
        }
      }
    }
  }
}

// ------------------------------------------------------------------ K4, sampled-threshold variant
// (launch_select_sampled). The radix select above reads all L n projections four times (three
// histogram rounds and the collection). Here a sample of s rows fixes, per (direction, tail), a
// threshold thr that about 5 m of the n points pass; K3's epilogue then appends (index, pi32) of
// exactly those points (P32 is not written), and one CTA per list finds the m-th best value T
// among them, CHECKS that the guard band [T - 2 eps, inf) lies inside [thr, inf) (then every
// point of the band was appended, so T and the band are exactly those of the radix path) and
// writes the band as the candidate list. A list that cannot be certified (fewer than m appended,
// band not inside, raw buffer full) sets sfail and the caller reruns the radix path.

// the rank-th largest key (1-based) among cnt keys key(v[i], tail) (top: order_key, bottom: its
// complement), one block of kSelThreads threads, 1 <= rank <= cnt. Radix digits of
// (key - min key) from the top bit of (max - min) down, 8 bits per round (adaptive: the values'
// own key range, not the full float range, so the first round already spreads them); warp-private
// histograms (shared atomics without return: a warp's clustered values serialise only within
// the warp); warp 0 scans the 256 bins. v: shared memory or global (L2-resident) values; hbuf:
// kSelHistWords words of (dynamic) shared memory.
constexpr int kSelThreads = 1024;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSelBins = 256;
constexpr int kSelHistWords = kSelWarps * kSelBins;
__device__ unsigned block_select_key(const float* v, int64_t cnt, unsigned rank, int t, unsigned* hbuf) {
  __shared__ unsigned tot[kSelBins];
  __shared__ unsigned wmin[kSelWarps], wmax[kSelWarps];
  __shared__ unsigned s_prefix, s_mask, s_rem;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  unsigned* hw = hbuf + w * kSelBins;
  auto key = [&](int64_t i) {
    const unsigned k0 = order_key(v[i]);
    return t == 0 ? k0 : ~k0;
  };
  unsigned kmin = 0xFFFFFFFFu, kmax = 0u;
  for (int64_t i = tid; i < cnt; i += kSelThreads) {
    const unsigned k = key(i);
    kmin = min(kmin, k);
    kmax = max(kmax, k);
  }
  kmin = __reduce_min_sync(0xffffffffu, kmin);
  kmax = __reduce_max_sync(0xffffffffu, kmax);
  if (lane == 0) {
    wmin[w] = kmin;
    wmax[w] = kmax;
  }
  if (tid == 0) {
    s_prefix = 0u;
    s_mask = 0u;
    s_rem = rank;
  }
  __syncthreads();
  kmin = wmin[0];
  kmax = wmax[0];
  for (int i = 1; i < kSelWarps; ++i) {
    kmin = min(kmin, wmin[i]);
    kmax = max(kmax, wmax[i]);
  }
  int rb = 32 - __clz(kmax - kmin);  // bits left to resolve
  while (rb > 0) {
    const int shift = rb > 8 ? rb - 8 : 0;
    const unsigned binmask = (1u << (rb - shift)) - 1u;
    for (int b = lane; b < kSelBins; b += 32) hw[b] = 0u;
    __syncwarp();
    const unsigned prefix = s_prefix, mask = s_mask;
    for (int64_t i = tid; i < cnt; i += kSelThreads) {
      const unsigned d = key(i) - kmin;
      if ((d & mask) == prefix) atomicAdd(&hw[(d >> shift) & binmask], 1u);
    }
    __syncthreads();
    if (tid < kSelBins) {
      unsigned c = 0;
      for (int j = 0; j < kSelWarps; ++j) c += hbuf[j * kSelBins + tid];
      tot[tid] = c;
    }
    __syncthreads();
    if (w == 0) {  // descending: lane owns bins 255 - 8 lane .. 248 - 8 lane
      unsigned hv[8], sum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        hv[j] = tot[kSelBins - 1 - (8 * lane + j)];
        sum += hv[j];
      }
      unsigned inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const unsigned rem = s_rem;
      unsigned cum = inc - sum;
      int hit = -1;
      unsigned cum_hit = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int pos = 8 * lane + j;  // descending position; bin = 255 - pos
        if (hit < 0 && cum + hv[j] >= rem && kSelBins - 1 - pos <= static_cast<int>(binmask)) {
          hit = pos;
          cum_hit = cum;
        }
        cum += hv[j];
      }
      const unsigned hm = __ballot_sync(0xffffffffu, hit >= 0);
      // rem <= the count of this round's candidates: some lane hits (bins above binmask are empty)
      if (hm != 0u && lane == __ffs(hm) - 1) {
        s_prefix = prefix | (static_cast<unsigned>(kSelBins - 1 - hit) << shift);
        s_mask = mask | (binmask << shift);
        s_rem = rem - cum_hit;
      }
    }
    __syncthreads();
    rb = shift;
  }
  return kmin + s_prefix;
}

constexpr int kSampleMax = 32768;  // sample rows (their projections staged in shared memory)
constexpr int kFilterStage = 16384;  // appended entries per list (shared memory, values + indices)
constexpr int kSlabCap = 64;         // entries per (epilogue warp, list) slab

// stage cnt floats into shared memory: 8 independent loads in flight per thread (one block
// streams from L2; a load-store loop would be one L2 latency per element)
__device__ __forceinline__ void stage_floats(float* dst, const float* __restrict__ src, int64_t cnt) {
  const int64_t nb = blockDim.x;
  for (int64_t base = threadIdx.x; base < cnt; base += 8 * nb) {
    float r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = base + k * nb < cnt ? __ldg(src + base + k * nb) : 0.0f;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (base + k * nb < cnt) dst[base + k * nb] = r[k];
  }
  __syncthreads();
}

// per list lt = 2 l + tail: the threshold = the r-th best sample projection -> state[lt * 4 + 0]
// (float bits), raw count state[lt * 4 + 1] = 0
__global__ void __launch_bounds__(kSelThreads) sample_thresh_kernel(const float* __restrict__ S, int s, const int* n_dirs,
                                                            unsigned r, unsigned* state) {
  extern __shared__ float sv[];  // [s] values, then the selection histograms
  const int lt = blockIdx.x, l = lt >> 1, t = lt & 1;
  if (l >= *n_dirs) {  // a dropped direction: nothing passes (K3 appends nothing)
    if (threadIdx.x == 0) {
      state[lt * 4 + 0] = __float_as_uint(t == 0 ? __int_as_float(0x7f800000) : __int_as_float(0xff800000));
      state[lt * 4 + 1] = 0u;
    }
    return;
  }
  stage_floats(sv, S + static_cast<int64_t>(l) * s, s);
  const unsigned k = block_select_key(sv, s, r, t, reinterpret_cast<unsigned*>(sv + s));
  if (threadIdx.x == 0) {
    state[lt * 4 + 0] = __float_as_uint(key_to_float(t == 0 ? k : ~k));
    state[lt * 4 + 1] = 0u;
  }
}

// per list: the slabs' entries gathered into shared memory, T = the m-th best of them,
// certification, the guard band as candidates (the same band as collect_kernel)
__global__ void __launch_bounds__(kSelThreads) cand_filter_kernel(const int* n_dirs, const unsigned* __restrict__ state,
                                                          const int* __restrict__ sidx, const float* __restrict__ sval,
                                                          const unsigned* __restrict__ wcount, int nslabs, int L,
                                                          int capw, int64_t m, const unsigned* maxnorm2,
                                                          double eps_coef, int* cand, unsigned* ccount, int64_t cap,
                                                          int* overflow, int* sfail) {
  extern __shared__ float sv[];
  int* si = reinterpret_cast<int*>(sv + kFilterStage);
  __shared__ unsigned wsum[kSelWarps];
  const int lt = blockIdx.x, l = lt >> 1, t = lt & 1;
  if (l >= *n_dirs) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int mybad = 0;
  // slabs [tid * per, (tid + 1) * per) (per <= 4): counts, exclusive block scan of the totals
  const int per = (nslabs + kSelThreads - 1) / kSelThreads;
  unsigned cs[4];
  unsigned tot = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int sl = tid * per + j;
    cs[j] = (j < per && sl < nslabs) ? __ldg(wcount + static_cast<int64_t>(sl) * 2 * L + lt) : 0u;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (cs[j] > static_cast<unsigned>(capw)) mybad = 1;
    tot += cs[j];
  }
  unsigned inc = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[w] = inc;
  const int bad = __syncthreads_or(mybad);
  unsigned off = inc - tot;
  for (int i = 0; i < w; ++i) off += wsum[i];
  unsigned total = 0;
  for (int i = 0; i < kSelWarps; ++i) total += wsum[i];
  if (bad || total > static_cast<unsigned>(kFilterStage) || total < m) {
    if (tid == 0) atomicOr(sfail, 1);
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int sl = tid * per + j;
    const unsigned c = cs[j];
    const int64_t e0 = (static_cast<int64_t>(sl) * 2 * L + lt) * capw;
    for (unsigned k0 = 0; k0 < c; k0 += 8) {  // 16 independent loads in flight
      float rv[8];
      int ri[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        rv[k] = k0 + k < c ? __ldg(sval + e0 + k0 + k) : 0.0f;
        ri[k] = k0 + k < c ? __ldg(sidx + e0 + k0 + k) : 0;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k0 + k < c) {
          sv[off + k0 + k] = rv[k];
          si[off + k0 + k] = ri[k];
        }
    }
    off += c;
  }
  __syncthreads();
  const unsigned key = block_select_key(sv, total, static_cast<unsigned>(m), t,
                                        reinterpret_cast<unsigned*>(si + kFilterStage));
  const double T = static_cast<double>(key_to_float(t == 0 ? key : ~key));
  const double thr = static_cast<double>(__uint_as_float(state[lt * 4 + 0]));
  const double eps = eps_coef * sqrt(static_cast<double>(__uint_as_float(*maxnorm2))) * 1.0625;
  const double lo = T - 2.0 * eps, hi = T + 2.0 * eps;
  if (!(t == 0 ? lo >= thr : hi <= thr)) {  // the band reaches past the threshold (or NaN)
    if (tid == 0) atomicOr(sfail, 1);
    return;
  }
  for (unsigned base = 0; base < total; base += blockDim.x) {
    const unsigned i = base + tid;
    const double x = i < total ? static_cast<double>(sv[i]) : 0.0;
    const bool keep = i < total && (t == 0 ? x >= lo : x <= hi);
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (bal == 0u) continue;
    unsigned pos0 = 0;
    if (lane == 0) pos0 = atomicAdd(&ccount[lt], static_cast<unsigned>(__popc(bal)));
    pos0 = __shfl_sync(0xffffffffu, pos0, 0);
    const unsigned pos = pos0 + __popc(bal & ((1u << lane) - 1u));
    if (keep) {
      if (pos < cap)
        cand[static_cast<int64_t>(lt) * cap + pos] = si[i];
      else
        *overflow = 1;
    }
  }
}

// fp64 projection of every candidate: one warp per candidate
__global__ void __launch_bounds__(256) cand_p64_kernel(const float* __restrict__ X, int D,
                                                       const double* __restrict__ U64, int L, const int* n_dirs,
                                                       const int* __restrict__ cand, const unsigned* ccount,
                                                       int64_t cap, double* cval) {
  const int lt = blockIdx.y;  // l*2 + t
  const int l = lt >> 1;
  if (l >= *n_dirs) return;
  const unsigned cnt = min(static_cast<int64_t>(ccount[lt]), cap);
  const int lane = threadIdx.x & 31;
  const double* u = U64 + static_cast<int64_t>(l) * D;
  for (int64_t c = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c < cnt;
       c += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int i = cand[static_cast<int64_t>(lt) * cap + c];
    const float* x = X + static_cast<int64_t>(i) * D;
    double s = 0.0;
    for (int d = lane; d < D; d += 32) s = fma(static_cast<double>(__ldg(x + d)), u[d], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) cval[static_cast<int64_t>(lt) * cap + c] = s;
  }
}

// rank of each candidate in its (direction, tail) total order; keep rank < m
__global__ void __launch_bounds__(256) rank_kernel(int L, const int* n_dirs, const int* __restrict__ cand,
                                                   const double* __restrict__ cval, const unsigned* ccount,
                                                   int64_t cap, int64_t m, int* lists, unsigned* bitmap,
                                                   double* cv_out, long long* ci_out, int64_t row_offset,
                                                   const unsigned* only) {
  const int lt = blockIdx.y;
  const int l = lt >> 1, t = lt & 1;
  if (l >= *n_dirs) return;
  // a list whose guard band overflowed the candidate buffer is left to the band-select fallback
  // (launch_select_fallback); in the fallback pass `only` restricts the ranking to those lists
  if (only != nullptr ? only[lt] == 0u : static_cast<int64_t>(ccount[lt]) > cap) return;
  const int64_t cnt = min(static_cast<int64_t>(ccount[lt]), cap);
  const int* ci = cand + static_cast<int64_t>(lt) * cap;
  const double* cv = cval + static_cast<int64_t>(lt) * cap;
  constexpr int kStage = 3072;  // candidates staged in shared memory (the band is usually ~m + a few)
  __shared__ double sv[kStage];
  __shared__ int si[kStage];
  const bool staged = cnt <= kStage;
  if (staged) {
    for (int64_t o = threadIdx.x; o < cnt; o += blockDim.x) {
      sv[o] = cv[o];
      si[o] = ci[o];
    }
    __syncthreads();
  }
  // four lanes per candidate, each counting over a quarter of the list (warp-uniform trip
  // counts: the loop runs to the warp's largest candidate slot, extra slots count nothing)
  const int q = threadIdx.x & 3;
  const int64_t per_pass = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 2);
  for (int64_t c0 = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 2); c0 < cnt; c0 += per_pass) {
    const int64_t c = c0 + (threadIdx.x >> 2);
    const bool live = c < cnt;
    const double v = live ? (staged ? sv[c] : cv[c]) : 0.0;
    const int i = live ? (staged ? si[c] : ci[c]) : 0;
    int64_t rank = 0;
    if (staged) {
      for (int o = q; o < static_cast<int>(cnt); o += 4) {
        const double w = sv[o];
        const int j = si[o];
        rank += ((t == 0) ? (w > v || (w == v && j < i)) : (w < v || (w == v && j < i))) ? 1 : 0;
      }
    } else {
      for (int64_t o = q; o < cnt; o += 4) {
        const double w = cv[o];
        const int j = ci[o];
        rank += ((t == 0) ? (w > v || (w == v && j < i)) : (w < v || (w == v && j < i))) ? 1 : 0;
      }
    }
    rank += __shfl_xor_sync(0xffffffffu, rank, 1);
    rank += __shfl_xor_sync(0xffffffffu, rank, 2);
    if (live && q == 0 && rank < m) {
      if (lists != nullptr) lists[static_cast<int64_t>(lt) * m + rank] = i;
      if (bitmap != nullptr) atomicOr(&bitmap[i >> 5], 1u << (i & 31));
      if (cv_out != nullptr) {
        cv_out[static_cast<int64_t>(lt) * m + rank] = v;
        ci_out[static_cast<int64_t>(lt) * m + rank] = row_offset + i;
      }
    }
  }
}

// K5 compaction of the n-bit bitmap into the sorted unique union, two launches over kCB
// CTAs, each owning a contiguous word range: (a) per-CTA popcounts, (b) each CTA adds the
// counts of the CTAs before it, scans its threads' counts and writes its indices in order.
constexpr int kCB = kCompactBlocks;
__global__ void __launch_bounds__(256) compact_count_kernel(const unsigned* __restrict__ bitmap, int64_t nwords,
                                                            unsigned* __restrict__ bcount) {
  const int64_t per = (nwords + kCB - 1) / kCB;
  const int64_t w0 = blockIdx.x * per, w1 = min(nwords, w0 + per);
  unsigned c = 0;
  for (int64_t w = w0 + threadIdx.x; w < w1; w += blockDim.x) c += __popc(bitmap[w]);
  __shared__ unsigned red[256];
  red[threadIdx.x] = c;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (static_cast<int>(threadIdx.x) < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) bcount[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(256) compact_write_kernel(const unsigned* __restrict__ bitmap, int64_t nwords,
                                                            const unsigned* __restrict__ bcount, long long* uidx,
                                                            unsigned* ucount) {
  __shared__ unsigned part[256];
  __shared__ unsigned base;
  if (threadIdx.x == 0) {
    unsigned b = 0;
    for (int q = 0; q < static_cast<int>(blockIdx.x); ++q) b += bcount[q];
    base = b;
    if (blockIdx.x == kCB - 1) *ucount = b + bcount[kCB - 1];
  }
  const int64_t per = (nwords + kCB - 1) / kCB;
  const int64_t w0 = blockIdx.x * per, w1 = min(nwords, w0 + per);
  const int64_t tper = (w1 - w0 + 255) / 256;  // contiguous words per thread
  const int64_t t0 = min(w1, w0 + threadIdx.x * tper), t1 = min(w1, t0 + tper);
  unsigned c = 0;
  for (int64_t w = t0; w < t1; ++w) c += __popc(bitmap[w]);
  part[threadIdx.x] = c;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {  // inclusive scan (Hillis-Steele)
    const unsigned v = static_cast<int>(threadIdx.x) >= o ? part[threadIdx.x - o] : 0u;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  unsigned pos = base + part[threadIdx.x] - c;
  for (int64_t w = t0; w < t1; ++w) {
    unsigned bits = bitmap[w];
    while (bits) {
      const int b = __ffs(bits) - 1;
      uidx[pos++] = w * 32 + b;
      bits &= bits - 1;
    }
  }
}

__global__ void iota_kernel(long long* idx, unsigned* count, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    idx[i] = i;
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = static_cast<unsigned>(n);
}

__global__ void __launch_bounds__(256) gather_kernel(const float* __restrict__ X, int D,
                                                     const long long* __restrict__ idx, const unsigned* count,
                                                     float* __restrict__ Y) {
  const unsigned n = *count;
  const int lane = threadIdx.x & 31;
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < n;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const float* src = X + idx[r] * D;
    float* dst = Y + r * D;
    for (int c = lane; c < D; c += 32) dst[c] = __ldg(src + c);
  }
}

// merge: rank every entry of list (l, t) among the G*m entries of all ranks; keep rank < m
__global__ void __launch_bounds__(256) merge_rank_kernel(const double* __restrict__ cval,
                                                         const long long* __restrict__ cidx, int G, int L,
                                                         const int* n_dirs, int64_t m, unsigned* bitmap) {
  const int lt = blockIdx.y;
  const int l = lt >> 1, t = lt & 1;
  if (l >= *n_dirs) return;
  const int64_t tot = static_cast<int64_t>(G) * m;
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c < tot;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t gc = c / m, jc = c % m;
    const int64_t off = (gc * L * 2 + lt) * m;
    const long long i = cidx[off + jc];
    if (i < 0) continue;
    const double v = cval[off + jc];
    int64_t rank = 0;
    for (int64_t o = 0; o < tot && rank < m; ++o) {
      const int64_t go = o / m, jo = o % m;
      const int64_t oo = (go * L * 2 + lt) * m + jo;
      const long long j = cidx[oo];
      if (j < 0) continue;
      const double w = cval[oo];
      const bool better = (t == 0) ? (w > v || (w == v && j < i)) : (w < v || (w == v && j < i));
      rank += better ? 1 : 0;
    }
    if (rank < m) atomicOr(&bitmap[i >> 5], 1u << (i & 31));
  }
}

__global__ void __launch_bounds__(256) gather_offset_kernel(const float* __restrict__ X, int D,
                                                            const long long* __restrict__ idx, int64_t lo,
                                                            int64_t cnt, int64_t row_offset,
                                                            float* __restrict__ Y) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < cnt;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const float* src = X + (idx[lo + r] - row_offset) * D;
    float* dst = Y + r * D;
    for (int c = lane; c < D; c += 32) dst[c] = __ldg(src + c);
  }
}

__global__ void dirs_to_f32_kernel(const double* U64, float* U32, int total) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x)
    U32[i] = static_cast<float>(U64[i]);
}

// ------------------------------------------------------------------ K4 band-select fallback
// When the guard band of a (direction, tail) list holds more candidates than the buffer (cap =
// m + 65536; e.g. > 65536 exact duplicates at the m-th value), the list is selected exactly by a
// streaming radix select over the composite key (fp64 projection, index) of every candidate
// (pi32 inside the collect range): 8 rounds of 8 bits over the order-preserving fp64 key, 4 over
// the index, each a pass over the projections that recomputes the fp64 dot of the candidates
// (no candidate storage). The m smallest keys are then gathered (exactly m: the key is unique)
// and ranked by rank_kernel like a normal list. Scratch lives in the (then idle) histogram
// buffer: hist[lt][256], then per list {k1 hi, k1 lo, k2, remaining}, a redo flag, a counter.
constexpr int kBandRounds = 12;
struct BandScratch {
  unsigned* hist;   // [2L][256]
  unsigned* st;     // [2L][4]
  unsigned* redo;   // [2L]
  unsigned* gcnt;   // [2L]
};
__device__ __forceinline__ BandScratch band_scratch(unsigned* base, int L) {
  BandScratch b;
  b.hist = base;
  b.st = base + 2 * L * 256;
  b.redo = b.st + 2 * L * 4;
  b.gcnt = b.redo + 2 * L;
  return b;
}
// smaller key = better: top tail (larger pi first), bottom tail (smaller pi first)
__device__ __forceinline__ unsigned long long band_k1(double pi, int t) {
  unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(pi == 0.0 ? 0.0 : pi));
  u = (u >> 63) ? ~u : (u | 0x8000000000000000ull);  // ascending order-preserving
  return t == 0 ? ~u : u;
}

__global__ void band_init_kernel(unsigned* base, int L, const int* n_dirs, const unsigned* ccount, int64_t cap,
                                 int64_t m) {
  const BandScratch b = band_scratch(base, L);
  for (int i = threadIdx.x; i < 2 * L * 256; i += blockDim.x) b.hist[i] = 0u;
  for (int lt = threadIdx.x; lt < 2 * L; lt += blockDim.x) {
    const bool ov = (lt >> 1) < *n_dirs && static_cast<int64_t>(ccount[lt]) > cap;
    b.redo[lt] = ov ? 1u : 0u;
    b.gcnt[lt] = 0u;
    b.st[lt * 4 + 0] = 0u;
    b.st[lt * 4 + 1] = 0u;
    b.st[lt * 4 + 2] = 0u;
    b.st[lt * 4 + 3] = static_cast<unsigned>(m);
  }
}

// one pass over the projections of list lt = blockIdx.y: every candidate's fp64 key, matched
// against the decided prefix; round r < kBandRounds histograms the next digit, r == kBandRounds
// gathers the m winners (key <= the selected key) into cand[lt][]
__global__ void __launch_bounds__(256) band_pass_kernel(const float* __restrict__ X, int D,
                                                        const double* __restrict__ U64, const float* __restrict__ P32,
                                                        int64_t n, int L, const unsigned* __restrict__ state,
                                                        const unsigned* maxnorm2, double eps_coef, unsigned* base,
                                                        int round, int* cand, int64_t cap) {
  const BandScratch b = band_scratch(base, L);
  const int lt = blockIdx.y, l = lt >> 1, t = lt & 1;
  if (b.redo[lt] == 0u) return;
  __shared__ unsigned sh[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0u;
  __syncthreads();
  const double eps = eps_coef * sqrt(static_cast<double>(__uint_as_float(*maxnorm2))) * 1.0625;
  const double lim = t == 0 ? static_cast<double>(key_to_float(state[(l * 2 + 0) * 4 + 0])) - 2.0 * eps
                            : static_cast<double>(key_to_float(~state[(l * 2 + 1) * 4 + 0])) + 2.0 * eps;
  const unsigned long long K1 = (static_cast<unsigned long long>(b.st[lt * 4 + 0]) << 32) | b.st[lt * 4 + 1];
  const unsigned K2 = b.st[lt * 4 + 2];
  const float* p = P32 + static_cast<int64_t>(l) * n;
  const double* u = U64 + static_cast<int64_t>(l) * D;
  const int lane = threadIdx.x & 31;
  const int64_t nwarp = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w0 = ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 32; w0 < n;
       w0 += nwarp * 32) {
    const int64_t i = w0 + lane;
    const double x32 = i < n ? static_cast<double>(p[i]) : 0.0;
    const bool c = i < n && (t == 0 ? x32 >= lim : x32 <= lim);
    unsigned ballot = __ballot_sync(0xffffffffu, c);
    double mine = 0.0;
    while (ballot) {  // the warp computes each candidate's fp64 projection together
      const int src = __ffs(ballot) - 1;
      ballot &= ballot - 1;
      const float* x = X + (w0 + src) * static_cast<int64_t>(D);
      double s = 0.0;
      for (int d = lane; d < D; d += 32) s = fma(static_cast<double>(__ldg(x + d)), u[d], s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == src) mine = s;
    }
    if (!c) continue;
    const unsigned long long k1 = band_k1(mine, t);
    const unsigned k2 = static_cast<unsigned>(i);
    if (round < kBandRounds) {
      bool match;
      unsigned digit;
      if (round < 8) {
        const int sh_hi = 64 - 8 * round;  // decided bits: the top 8 * round of k1
        match = round == 0 || (k1 >> sh_hi) == (K1 >> sh_hi);
        digit = static_cast<unsigned>(k1 >> (56 - 8 * round)) & 255u;
      } else {
        const int r2 = round - 8;
        match = k1 == K1 && (r2 == 0 || (k2 >> (32 - 8 * r2)) == (K2 >> (32 - 8 * r2)));
        digit = (k2 >> (24 - 8 * r2)) & 255u;
      }
      if (match) atomicAdd(&sh[digit], 1u);
    } else if (k1 < K1 || (k1 == K1 && k2 <= K2)) {
      const unsigned pos = atomicAdd(&b.gcnt[lt], 1u);
      if (pos < cap) cand[static_cast<int64_t>(lt) * cap + pos] = static_cast<int>(i);
    }
  }
  if (round < kBandRounds) {
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
      if (sh[i]) atomicAdd(&b.hist[lt * 256 + i], sh[i]);
  }
}

// the digit holding the remaining-th best key; the decided prefix grows by 8 bits
__global__ void band_scan_kernel(int L, unsigned* base, int round) {
  const BandScratch b = band_scratch(base, L);
  const int lt = blockIdx.x;
  if (b.redo[lt] == 0u || threadIdx.x != 0) return;
  unsigned* h = b.hist + lt * 256;
  unsigned rem = b.st[lt * 4 + 3], cum = 0u;
  int d = 0;
  for (; d < 255; ++d) {
    if (cum + h[d] >= rem) break;
    cum += h[d];
  }
  b.st[lt * 4 + 3] = rem - cum;
  if (round < 4) b.st[lt * 4 + 0] |= static_cast<unsigned>(d) << (24 - 8 * round);
  else if (round < 8) b.st[lt * 4 + 1] |= static_cast<unsigned>(d) << (24 - 8 * (round - 4));
  else b.st[lt * 4 + 2] |= static_cast<unsigned>(d) << (24 - 8 * (round - 8));
  for (int i = 0; i < 256; ++i) h[i] = 0u;
}

__global__ void band_finish_kernel(int L, unsigned* base, unsigned* ccount) {
  const BandScratch b = band_scratch(base, L);
  for (int lt = threadIdx.x; lt < 2 * L; lt += blockDim.x)
    if (b.redo[lt]) ccount[lt] = b.gcnt[lt];
}

__global__ void init_state_kernel(unsigned* state, int L, int64_t m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 2 * L) {
    state[i * 4 + 0] = 0u;
    state[i * 4 + 1] = 0u;
    state[i * 4 + 2] = static_cast<unsigned>(m);
    state[i * 4 + 3] = 0u;
  }
}

}  // namespace

cudaError_t launch_dirs_to_f32(const double* U64, float* U32, int rows, int D, cudaStream_t st) {
  count_launch();
  dirs_to_f32_kernel<<<(rows * D + 255) / 256, 256, 0, st>>>(U64, U32, rows * D);
  return cudaGetLastError();
}

// K3: the tcgen05 3xTF32 kernel (k_project_tc.cu) where it applies, else the SIMT kernels;
// *eps_coef receives the coefficient of max||x|| that bounds |pi32 - pi64| for the kernel run.
cudaError_t launch_project(const float* X, int64_t n, int D, const float* U32, int L, float* P32,
                                  unsigned* maxnorm2, cudaStream_t st, double* eps_coef) {
  cudaError_t e = cudaSuccess;
  if (project_tc_supported(n, D, L)) {
    static int sms = 0;
    if (sms == 0) {
      int dev = 0;
      if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) !=
                                                    cudaSuccess || sms <= 0)
        sms = 148;
    }
    *eps_coef = project_tc_eps_coef(D);
    return launch_project_tc(X, n, D, U32, L, P32, maxnorm2, sms, st);
  }
  *eps_coef = (D + 8) * 0x1p-24;  // sequential fp32 FMA sums of D + 1 terms, u rounded to fp32
  const size_t tsmem0 = sizeof(float) * (((L * D + 3) & ~3) + 2 * kPP * kXS);
  if (D % 4 == 0 && L <= 32 && tsmem0 <= 200 * 1024) {
    int64_t tiles = (n + kPP - 1) / kPP;
    if (tiles > 2 * 148) tiles = 2 * 148;
    auto launch = [&](auto kern) -> cudaError_t {
      cudaError_t ee = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(tsmem0));
      if (ee != cudaSuccess) return ee;
      count_launch();
      kern<<<static_cast<int>(tiles), kPP, tsmem0, st>>>(X, n, D, U32, L, P32, maxnorm2);
      return cudaGetLastError();
    };
    switch (L) {  // exact direction counts of the BASELINE configs (k+1 = 5, 9, 17) unroll fully
      case 1: e = launch(project_tile_kernel<1, true>); break;
      case 5: e = launch(project_tile_kernel<5, true>); break;
      case 9: e = launch(project_tile_kernel<9, true>); break;
      case 17: e = launch(project_tile_kernel<17, true>); break;
      default:
        if (L <= 8)
          e = launch(project_tile_kernel<8, false>);
        else if (L <= 16)
          e = launch(project_tile_kernel<16, false>);
        else if (L <= 24)
          e = launch(project_tile_kernel<24, false>);
        else
          e = launch(project_tile_kernel<32, false>);
    }
    if (e != cudaSuccess) return e;
  } else {
    const size_t psmem = sizeof(float) * L * D;
    if ((e = cudaFuncSetAttribute(project_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(psmem))) != cudaSuccess)
      return e;
    int64_t pblocks = (n + 7) / 8;
    if (pblocks > 148 * 8) pblocks = 148 * 8;
    count_launch();
    project_kernel<<<static_cast<int>(pblocks), 256, psmem, st>>>(X, n, D, U32, L, P32, maxnorm2);
  }
  return e;
}

cudaError_t launch_select(const float* X, int64_t n, int D, const double* U64, const float* U32, int L,
                          const int* n_dirs, int64_t m, const SelectBufs& b, cudaStream_t st, bool first,
                          bool last, double* eps_out) {
  cudaError_t e;
  if (first) {
    if ((e = cudaMemsetAsync(b.maxnorm2, 0, sizeof(unsigned), st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(b.bitmap, 0, sizeof(unsigned) * ((n + 31) / 32), st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(b.overflow, 0, sizeof(int), st)) != cudaSuccess) return e;
  }
  if ((e = cudaMemsetAsync(b.hist, 0, sizeof(unsigned) * 3 * L * 2 * kRadixBins, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(b.ccount, 0, sizeof(unsigned) * 2 * L, st)) != cudaSuccess) return e;
  count_launch();
  init_state_kernel<<<1, 2 * L < 1024 ? 1024 : 2 * L, 0, st>>>(b.state, L, m);
  // K3
  double eps_coef = 0.0;
  if ((e = launch_project(X, n, D, U32, L, b.P32, b.maxnorm2, st, &eps_coef)) != cudaSuccess) return e;
  if (eps_out != nullptr) *eps_out = eps_coef;
  // K4: three radix rounds
  int64_t hb = (n + 255) / 256;
  if (hb > 148 * 2) hb = 148 * 2;
  for (int r = 0; r < 3; ++r) {
    count_launch();
    radix_hist_kernel<<<dim3(static_cast<unsigned>(hb), L), 256, 0, st>>>(b.P32, n, L, n_dirs, r, b.state, b.hist);
    count_launch();
    radix_scan_kernel<<<2 * L, kScanT, 0, st>>>(b.hist, L, n_dirs, r, b.state);
  }
  count_launch();
  collect_kernel<<<dim3(static_cast<unsigned>(hb), L), 256, 0, st>>>(b.P32, n, D, L, n_dirs, b.state, b.maxnorm2,
                                                                     b.cand, b.ccount, b.cap, b.overflow, 0, eps_coef);
  count_launch();
  cand_p64_kernel<<<dim3(16, 2 * L), 256, 0, st>>>(X, D, U64, L, n_dirs, b.cand, b.ccount, b.cap, b.cval);
  count_launch();
  rank_kernel<<<dim3(32, 2 * L), 256, 0, st>>>(L, n_dirs, b.cand, b.cval, b.ccount, b.cap, m, b.lists, b.bitmap,
                                              nullptr, nullptr, 0, nullptr);
  // K5
  if (last) {
    count_launch();
    compact_count_kernel<<<kCB, 256, 0, st>>>(b.bitmap, (n + 31) / 32, b.ucount + 1);
    count_launch();
    compact_write_kernel<<<kCB, 256, 0, st>>>(b.bitmap, (n + 31) / 32, b.ucount + 1, b.uidx, b.ucount);
  }
  return cudaGetLastError();
}

bool select_sampled_plan(int64_t n, int D, int L, int64_t m, int* s_out, unsigned* r_out) {
  const long long o = opt(OPT_K4_SAMPLED);
  if (o == 0 || (o < 0 && n < 262144)) return false;
  if (!project_tc_supported(n, D, L) || m < 1 || 2 * m >= n) return false;
  const int s = static_cast<int>(n < kSampleMax ? n : kSampleMax);
  // about mu of the s sample points lie beyond the true m-th value; the r-th best sample value
  // is then passed by ~(r / mu) m points (r / mu ~ 3.5 at cfg5, 2.4 at cfg2), and by fewer than
  // m only if the sample holds r >= 2 mu + 4 sqrt(mu) + 8 points beyond the m-th value (Poisson
  // tail < 1e-13 for mu >= 16); the filter certifies every list anyway
  const double mu = static_cast<double>(s) * static_cast<double>(m) / static_cast<double>(n);
  const double r = std::ceil(2.0 * mu + 4.0 * std::sqrt(mu)) + 8.0;
  if (r > s / 8) return false;  // not a tail: the radix path
  // about r n / s points pass the threshold: they must fit the filter's shared-memory stage
  if (r * static_cast<double>(n / s) > kFilterStage / 2) return false;
  *s_out = s;
  *r_out = static_cast<unsigned>(r);
  return true;
}

cudaError_t launch_select_sampled(const float* X, int64_t n, int D, const double* U64, const float* U32, int L,
                                  const int* n_dirs, int64_t m, const SelectBufs& b, cudaStream_t st,
                                  double* eps_out, bool* used) {
  *used = false;
  int s = 0;
  unsigned r = 0;
  if (b.sfail == nullptr || !select_sampled_plan(n, D, L, m, &s, &r)) return cudaSuccess;
  int sms = 0, dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) !=
                                                cudaSuccess || sms <= 0)
    sms = 148;
  // the appended slabs and the sample projections live in the P32 buffer (L n floats), which this
  // path does not otherwise use: per epilogue warp (4 per K3 CTA) and list kSlabCap indices and
  // values, then the fill counts
  const int64_t ntiles = (n + 127) / 128;
  // K3 CTAs: one per SM, fewer for small n so that the slabs fit the buffer (sample-size tests)
  int64_t ctas = ntiles < sms ? ntiles : sms;
  const int64_t fit = static_cast<int64_t>(L) * n / (8 * L * (2 * kSlabCap + 1));
  if (ctas > fit) ctas = fit;
  if (ctas > 1024) ctas = 1024;  // cand_filter_kernel: <= 4 slabs per thread
  if (ctas < 1) return cudaSuccess;
  const int nslabs = 4 * static_cast<int>(ctas);
  *used = true;
  ProjectFuse fz;
  fz.state = b.state;
  fz.capw = kSlabCap;
  fz.ablate = opt(OPT_K4_SAMPLED) >= 2 ? static_cast<int>(opt(OPT_K4_SAMPLED)) - 1 : 0;
  fz.sidx = reinterpret_cast<int*>(b.P32);
  fz.sval = b.P32 + static_cast<int64_t>(nslabs) * 2 * L * kSlabCap;
  fz.wcount = reinterpret_cast<unsigned*>(b.P32 + static_cast<int64_t>(nslabs) * 2 * L * kSlabCap * 2);
  cudaError_t e;
  if ((e = cudaMemsetAsync(b.maxnorm2, 0, sizeof(unsigned), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(b.bitmap, 0, sizeof(unsigned) * ((n + 31) / 32), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(b.overflow, 0, sizeof(int), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(b.sfail, 0, sizeof(int), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(b.ccount, 0, sizeof(unsigned) * 2 * L, st)) != cudaSuccess) return e;
  // sample projections: K3 itself on rows 0, step, 2 step, ... (a strided TMA view), into the
  // P32 buffer (consumed by sample_thresh_kernel before K3 proper writes the raw lists there)
  const int64_t step = n / s;
  float* S = b.P32;
  if ((e = launch_project_tc(X, s, D, U32, L, S, b.maxnorm2, sms, st, nullptr, step * D)) != cudaSuccess) return e;
  const size_t tsmem = sizeof(float) * static_cast<size_t>(s) + sizeof(unsigned) * kSelHistWords;
  const size_t fsmem = (sizeof(float) + sizeof(int)) * static_cast<size_t>(kFilterStage) +
                       sizeof(unsigned) * kSelHistWords;
  if ((e = cudaFuncSetAttribute(sample_thresh_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(tsmem))) != cudaSuccess ||
      (e = cudaFuncSetAttribute(cand_filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(fsmem))) != cudaSuccess)
    return e;
  count_launch();
  sample_thresh_kernel<<<2 * L, kSelThreads, tsmem, st>>>(S, s, n_dirs, r, b.state);
  const double eps_coef = project_tc_eps_coef(D);
  if (eps_out != nullptr) *eps_out = eps_coef;
  if ((e = launch_project_tc(X, n, D, U32, L, b.P32, b.maxnorm2, static_cast<int>(ctas), st, &fz)) != cudaSuccess)
    return e;
  count_launch();
  cand_filter_kernel<<<2 * L, kSelThreads, fsmem, st>>>(n_dirs, b.state, fz.sidx, fz.sval, fz.wcount, nslabs, L, kSlabCap,
                                                m, b.maxnorm2, eps_coef, b.cand, b.ccount, b.cap, b.overflow,
                                                b.sfail);
  count_launch();
  cand_p64_kernel<<<dim3(16, 2 * L), 256, 0, st>>>(X, D, U64, L, n_dirs, b.cand, b.ccount, b.cap, b.cval);
  count_launch();
  rank_kernel<<<dim3(32, 2 * L), 256, 0, st>>>(L, n_dirs, b.cand, b.cval, b.ccount, b.cap, m, b.lists, b.bitmap,
                                              nullptr, nullptr, 0, nullptr);
  count_launch();
  compact_count_kernel<<<kCB, 256, 0, st>>>(b.bitmap, (n + 31) / 32, b.ucount + 1);
  count_launch();
  compact_write_kernel<<<kCB, 256, 0, st>>>(b.bitmap, (n + 31) / 32, b.ucount + 1, b.uidx, b.ucount);
  return cudaGetLastError();
}

__global__ void minus_one_kernel(const int* a, int* b) { *b = *a > 0 ? *a - 1 : 0; }

cudaError_t launch_select_fallback(const float* X, int64_t n, int D, const double* U64, int L, const int* n_dirs,
                                   int64_t m, const SelectBufs& b, double eps_coef, cudaStream_t st, bool compact,
                                   double* cval_out, long long* cidx_out, int64_t row_offset) {
  // the histogram buffer (3 L 2 kRadixBins words) holds the band scratch (2L (256 + 6) words)
  int64_t hb = (n + 255) / 256;
  if (hb > 148 * 2) hb = 148 * 2;
  count_launch();
  band_init_kernel<<<1, 256, 0, st>>>(b.hist, L, n_dirs, b.ccount, b.cap, m);
  for (int r = 0; r <= kBandRounds; ++r) {
    count_launch();
    band_pass_kernel<<<dim3(static_cast<unsigned>(hb), 2 * L), 256, 0, st>>>(X, D, U64, b.P32, n, L, b.state,
                                                                             b.maxnorm2, eps_coef, b.hist, r,
                                                                             b.cand, b.cap);
    if (r < kBandRounds) {
      count_launch();
      band_scan_kernel<<<2 * L, 32, 0, st>>>(L, b.hist, r);
    }
  }
  count_launch();
  band_finish_kernel<<<1, 256, 0, st>>>(L, b.hist, b.ccount);
  count_launch();
  cand_p64_kernel<<<dim3(16, 2 * L), 256, 0, st>>>(X, D, U64, L, n_dirs, b.cand, b.ccount, b.cap, b.cval);
  const unsigned* redo = b.hist + 2 * L * 256 + 2 * L * 4;
  count_launch();
  if (cval_out != nullptr)
    rank_kernel<<<dim3(32, 2 * L), 256, 0, st>>>(L, n_dirs, b.cand, b.cval, b.ccount, b.cap, m, nullptr, nullptr,
                                                cval_out, cidx_out, row_offset, redo);
  else
    rank_kernel<<<dim3(32, 2 * L), 256, 0, st>>>(L, n_dirs, b.cand, b.cval, b.ccount, b.cap, m, b.lists, b.bitmap,
                                                nullptr, nullptr, 0, redo);
  if (compact) {
    count_launch();
    compact_count_kernel<<<kCB, 256, 0, st>>>(b.bitmap, (n + 31) / 32, b.ucount + 1);
    count_launch();
    compact_write_kernel<<<kCB, 256, 0, st>>>(b.bitmap, (n + 31) / 32, b.ucount + 1, b.uidx, b.ucount);
  }
  return cudaGetLastError();
}

// prohd_estimate's host reads, gathered into one small buffer (one D2H copy per read point):
// status: [0,1] union sizes, [2,3] overflow flags, [4,5] max squared-norm bits, [6] n_dirs,
// [7] int8-Gram range flag, [8,9] sampled-threshold certification failures (0 for null sources)
__global__ void pack_status_kernel(StatusSrc src, unsigned* out) {
  const int t = threadIdx.x;
  unsigned v = 0;
  switch (t) {
    case 0: v = *src.uc[0]; break;
    case 1: v = *src.uc[1]; break;
    case 2: v = static_cast<unsigned>(*src.ovf[0]); break;
    case 3: v = static_cast<unsigned>(*src.ovf[1]); break;
    case 4: v = *src.maxn[0]; break;
    case 5: v = *src.maxn[1]; break;
    case 6: v = static_cast<unsigned>(*src.ndirs); break;
    case 7: v = src.i8ovf ? *src.i8ovf : 0u; break;
    case 8: v = src.sfail[0] ? static_cast<unsigned>(*src.sfail[0]) : 0u; break;
    case 9: v = src.sfail[1] ? static_cast<unsigned>(*src.sfail[1]) : 0u; break;
    default: return;
  }
  out[t] = v;
}
cudaError_t launch_pack_status(const StatusSrc& src, unsigned* out, cudaStream_t st) {
  count_launch();
  pack_status_kernel<<<1, 32, 0, st>>>(src, out);
  return cudaGetLastError();
}

// the end of prohd_estimate: both directed results with the witness rows mapped to original
// indices through the unions (uA, uB; null = the columns already are original indices)
__global__ void pack_result_kernel(const unsigned long long* keys, const double* nn_d, const long long* nn_j,
                                   const long long* uA, const long long* uB, bool map_cols, EstResultDev* out) {
  if (threadIdx.x != 0) return;
  for (int s = 0; s < 2; ++s) {
    const unsigned long long key = keys[s];
    const long long row = static_cast<long long>(0xFFFFFFFFu - static_cast<unsigned>(key & 0xFFFFFFFFull));
    const long long* ur = s == 0 ? uA : uB;  // rows: subset of the first set of this direction
    const long long* uc = s == 0 ? uB : uA;
    out->key[s] = key;
    out->d2[s] = nn_d[s];
    out->a[s] = ur[row];
    out->b[s] = map_cols ? uc[nn_j[s]] : nn_j[s];
  }
}
cudaError_t launch_pack_result(const unsigned long long* keys, const double* nn_d, const long long* nn_j,
                               const long long* uA, const long long* uB, bool map_cols, EstResultDev* out,
                               cudaStream_t st) {
  count_launch();
  pack_result_kernel<<<1, 32, 0, st>>>(keys, nn_d, nn_j, uA, uB, map_cols, out);
  return cudaGetLastError();
}

__global__ void set_int_kernel(int* a, int v) { *a = v; }
cudaError_t launch_set_int(int* a, int v, cudaStream_t st) {
  count_launch();
  set_int_kernel<<<1, 1, 0, st>>>(a, v);
  return cudaGetLastError();
}

__global__ void pack_exact_kernel(const unsigned long long* keys, const double* nn_d, const long long* nn_j,
                                  const int* bad, ExactResDev* out) {
  if (threadIdx.x != 0) return;
  for (int s = 0; s < 2; ++s) {
    out->key[s] = keys[s];
    out->d2[s] = nn_d[s];
    out->j[s] = nn_j[s];
  }
  out->bad = *bad;
  out->_pad = 0;
}
cudaError_t launch_pack_exact(const unsigned long long* keys, const double* nn_d, const long long* nn_j,
                              const int* bad, ExactResDev* out, cudaStream_t st) {
  count_launch();
  pack_exact_kernel<<<1, 32, 0, st>>>(keys, nn_d, nn_j, bad, out);
  return cudaGetLastError();
}

cudaError_t launch_minus_one(const int* a, int* b, cudaStream_t st) {
  count_launch();
  minus_one_kernel<<<1, 1, 0, st>>>(a, b);
  return cudaGetLastError();
}

cudaError_t launch_local_candidates(const float* X, int64_t n, int64_t row_offset, int D, const double* U64,
                                    const float* U32, int L, const int* n_dirs, int64_t m, const SelectBufs& b,
                                    double* cval_out, long long* cidx_out, cudaStream_t st, double* eps_out) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(cidx_out, 0xFF, sizeof(long long) * L * 2 * m, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(cval_out, 0, sizeof(double) * L * 2 * m, st)) != cudaSuccess) return e;
  if (n <= 0) return cudaSuccess;
  if ((e = cudaMemsetAsync(b.maxnorm2, 0, sizeof(unsigned), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(b.hist, 0, sizeof(unsigned) * 3 * L * 2 * kRadixBins, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(b.ccount, 0, sizeof(unsigned) * 2 * L, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(b.overflow, 0, sizeof(int), st)) != cudaSuccess) return e;
  const bool all = m >= n;
  count_launch();
  init_state_kernel<<<1, 2 * L < 1024 ? 1024 : 2 * L, 0, st>>>(b.state, L, all ? 1 : m);
  double eps_coef = 0.0;
  if ((e = launch_project(X, n, D, U32, L, b.P32, b.maxnorm2, st, &eps_coef)) != cudaSuccess) return e;
  if (eps_out != nullptr) *eps_out = eps_coef;
  int64_t hb = (n + 255) / 256;
  if (hb > 148 * 2) hb = 148 * 2;
  if (!all) {
    for (int r = 0; r < 3; ++r) {
      count_launch();
      radix_hist_kernel<<<dim3(static_cast<unsigned>(hb), L), 256, 0, st>>>(b.P32, n, L, n_dirs, r, b.state, b.hist);
      count_launch();
      radix_scan_kernel<<<2 * L, kScanT, 0, st>>>(b.hist, L, n_dirs, r, b.state);
    }
  }
  count_launch();
  collect_kernel<<<dim3(static_cast<unsigned>(hb), L), 256, 0, st>>>(b.P32, n, D, L, n_dirs, b.state, b.maxnorm2,
                                                                     b.cand, b.ccount, b.cap, b.overflow, all ? 1 : 0,
                                                                     eps_coef);
  count_launch();
  cand_p64_kernel<<<dim3(16, 2 * L), 256, 0, st>>>(X, D, U64, L, n_dirs, b.cand, b.ccount, b.cap, b.cval);
  count_launch();
  rank_kernel<<<dim3(32, 2 * L), 256, 0, st>>>(L, n_dirs, b.cand, b.cval, b.ccount, b.cap, m, nullptr, nullptr,
                                              cval_out, cidx_out, row_offset, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_merge_union(const double* cval, const long long* cidx, int G, int L, int64_t m, int64_t n_total,
                               unsigned* bitmap, long long* uidx, unsigned* ucount, const int* n_dirs,
                               cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(bitmap, 0, sizeof(unsigned) * ((n_total + 31) / 32), st);
  if (e != cudaSuccess) return e;
  count_launch();
  merge_rank_kernel<<<dim3(16, 2 * L), 256, 0, st>>>(cval, cidx, G, L, n_dirs, m, bitmap);
  count_launch();
  compact_count_kernel<<<kCB, 256, 0, st>>>(bitmap, (n_total + 31) / 32, ucount + 1);
  count_launch();
  compact_write_kernel<<<kCB, 256, 0, st>>>(bitmap, (n_total + 31) / 32, ucount + 1, uidx, ucount);
  return cudaGetLastError();
}

cudaError_t launch_gather_offset(const float* X, int D, const long long* idx, int64_t lo, int64_t cnt,
                                 int64_t row_offset, float* rows_out, cudaStream_t st) {
  if (cnt <= 0) return cudaSuccess;
  int64_t blocks = (cnt + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  count_launch();
  gather_offset_kernel<<<static_cast<int>(blocks), 256, 0, st>>>(X, D, idx, lo, cnt, row_offset, rows_out);
  return cudaGetLastError();
}

cudaError_t launch_iota(long long* idx, unsigned* count, int64_t n, cudaStream_t st) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  count_launch();
  iota_kernel<<<static_cast<int>(blocks), 256, 0, st>>>(idx, count, n);
  return cudaGetLastError();
}

cudaError_t launch_gather(const float* X, int D, const long long* idx, const unsigned* count, int64_t cap,
                          float* Y, cudaStream_t st) {
  int64_t blocks = (cap + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  count_launch();
  gather_kernel<<<static_cast<int>(blocks), 256, 0, st>>>(X, D, idx, count, Y);
  return cudaGetLastError();
}

}  // namespace prohd
