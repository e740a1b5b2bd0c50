// k_moments.cu — K1: centroid sums and the covariance of A u B (ProHD step 1a).
//
// PAPER.md Alg. 1 line 1 (centroids) and Alg. 2 lines 1-2 (P:231-232,
// "Stack points Z~ = [X;Y]" / "Compute the top m principal components"): the
// principal components are eigenvectors of
//     C = (1/N) sum_{p in A u B} (p - mu)(p - mu)^T,   N = nA + nB.
// One pass over the data with a shift s (fp64 mean of the first <= 4096 rows of
// A and of B) so no large-mean cancellation occurs:
//     S_X = sum_{x in X} (x - s),  G = sum_{p in A u B} (p - s)(p - s)^T
//     mu_X = S_X / n_X + s,  C = G / N - (mu - s)(mu - s)^T.
// Arithmetic: fp64 (products of exact fp64 differences, fp64 accumulation). The
// direction parity bar (near-degenerate spectra down to
// relative gaps 1.1e-4) needs C far more accurate than fp32 tensor-core
// accumulation gives, so this step runs on the fp64 pipes.
//
// Decomposition: the upper triangle of G in 64x64 feature blocks (pair bi <= bj);
// grid = (pair, point range). 256 threads = 4 groups x 64; each thread owns an
// 8x8 register block; each group streams its share of every 64-point chunk from
// shared memory. Per-CTA partials are written to their own slot and reduced in a
// fixed order (deterministic, run-to-run bit-identical).
#include "internal.cuh"
#include "prohd_kernels.cuh"

#include <cooperative_groups.h>

#include <cstdlib>

namespace prohd {
namespace {

constexpr int kFB = 64;       // feature block

// Shift s (fp64, D values; s + D: D doubles of scratch). m = fp64 mean of the first
// <= 4096 rows of A and of B, v = their per-feature variance. One CTA per 32 features:
// lane = feature (coalesced 128-B rows), warp w sums rows w, w + 32, ... then a
// fixed-order tree over the 32 warps (deterministic). shift_decide_kernel then keeps
// s = m only if the mean offset is large against the spread (sum m^2 > 1024 sum v): the
// Gram pass subtracts s in fp64, which costs fp64-pipe time; with s = 0 it multiplies
// the raw fp32 values, whose products are exact in fp64, and the centring happens in
// moments_finalize (C = G/N - mu mu^T), whose cancellation grows with the ratio. Measured
// at full size (tools/dir_accuracy.py): cfg4 (ratio 31.7, top-16 gaps down to 1.1e-4)
// gives PC sin-angles of 2.7e-12 unshifted vs 1.2e-13 shifted, against a selection
// margin of 5e-8; linear in the ratio, the 1024 bound keeps them below ~1e-10.
// One 8-CTA cluster per 32 features: CTA q of the cluster takes rows [512 q, 512 q + 512) of
// the first <= 4096 rows of each set (warp w: rows 512 q + w + 32 u), the 32 warps combine in a
// fixed tree, and CTA 0 adds the 8 CTA partials in rank order through distributed shared
// memory (latency-bound kernel: 8x the memory-level parallelism of one CTA per 32 features).
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(1024) shift_kernel(const float* __restrict__ A, int64_t nA,
                                                                               const float* __restrict__ B, int64_t nB,
                                                                               int D, double* __restrict__ s) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double part[4][32][33];  // sum and sum of squares, of A and of B
  __shared__ double clpart[8][4][32];  // CTA partials (used in rank 0)
  const int rank = static_cast<int>(cl.block_rank());
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int f = (blockIdx.x / 8) * 32 + lane;
  const int64_t ca = nA < 4096 ? nA : 4096;
  const int64_t cb = nB < 4096 ? nB : 4096;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (f < D) {
    const int64_t r0 = 512 * rank + w;
    float va[16], vb[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int64_t r = r0 + 32 * u;
      va[u] = r < ca ? __ldg(A + r * D + f) : 0.0f;
      vb[u] = r < cb ? __ldg(B + r * D + f) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const double x = static_cast<double>(va[u]), y = static_cast<double>(vb[u]);
      acc[0] += x;
      acc[1] += x * x;
      acc[2] += y;
      acc[3] += y * y;
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) part[q][w][lane] = acc[q];
  __syncthreads();
  for (int o = 16; o > 0; o >>= 1) {
    if (w < o)
#pragma unroll
      for (int q = 0; q < 4; ++q) part[q][w][lane] += part[q][w + o][lane];
    __syncthreads();
  }
  if (w < 4) *cl.map_shared_rank(&clpart[rank][w][lane], 0) = part[w][0][lane];
  cl.sync();
  if (rank == 0 && w == 0 && f < D) {
    double t[4] = {0.0, 0.0, 0.0, 0.0};
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int k = 0; k < 4; ++k) t[k] += clpart[q][k][lane];
    // per-set sums added last: the same bits for (A, B) and (B, A)
    const double cnt = static_cast<double>(ca + cb);
    const double m = (t[0] + t[2]) / cnt;
    s[f] = m;
    s[D + f] = fmax((t[1] + t[3]) / cnt - m * m, 0.0);
  }
}

__global__ void __launch_bounds__(256) shift_decide_kernel(double* __restrict__ s, int D, int force) {
  __shared__ double r1[256], r2[256];
  double a = 0.0, b = 0.0;
  for (int f = threadIdx.x; f < D; f += 256) {
    a += s[f] * s[f];
    b += s[D + f];
  }
  r1[threadIdx.x] = a;
  r2[threadIdx.x] = b;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      r1[threadIdx.x] += r1[threadIdx.x + o];
      r2[threadIdx.x] += r2[threadIdx.x + o];
    }
    __syncthreads();
  }
  const bool keep = force >= 0 ? force != 0 : r1[0] > 1024.0 * r2[0];
  if (!keep)
    for (int f = threadIdx.x; f < D; f += 256) s[f] = 0.0;
}

struct MomArgs {
  const float* A;
  const float* B;
  int64_t nA, nB;  // the CTAs of a pair split the concatenated index space [0, nA + nB)
  int D;
  const double* s;
  int nb;          // feature blocks
  int c_diag;      // CTAs per diagonal pair (bi == bj)
  int c_off;       // CTAs per off-diagonal pair
  int nslots;      // max(c_diag, c_off): partial-slot stride of a pair
  double* Gpart;   // [pair][nslots][64][64]
  double* Spart;   // [bi][c_diag][2 sets][64]
};

__device__ __forceinline__ void pair_of(int p, int nb, int& bi, int& bj) {
  // enumerate (bi <= bj) row-major
  int r = 0;
  while (p >= nb - r) {
    p -= nb - r;
    ++r;
  }
  bi = r;
  bj = r + p;
}

// fp64 tensor-core MMA (legacy warp-level DMMA): D[8x8] += A[8x4] * B[4x8], fp64 in and out.
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Row stride (doubles) of the chunk tile: 128 features + 4 pad. A fragment load reads
// rows k0 + (lane & 3) at columns base + (lane >> 2); a 64-bit load is served per
// half-warp, whose 16 addresses (fk * kLds + fr, fk, fr < 4) fall in distinct bank pairs
// iff kLds = 4 (mod 16).
constexpr int kLds = 132;
constexpr int kMT = 128;    // threads per CTA (4 warps)
constexpr int kMC = 32;     // points per chunk
// resident CTAs per SM (register-limited: 160 regs at 3, 128 at 4). option k1_ctas = 3|4 (dev A/B).
static int mom_ctas_per_sm() {
  return opt(OPT_K1_CTAS) == 3 ? 3 : 4;
}

// CTA -> (bi, bj, pair index, slot). Pairs (bi <= bj) are enumerated row-major; row r
// holds the diagonal pair (c_diag CTAs) then nb-1-r off-diagonal pairs (c_off CTAs each).
__device__ __forceinline__ void cta_work(int cta, int nb, int c_diag, int c_off, int& bi, int& bj, int& pair,
                                         int& slot) {
  int r = 0, pbase = 0;
  for (;;) {
    const int row_ctas = c_diag + (nb - 1 - r) * c_off;
    if (cta < row_ctas || r == nb - 1) break;
    cta -= row_ctas;
    pbase += nb - r;
    ++r;
  }
  bi = r;
  if (cta < c_diag) {
    bj = r;
    slot = cta;
  } else {
    cta -= c_diag;
    bj = r + 1 + cta / c_off;
    slot = cta % c_off;
  }
  pair = pbase + (bj - r);
}

// One CTA: one 64x64 block (bi, bj) of G over one range of the concatenated points of
// A u B (G is a sum over the union; the column sums S_A, S_B are kept apart). 4 warps,
// warp w owns the 32x32 tile (w/2, w%2) = 4 x 4 DMMA tiles (16 MMAs per 8 fragment
// loads). In diagonal blocks the strictly-lower warp tile (1,0) is skipped (its mirror
// (0,1) is computed). The grid is one wave (kMomCtasPerSm per SM) with CTA counts per
// pair proportional to the pair's warp tiles (3 diagonal, 4 off-diagonal), so every CTA
// carries about the same work. The next 32-point chunk is prefetched into registers
// while the current one is multiplied.
template <int kCtas>
__global__ void __launch_bounds__(kMT, kCtas) moments_kernel(MomArgs a) {
  extern __shared__ double cs[];  // [kMC][kLds]: features of block bi (0..63) then bj (64..127)
  int bi, bj, pair, slot;
  cta_work(blockIdx.x, a.nb, a.c_diag, a.c_off, bi, bj, pair, slot);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t N = a.nA + a.nB;
  const int cp = bi == bj ? a.c_diag : a.c_off;
  const int64_t per = (N + cp - 1) / cp;
  const int64_t p0 = static_cast<int64_t>(slot) * per;
  const int64_t p1 = p0 + per < N ? p0 + per : N;

  // loader mapping: thread -> feature column lf (0..127)
  const int lf = tid;
  const int feat = lf < 64 ? bi * kFB + lf : bj * kFB + (lf - 64);
  const bool fvalid = feat < a.D;
  const double sf = fvalid ? a.s[feat] : 0.0;
  double ssA = 0.0, ssB = 0.0;  // column sums of (x - s) over A and over B (used by diagonal pairs)

  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const bool active = !(bi == bj && wm > wn);
  const int fr = lane >> 2, fk = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  float pre[kMC];
  auto load = [&](int64_t c0) {
#pragma unroll
    for (int r = 0; r < kMC; ++r) {
      const int64_t p = c0 + r;
      const float* src = p < a.nA ? a.A + p * a.D : a.B + (p - a.nA) * a.D;
      pre[r] = (p < p1 && fvalid) ? __ldg(src + feat) : 0.0f;
    }
  };
  if (p0 < p1) load(p0);
  for (int64_t c0 = p0; c0 < p1; c0 += kMC) {
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kMC; ++r) {
      const int64_t p = c0 + r;
      const double v = (p < p1 && fvalid) ? static_cast<double>(pre[r]) - sf : 0.0;
      cs[r * kLds + lf] = v;
      if (p < a.nA)
        ssA += v;
      else
        ssB += v;
    }
    __syncthreads();
    if (c0 + kMC < p1) load(c0 + kMC);  // in flight during the MMAs below
    if (active) {
#pragma unroll 2
      for (int k0 = 0; k0 < kMC; k0 += 4) {
        const double* row = cs + (k0 + fk) * kLds;
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = row[wm + i * 8 + fr];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = row[64 + wn + j * 8 + fr];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
      }
    }
  }
  double* out = a.Gpart + (static_cast<int64_t>(pair) * a.nslots + slot) * (kFB * kFB);
  if (active) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = wm + i * 8 + fr;
        const int c = wn + j * 8 + 2 * fk;
        *reinterpret_cast<double2*>(out + r * 64 + c) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
  }
  // column sums: only diagonal pairs, features of block bi (lf < 64)
  if (bi == bj && lf < 64) {
    double* sp = a.Spart + (static_cast<int64_t>(bi) * a.c_diag + slot) * (2 * kFB);
    sp[lf] = ssA;
    sp[kFB + lf] = ssB;
  }
}

// G (full symmetric D x D) and S_A, S_B from the partials, fixed summation order.
__global__ void __launch_bounds__(256) moments_reduce_kernel(const double* __restrict__ Gpart,
                                                             const double* __restrict__ Spart, int nb, int D,
                                                             int c_diag, int c_off, int nslots,
                                                             double* __restrict__ G, double* __restrict__ SA,
                                                             double* __restrict__ SB) {
  const int npairs = nb * (nb + 1) / 2;
  const int64_t total = static_cast<int64_t>(npairs) * kFB * kFB;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int pair = static_cast<int>(e / (kFB * kFB));
    const int w = static_cast<int>(e % (kFB * kFB));
    int bi, bj;
    pair_of(pair, nb, bi, bj);
    if (bi == bj && (w / kFB) > (w % kFB)) continue;  // diagonal blocks: upper triangle is authoritative
    const int i = bi * kFB + w / kFB, j = bj * kFB + w % kFB;
    if (i >= D || j >= D) continue;
    const int cp = bi == bj ? c_diag : c_off;
    double acc = 0.0;
    const double* src = Gpart + static_cast<int64_t>(pair) * nslots * (kFB * kFB) + w;
    for (int s = 0; s < cp; ++s) acc += src[static_cast<int64_t>(s) * (kFB * kFB)];
    G[static_cast<int64_t>(i) * D + j] = acc;
    G[static_cast<int64_t>(j) * D + i] = acc;
  }
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < D; f += gridDim.x * blockDim.x) {
    const double* sp = Spart + static_cast<int64_t>(f / kFB) * c_diag * (2 * kFB) + (f % kFB);
    double sa = 0.0, sb = 0.0;
    for (int s = 0; s < c_diag; ++s) {
      sa += sp[static_cast<int64_t>(s) * (2 * kFB)];
      sb += sp[static_cast<int64_t>(s) * (2 * kFB) + kFB];
    }
    SA[f] = sa;
    SB[f] = sb;
  }
}

// mu and u0 (Alg. 1 line 2) and C (in place over G). One block.
__global__ void __launch_bounds__(256) moments_finalize_kernel(double* __restrict__ G, const double* __restrict__ SA,
                                                               const double* __restrict__ SB,
                                                               const double* __restrict__ s, int64_t nA, int64_t nB,
                                                               int D, double* __restrict__ mu_out,
                                                               double* __restrict__ u0, double* __restrict__ dnorm) {
  __shared__ double red[256];
  const double N = static_cast<double>(nA + nB);
  double part = 0.0;
  for (int f = threadIdx.x; f < D; f += blockDim.x) {
    const double d = SB[f] / static_cast<double>(nB) - SA[f] / static_cast<double>(nA);  // mu_B - mu_A
    u0[f] = d;
    part += d * d;
    mu_out[f] = (SA[f] + SB[f]) / N + s[f];
  }
  red[threadIdx.x] = part;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  const double nrm = sqrt(red[0]);
  __syncthreads();
  for (int f = threadIdx.x; f < D; f += blockDim.x) {
    if (nrm < 1e-9)
      u0[f] = f == 0 ? 1.0 : 0.0;  // "If ||u|| < 1e-9, set u = e1"
    else
      u0[f] = u0[f] / nrm;
  }
  if (threadIdx.x == 0) *dnorm = nrm;
}

// C = G / N - (mu - s)(mu - s)^T in place, one element per thread
__global__ void __launch_bounds__(256) covariance_kernel(double* __restrict__ G, const double* __restrict__ SA,
                                                         const double* __restrict__ SB, int64_t nA, int64_t nB,
                                                         int D) {
  const double N = static_cast<double>(nA + nB);
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<int64_t>(D) * D) return;
  const int i = static_cast<int>(e / D), j = static_cast<int>(e % D);
  const double mi = (SA[i] + SB[i]) / N, mj = (SA[j] + SB[j]) / N;  // mu - s
  G[e] = G[e] / N - mi * mj;
}

}  // namespace

MomentsPlan plan_moments(int64_t nA, int64_t nB, int D, int num_sms) {
  MomentsPlan p;
  p.nb = (D + kFB - 1) / kFB;
  p.npairs = p.nb * (p.nb + 1) / 2;
  const int ndiag = p.nb, noff = p.npairs - p.nb;
  // one wave of CTAs, split over the pairs in proportion to their warp tiles (3 / 4)
  int T = mom_ctas_per_sm() * (num_sms > 0 ? num_sms : 148);
  const int64_t N = nA + nB;
  const int64_t chunks = (N + kMC - 1) / kMC;
  int cd = 1, co = noff > 0 ? 1 : 0;
  if (T < ndiag + noff) T = ndiag + noff;
  // greedy: add a CTA where it lowers the larger per-CTA work (3/cd vs 4/co) most, within T
  while (true) {
    const int used = ndiag * cd + noff * co;
    const bool can_d = used + ndiag <= T && cd < chunks;
    const bool can_o = noff > 0 && used + noff <= T && co < chunks;
    if (!can_d && !can_o) break;
    const double wd = 3.0 / cd, wo = noff > 0 ? 4.0 / co : 0.0;
    if (can_o && (wo >= wd || !can_d))
      ++co;
    else if (can_d)
      ++cd;
    else
      break;
  }
  p.c_diag = cd;
  p.c_off = co > 0 ? co : 1;
  p.nctas = ndiag * cd + noff * co;
  p.nslots = cd > p.c_off ? cd : p.c_off;
  p.gpart_doubles = static_cast<int64_t>(p.npairs) * p.nslots * kFB * kFB;
  p.spart_doubles = static_cast<int64_t>(p.nb) * p.c_diag * 2 * kFB;
  p.gram = opt(OPT_K1_PATH) != 2 && plan_gram(nA, nB, D, num_sms, p.gp);
  if (p.gram) {
    if (p.gp.gpart_doubles > p.gpart_doubles) p.gpart_doubles = p.gp.gpart_doubles;
    if (p.gp.spart_doubles > p.spart_doubles) p.spart_doubles = p.gp.spart_doubles;
  }
  // The int8 tensor-core Gram (k_gram_i8.cu) is the default for D <= 256, D % 4 == 0 (option k1_path:
  // 0 forces the fp64 DMMA Gram, 2 the legacy tile kernel).
  p.i8 = (opt(OPT_K1_PATH) == -1 || opt(OPT_K1_PATH) == 1) && plan_gram_i8(nA, nB, D, num_sms, p.ip);
  if (p.i8) p.i8_bytes = static_cast<int64_t>(gram_i8_ws_bytes(p.ip));
  return p;
}

cudaError_t launch_centre(const float* X, int64_t nX, const float* Y, int64_t nY, int D, double* c,
                          cudaStream_t st) {
  count_launch();
  shift_kernel<<<8 * ((D + 31) / 32), 1024, 0, st>>>(X, nX, Y, nY, D, c);
  return cudaGetLastError();
}

cudaError_t launch_shift(const float* A, int64_t nA, const float* B, int64_t nB, int D, double* s,
                         cudaStream_t st) {
  count_launch();
  shift_kernel<<<8 * ((D + 31) / 32), 1024, 0, st>>>(A, nA, B, nB, D, s);
  count_launch();
  const long long fo = opt(OPT_SHIFT);  // dev A/B only: 0 = never shift, 1 = always
  const int force = (fo == 0 || fo == 1) ? static_cast<int>(fo) : -1;
  shift_decide_kernel<<<1, 256, 0, st>>>(s, D, force);
  return cudaGetLastError();
}

cudaError_t launch_moments_partial(const MomentsPlan& p, const float* A, int64_t nA, const float* B, int64_t nB,
                                   int D, const MomentsBufs& b, cudaStream_t st, bool use_i8) {
  if (use_i8 && p.i8 && b.i8ws != nullptr && b.i8ovf != nullptr)
    return launch_gram_i8(p.ip, A, nA, B, nB, b.i8ws, b.s, b.C, b.SA, b.SB, b.i8ovf, st);
  if (p.gram) return launch_gram(p.gp, A, nA, B, nB, D, b.s, b.Gpart, b.Spart, b.C, b.SA, b.SB, st);
  const size_t smem = sizeof(double) * kMC * kLds;
  auto kern = mom_ctas_per_sm() == 3 ? moments_kernel<3> : moments_kernel<4>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  MomArgs a{A, B, nA, nB, D, b.s, p.nb, p.c_diag, p.c_off, p.nslots, b.Gpart, b.Spart};
  count_launch();
  kern<<<p.nctas, kMT, smem, st>>>(a);
  count_launch();
  moments_reduce_kernel<<<148 * 2, 256, 0, st>>>(b.Gpart, b.Spart, p.nb, D, p.c_diag, p.c_off, p.nslots, b.C,
                                                 b.SA, b.SB);
  return cudaGetLastError();
}

cudaError_t launch_moments_finalize(int64_t nA, int64_t nB, int D, const MomentsBufs& b, cudaStream_t st) {
  count_launch();
  moments_finalize_kernel<<<1, 256, 0, st>>>(b.C, b.SA, b.SB, b.s, nA, nB, D, b.mu, b.u0, b.dnorm);
  count_launch();
  covariance_kernel<<<static_cast<int>((static_cast<int64_t>(D) * D + 255) / 256), 256, 0, st>>>(b.C, b.SA, b.SB,
                                                                                                 nA, nB, D);
  return cudaGetLastError();
}

cudaError_t launch_moments(const MomentsPlan& p, const float* A, int64_t nA, const float* B, int64_t nB, int D,
                           const MomentsBufs& b, cudaStream_t st) {
  cudaError_t e = launch_shift(A, nA, B, nB, D, b.s, st);
  if (e != cudaSuccess) return e;
  if ((e = launch_moments_partial(p, A, nA, B, nB, D, b, st, true)) != cudaSuccess) return e;
  return launch_moments_finalize(nA, nB, D, b, st);
}

}  // namespace prohd
