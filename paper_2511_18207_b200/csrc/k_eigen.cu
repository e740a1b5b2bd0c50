// k_eigen.cu — K2: top-k eigenvectors of the D x D covariance on the device (fp64).
//
// PAPER.md Alg. 2 line 2 "Compute the top m principal components" and
// line 5 "u <- u/||u||". The paper obtains them by "randomized or
// truncated SVD"; here C is already formed (K1), so an exact
// symmetric eigensolver is used:
//   1. Householder tridiagonalisation  T = Q^T C Q  (Golub & Van Loan 8.3.1)
//   2. top-k eigenvalues of T by Sturm-sequence multisection (one warp per
//      eigenvalue, 32 probes per step)
//   3. eigenvectors of T by inverse iteration with re-orthogonalisation inside
//      clusters of close eigenvalues (as LAPACK's dstein)
//   4. back-transformation y = Q x, normalisation, sign rule (largest-|coord|
//      entry positive, lowest index on ties), rank drop
//      (lambda <= D 2^-52 lambda_1).
//
// Layout: ONE thread-block cluster of 8 CTAs. The matrix is kept on chip: row r
// lives in CTA r % 8 (cyclic, so every CTA keeps work as the trailing block
// shrinks), <= 32 rows x 256 fp64 = 64 KB of shared memory per CTA. Each
// Householder step needs three cluster barriers: (1) column norm partials,
// (2) the Householder vector v, (3) p = 2 A v and v^T p; the vectors are
// exchanged by direct stores into every CTA's shared memory (DSMEM).
// Latency-bound: ~3 x (D-2) cluster barriers.
#include "internal.cuh"
#include "prohd_kernels.cuh"

#include <cooperative_groups.h>

#include <cfloat>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace prohd {
namespace {

constexpr int kCl = 8;       // CTAs per cluster
constexpr int kT = 256;      // threads per CTA
constexpr int kWarps = kT / 32;
constexpr int kMaxD = 256;
constexpr int kRows = kMaxD / kCl;  // rows per CTA (max)
constexpr size_t kEigDynMax = 220 * 1024;  // tail kernel's dynamic smem budget (static use ~6.5 KB)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = (l < kWarps) ? red[l] : 0.0;
  return warp_sum(t);
}

// number of eigenvalues of T (d, e2 = e^2) strictly less than x (Sturm count)
__device__ int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  if (q < 0) ++cnt;
  for (int i = 1; i < n; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    if (q < 0) ++cnt;
  }
  return cnt;
}

struct EigArgs {
  const double* C;  // D x D symmetric (read)
  int D;
  int k;          // requested PCs
  double* V;      // Householder vectors [D][D] (row j = v_j), workspace (global)
  double* X;      // [k][D] eigenvectors of T, then of C (workspace)
  double* out64;  // U64 rows 1..k: [k+1][D] (row 0 = u0, untouched)
  float* out32;   // U32 rows
  double* lam;    // [k] eigenvalues (desc)
  int* n_dirs;    // 1 + kept
  int j0;         // Householder steps done by the cluster; the rest by CTA 0 in shared memory
  int stop;       // dev timing only (PROHD_EIG_STOP): return after phase `stop` (0 = run all)
  double* de;     // [2][kMaxD]: diagonal d, then off-diagonal e of T (global hand-off)
};

// inverse iteration for eigenvalue `lam` of T (one warp; lane 0 runs the serial solve)
__device__ void inverse_iteration(const double* d, const double* e, int D, double lam, double tnorm, double pivmin,
                                  double* x, double* u0, double* u1, double* u2, const double* X, const int* prev,
                                  int nprev, int w, int lane) {
  for (int i = lane; i < D; i += 32) {
    unsigned h = static_cast<unsigned>(i) * 2654435761u ^ (static_cast<unsigned>(w) * 40503u + 17u);
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    x[i] = 0.5 + (h & 0xffff) / 65536.0;
  }
  __syncwarp();
  const double eps_p = DBL_EPSILON * tnorm + pivmin;
  for (int iter = 0; iter < 3; ++iter) {
    if (lane == 0) {
      // (T - lam I) y = x, Gaussian elimination with partial pivoting (tridiagonal, fill u2)
      double dd = d[0] - lam, ee = (D > 1) ? e[0] : 0.0;
      for (int i = 0; i < D - 1; ++i) {
        const double sub = e[i];
        const double dn = d[i + 1] - lam;
        const double en = (i + 2 < D) ? e[i + 1] : 0.0;
        if (fabs(dd) >= fabs(sub)) {
          if (dd == 0.0) dd = eps_p;
          const double mlt = sub / dd;
          u0[i] = dd;
          u1[i] = ee;
          u2[i] = 0.0;
          x[i + 1] -= mlt * x[i];
          dd = dn - mlt * ee;
          ee = en;
        } else {
          const double mlt = dd / sub;
          u0[i] = sub;
          u1[i] = dn;
          u2[i] = en;
          const double t = x[i];
          x[i] = x[i + 1];
          x[i + 1] = t - mlt * x[i + 1];
          dd = ee - mlt * dn;
          ee = -mlt * en;
        }
      }
      if (dd == 0.0) dd = eps_p;
      u0[D - 1] = dd;
      x[D - 1] /= u0[D - 1];
      if (D >= 2) x[D - 2] = (x[D - 2] - u1[D - 2] * x[D - 1]) / u0[D - 2];
      for (int i = D - 3; i >= 0; --i) x[i] = (x[i] - u1[i] * x[i + 1] - u2[i] * x[i + 2]) / u0[i];
    }
    __syncwarp();
    // modified Gram-Schmidt against the earlier vectors of the same cluster, then normalise
    for (int q = 0; q < nprev; ++q) {
      const double* y = X + static_cast<int64_t>(prev[q]) * D;
      double s = 0.0;
      for (int i = lane; i < D; i += 32) s += y[i] * x[i];
      s = warp_sum(s);
      for (int i = lane; i < D; i += 32) x[i] -= s * y[i];
      __syncwarp();
    }
    double s = 0.0;
    for (int i = lane; i < D; i += 32) s += x[i] * x[i];
    s = warp_sum(s);
    const double inv = 1.0 / sqrt(s);
    for (int i = lane; i < D; i += 32) x[i] *= inv;
    __syncwarp();
  }
}

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kT, 1) eigen_reduce_cluster_kernel(EigArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = static_cast<int>(cl.block_rank());
  extern __shared__ double dyn[];
  double* M = dyn;  // [kRows][D] own rows (row r -> M[(r/8)*D])
  __shared__ double red[kWarps];
  __shared__ double vfull[kMaxD], pfull[kMaxD], wfull[kMaxD];
  __shared__ double part[kCl], part2[kCl];
  __shared__ double d[kMaxD], e[kMaxD];
  __shared__ double s_x0;
  const int D = a.D;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nloc = (D - rank + kCl - 1) / kCl;  // rows r = rank + 8*i, i < nloc
  for (int t = tid; t < nloc * D; t += kT) {
    const int i = t / D, c = t % D;
    M[i * D + c] = a.C[static_cast<int64_t>(rank + kCl * i) * D + c];
  }
  cl.sync();

  // ---------------------------------------------------------------- 1. tridiagonalise
  // 1a. steps j < j0 on the cluster (the trailing matrix does not fit one SM yet)
  for (int j = 0; j + 2 < D && j < a.j0; ++j) {
    // phase 1: publish d[j], x0 = M[j+1][j], and this CTA's sum of squares of column j below j
    if (tid == 0 && (j % kCl) == rank) {
      const double v = M[(j / kCl) * D + j];
      for (int q = 0; q < kCl; ++q) *cl.map_shared_rank(&d[j], q) = v;
    }
    if (tid == 0 && ((j + 1) % kCl) == rank) {
      const double v = M[((j + 1) / kCl) * D + j];
      for (int q = 0; q < kCl; ++q) *cl.map_shared_rank(&s_x0, q) = v;
    }
    double ps = 0.0;
    for (int i = tid; i < nloc; i += kT) {
      const int r = rank + kCl * i;
      if (r > j) {
        const double x = M[i * D + j];
        ps += x * x;
      }
    }
    ps = block_sum(ps, red);
    if (tid < kCl) *cl.map_shared_rank(&part[rank], tid) = ps;
    cl.sync();
    // phase 2: every CTA forms alpha and the scale redundantly; publish own entries of v
    double nrm2 = 0.0;
#pragma unroll
    for (int q = 0; q < kCl; ++q) nrm2 += part[q];
    const double nrm = sqrt(nrm2);
    const double x0 = s_x0;
    const double alpha = (x0 > 0.0) ? -nrm : nrm;
    const double v0 = x0 - alpha;
    const double vn2 = nrm2 - x0 * x0 + v0 * v0;
    const double sc = (vn2 > 0.0 && nrm > 0.0) ? 1.0 / sqrt(vn2) : 0.0;
    if (tid == 0) e[j] = (sc != 0.0) ? alpha : 0.0;
    for (int t = tid; t < nloc * kCl; t += kT) {
      const int i = t / kCl, q = t % kCl;
      const int r = rank + kCl * i;
      double v = 0.0;
      if (r > j) v = ((r == j + 1) ? v0 : M[i * D + j]) * sc;
      if (r > j) *cl.map_shared_rank(&vfull[r], q) = v;
      if (q == 0) a.V[static_cast<int64_t>(j) * D + r] = v;
    }
    cl.sync();
    if (sc == 0.0) continue;  // column already zero below the subdiagonal: H = I (uniform decision)
    // phase 3: p_r = 2 sum_c M[r][c] v_c (own rows r > j), and v^T p partial
    double vp = 0.0;
    for (int i = warp; i < nloc; i += kWarps) {
      const int r = rank + kCl * i;
      if (r <= j) continue;
      const double* row = M + i * D;
      double s = 0.0;
      for (int c = j + 1 + lane; c < D; c += 32) s += row[c] * vfull[c];
      s = 2.0 * warp_sum(s);
      if (lane < kCl) *cl.map_shared_rank(&pfull[r], lane) = s;
      vp += (lane == 0) ? s * vfull[r] : 0.0;
    }
    vp = block_sum(vp, red);
    if (tid < kCl) *cl.map_shared_rank(&part2[rank], tid) = vp;
    cl.sync();
    // phase 4: w = p - (v^T p) v, then A' -= v w^T + w v^T on own rows
    double K = 0.0;
#pragma unroll
    for (int q = 0; q < kCl; ++q) K += part2[q];
    for (int c = j + 1 + tid; c < D; c += kT) wfull[c] = pfull[c] - K * vfull[c];
    __syncthreads();
    for (int t = tid; t < nloc * (D - j - 1); t += kT) {
      const int i = t / (D - j - 1), c = j + 1 + t % (D - j - 1);
      const int r = rank + kCl * i;
      if (r <= j) continue;
      M[i * D + c] -= vfull[r] * wfull[c] + wfull[r] * vfull[c];
    }
    __syncthreads();
  }
  // hand-off of the trailing lower triangle (rows/cols >= j0) through global scratch P,
  // packed row by row: L(r, c) at po(r) + c - j0, po(r) = t (t + 1) / 2 with t = r - j0;
  // and d, e of the cluster steps
  const int j0 = a.j0;
  double* P = a.V + static_cast<int64_t>(j0) * D;
  for (int i = 0; i < nloc; ++i) {
    const int r = rank + kCl * i;
    if (r < j0) continue;
    const int t = r - j0;
    for (int c = j0 + tid; c <= r; c += kT) P[t * (t + 1) / 2 + (c - j0)] = M[i * D + c];
  }
  if (rank == 0)
    for (int j = tid; j < j0; j += kT) {
      a.de[j] = d[j];
      a.de[kMaxD + j] = e[j];
    }
}

// Steps j0 .. D-3 of the Householder tridiagonalisation on ONE CTA of 1024 threads with the
// packed trailing lower triangle in shared memory (every step needs only CTA barriers):
//   column j -> v (V row j), p = 2 M v (warp per row: lanes along the row for the stored
//   lower part, down the column for the mirrored upper part, 8 rows per warp reduced by one
//   butterfly), K = v.p, w = p - K v, L -= v w^T + w v^T (warp per row).
// j0 = 0: the triangle is read from C directly. Writes d, e (de) and V rows j0 .. D-3.
constexpr int kTT = 1024;
constexpr int kTW = kTT / 32;

__device__ __forceinline__ double block_sum_t(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = (l < kTW) ? red[l] : 0.0;
  return warp_sum(t);
}

__global__ void __launch_bounds__(kTT, 1) eigen_reduce_tail_kernel(EigArgs a) {
  extern __shared__ double L[];
  __shared__ double red[kTW];
  __shared__ double vfull[kMaxD], pfull[kMaxD], wfull[kMaxD];
  __shared__ double s_x0;
  const int D = a.D, j0 = a.j0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto po = [&](int r) { return (r - j0) * (r - j0 + 1) / 2; };
  const int nt = (D - j0) * (D - j0 + 1) / 2;
  if (j0 == 0) {
    for (int r = warp; r < D; r += kTW)
      for (int c = lane; c <= r; c += 32) L[po(r) + c] = a.C[static_cast<int64_t>(r) * D + c];
  } else {
    const double* P = a.V + static_cast<int64_t>(j0) * D;
    for (int t = tid; t < nt; t += kTT) L[t] = P[t];
  }
  __syncthreads();
  double* dg = a.de;
  double* eg = a.de + kMaxD;
  for (int j = j0; j + 2 < D; ++j) {
    const int n1 = D - j - 1;  // rows r = j+1 .. D-1
    const double x = tid < n1 ? L[po(j + 1 + tid) + (j - j0)] : 0.0;
    if (tid == 0) {
      dg[j] = L[po(j) + (j - j0)];
      s_x0 = x;
    }
    const double nrm2 = block_sum_t(x * x, red);
    const double nrm = sqrt(nrm2);
    const double x0 = s_x0;
    const double alpha = (x0 > 0.0) ? -nrm : nrm;
    const double v0 = x0 - alpha;
    const double vn2 = nrm2 - x0 * x0 + v0 * v0;
    const double sc = (vn2 > 0.0 && nrm > 0.0) ? 1.0 / sqrt(vn2) : 0.0;
    if (tid == 0) eg[j] = (sc != 0.0) ? alpha : 0.0;
    if (tid < n1) {
      const double v = ((tid == 0) ? v0 : x) * sc;
      vfull[j + 1 + tid] = v;
      a.V[static_cast<int64_t>(j) * D + j + 1 + tid] = v;
    }
    __syncthreads();
    if (sc == 0.0) continue;  // uniform
    // p = 2 M v: warp w owns rows r_i = j+1+w+32 i (i < 8)
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      acc[i] = 0.0;
      const int r = j + 1 + warp + kTW * i;
      if (r < D) {
        const double* row = L + po(r) - j0;
        double s = 0.0;
        for (int c = j + 1 + lane; c <= r; c += 32) s = fma(row[c], vfull[c], s);
        for (int c = r + 1 + lane; c < D; c += 32) s = fma(L[po(c) + (r - j0)], vfull[c], s);
        acc[i] = s;
      }
    }
    // butterfly reduce-scatter of the 8 row sums: lane l ends with row i = (l >> 2) & 7
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool up = (lane & 16) != 0;
      const double send = up ? acc[i] : acc[i + 4];
      const double keep = up ? acc[i + 4] : acc[i];
      acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const bool up = (lane & 8) != 0;
      const double send = up ? acc[i] : acc[i + 2];
      const double keep = up ? acc[i + 2] : acc[i];
      acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    {
      const bool up = (lane & 4) != 0;
      const double send = up ? acc[0] : acc[1];
      const double keep = up ? acc[1] : acc[0];
      acc[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 2);
    acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
    double vp = 0.0;
    {
      const int ri = (lane >> 2) & 7;
      const int r = j + 1 + warp + kTW * ri;
      if ((lane & 3) == 0 && r < D) {
        const double pr = 2.0 * acc[0];
        pfull[r] = pr;
        vp = pr * vfull[r];
      }
    }
    const double K = block_sum_t(vp, red);
    if (tid < n1) wfull[j + 1 + tid] = pfull[j + 1 + tid] - K * vfull[j + 1 + tid];
    __syncthreads();
    for (int r = j + 1 + warp; r < D; r += kTW) {
      double* row = L + po(r) - j0;
      const double vr = vfull[r], wr = wfull[r];
      for (int c = j + 1 + lane; c <= r; c += 32) row[c] -= vr * wfull[c] + wr * vfull[c];
    }
    __syncthreads();
  }
  if (tid == 0) {
    const int jl = D >= 2 ? D - 2 : 0;
    if (D >= 2 && jl >= j0) dg[D - 2] = L[po(D - 2) + (D - 2 - j0)];
    dg[D - 1] = L[po(D - 1) + (D - 1 - j0)];
    if (D >= 2) eg[D - 2] = L[po(D - 1) + (D - 2 - j0)];
  }
}

// Eigenvalues (bisection), eigenvectors of T (inverse iteration) and the back-transform,
// on the cluster, from d, e (de) and the Householder vectors (V).
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kT, 1) eigen_vectors_cluster_kernel(EigArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = static_cast<int>(cl.block_rank());
  extern __shared__ double dyn[];
  double* lu = dyn;  // [kWarps][3][kMaxD] LU scratch
  __shared__ double d[kMaxD], e[kMaxD], e2[kMaxD], lamv[kMaxD];
  __shared__ int s_prev[kWarps][16];
  const int D = a.D;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < D; i += kT) {
    d[i] = a.de[i];
    e[i] = i < D - 1 ? a.de[kMaxD + i] : 0.0;
  }
  __syncthreads();
  if (a.stop == 1) return;
  for (int i = tid; i < D - 1; i += kT) e2[i] = e[i] * e[i];
  __syncthreads();
  // ---------------------------------------------------------------- 2. eigenvalues (every CTA, redundantly)
  double gl = DBL_MAX, gu = -DBL_MAX;
  for (int i = 0; i < D; ++i) {
    const double rr = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < D ? fabs(e[i]) : 0.0);
    gl = fmin(gl, d[i] - rr);
    gu = fmax(gu, d[i] + rr);
  }
  const double tnorm = fmax(fabs(gl), fabs(gu));
  const double pivmin = fmax(DBL_MIN, 1e-300 * tnorm) + DBL_MIN;
  const int kk = a.k < D ? a.k : D;
  // one warp per eigenvalue across the whole cluster (warp slot rank * kWarps + warp)
  for (int w = rank * kWarps + warp; w < kk; w += kCl * kWarps) {
    const int target = D - 1 - w;  // the eigenvalue with exactly `target` eigenvalues below it
    double lo = gl - 1e-12 * tnorm - pivmin, hi = gu + 1e-12 * tnorm + pivmin;
    for (int it = 0; it < 64; ++it) {
      const double width = hi - lo;
      if (width <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + 4.0 * pivmin) break;
      const double x = lo + width * (lane + 1) / 33.0;
      const int cnt = sturm_count(d, e2, D, x, pivmin);
      const unsigned below = __ballot_sync(0xffffffffu, cnt <= target);
      const int nb = __popc(below);  // monotone: probes 0..nb-1 are at or below the eigenvalue
      const double nlo = (nb == 0) ? lo : lo + width * nb / 33.0;
      const double nhi = (nb == 32) ? hi : lo + width * (nb + 1) / 33.0;
      lo = nlo;
      hi = nhi;
    }
    if (lane < kCl) *cl.map_shared_rank(&lamv[w], lane) = 0.5 * (lo + hi);
  }
  cl.sync();
  if (a.stop == 2) return;

  // ---------------------------------------------------------------- 3. inverse iteration
  // Consecutive eigenvalues closer than 1e-6 ||T|| form a cluster, handled by one warp in
  // order with re-orthogonalisation (as LAPACK's dstein); every other eigenvector comes from
  // an independent inverse iteration on its own warp, whose error eps ||T|| / gap stays
  // below ~1e-10 at that gap (dstein's 1e-3 ||T|| would serialise spectra such as cfg4's,
  // top-16 relative gaps ~1e-4, onto a single warp).
  const double clus = 1e-6 * tnorm;
  {
    int c = 0;  // cluster index
    int start = 0;
    while (start < kk) {
      int end = start + 1;
      while (end < kk && fabs(lamv[end - 1] - lamv[end]) <= clus) ++end;
      const int slot = c % (kCl * kWarps);
      if (slot / kWarps == rank && slot % kWarps == warp) {
        double* u0 = lu + warp * 3 * kMaxD;
        int nprev = 0;
        for (int w = start; w < end; ++w) {
          inverse_iteration(d, e, D, lamv[w], tnorm, pivmin, a.X + static_cast<int64_t>(w) * D, u0, u0 + kMaxD,
                            u0 + 2 * kMaxD, a.X, s_prev[warp], nprev, w, lane);
          if (lane == 0 && nprev < 16) s_prev[warp][nprev] = w;
          __syncwarp();
          if (nprev < 16) ++nprev;
        }
      }
      ++c;
      start = end;
    }
  }
  cl.sync();  // eigenvectors of T (global memory) visible to the whole cluster
  if (a.stop == 3) return;

  // ---------------------------------------------------------------- 4. back-transform, sign, output
  for (int w = rank * kWarps + warp; w < kk; w += kCl * kWarps) {
    double* y = a.X + static_cast<int64_t>(w) * D;
    for (int j = D - 3; j >= 0; --j) {
      const double* v = a.V + static_cast<int64_t>(j) * D;
      double s = 0.0;
      for (int i = j + 1 + lane; i < D; i += 32) s += v[i] * y[i];
      s = warp_sum(s);
      for (int i = j + 1 + lane; i < D; i += 32) y[i] -= 2.0 * s * v[i];
      __syncwarp();
    }
    double s = 0.0;
    for (int i = lane; i < D; i += 32) s += y[i] * y[i];
    s = warp_sum(s);
    const double inv = 1.0 / sqrt(s);
    double best = -1.0;
    int bidx = D;
    for (int i = lane; i < D; i += 32) {
      const double v = fabs(y[i]);
      if (v > best) {
        best = v;
        bidx = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ob > best || (ob == best && oi < bidx)) {
        best = ob;
        bidx = oi;
      }
    }
    const double sgn = (y[bidx] < 0.0) ? -inv : inv;
    for (int i = lane; i < D; i += 32) {
      const double v = y[i] * sgn;
      a.out64[static_cast<int64_t>(w + 1) * D + i] = v;
      a.out32[static_cast<int64_t>(w + 1) * D + i] = static_cast<float>(v);
    }
    if (lane == 0) a.lam[w] = lamv[w];
  }
  if (rank == 0 && tid == 0) {
    const double lam1 = kk > 0 ? lamv[0] : 0.0;
    int kept = 0;
    if (lam1 > 0.0) {
      for (int w = 0; w < kk; ++w) {
        if (lamv[w] <= D * 0x1p-52 * lam1) break;
        ++kept;
      }
    }
    *a.n_dirs = 1 + kept;
  }
}

}  // namespace

cudaError_t launch_eigen_topk(double* C, int D, int k, double* V, double* X, double* out64, float* out32,
                              double* lam, int* n_dirs, cudaStream_t st) {
  if (D > kMaxD) return cudaErrorInvalidValue;
  // cluster steps until the packed trailing triangle fits the tail kernel's shared memory
  int npk = D;
  while (npk > 2 && sizeof(double) * static_cast<size_t>(npk) * (npk + 1) / 2 > kEigDynMax) --npk;
  const int j0 = D - npk;
  const size_t packed = sizeof(double) * static_cast<size_t>(npk) * (npk + 1) / 2;
  const char* es = getenv("PROHD_EIG_STOP");
  EigArgs a{C, D, k, V, X, out64, out32, lam, n_dirs, j0, es != nullptr ? atoi(es) : 0,
            V + static_cast<int64_t>(D) * D};
  cudaError_t e;
  if (j0 > 0) {
    const size_t smem = sizeof(double) * static_cast<size_t>(kRows) * kMaxD;
    if ((e = cudaFuncSetAttribute(eigen_reduce_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem))) != cudaSuccess)
      return e;
    count_launch();
    eigen_reduce_cluster_kernel<<<kCl, kT, smem, st>>>(a);
  }
  if ((e = cudaFuncSetAttribute(eigen_reduce_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(packed))) != cudaSuccess)
    return e;
  count_launch();
  eigen_reduce_tail_kernel<<<1, kTT, packed, st>>>(a);
  const size_t smem3 = sizeof(double) * static_cast<size_t>(kWarps) * 3 * kMaxD;
  if ((e = cudaFuncSetAttribute(eigen_vectors_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem3))) != cudaSuccess)
    return e;
  count_launch();
  eigen_vectors_cluster_kernel<<<kCl, kT, smem3, st>>>(a);
  return cudaGetLastError();
}

}  // namespace prohd
