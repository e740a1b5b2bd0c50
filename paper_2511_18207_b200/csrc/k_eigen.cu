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
// One CTA of 1024 threads; the matrix lives in shared memory when it fits
// (D <= 160) and in global memory (L2-resident) otherwise. Latency-bound.
#include "internal.cuh"
#include "prohd_kernels.cuh"

#include <cfloat>

namespace prohd {
namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum; `red` has >= kWarps doubles; result broadcast to all threads
__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = (l < kWarps) ? red[l] : 0.0;
  t = warp_sum(t);
  return t;
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
  double* C;  // D x D (destroyed); used as the working matrix when it does not fit in smem
  int D;
  int k;           // requested PCs
  double* V;       // Householder vectors [D][D] (row j = v_j), workspace
  double* X;       // [k][D] eigenvectors of T, then of C (workspace)
  double* out64;   // U64 rows 1..k: [k+1][D] (row 0 = u0, untouched)
  float* out32;    // U32 rows
  double* lam;     // [k] eigenvalues (desc)
  int* n_dirs;     // 1 + kept
  int use_smem;
};

__global__ void __launch_bounds__(kThreads, 1) eigen_topk_kernel(EigArgs a) {
  extern __shared__ double sm[];
  __shared__ double red[kWarps];
  __shared__ double d[256], e[256], e2[256], lamv[256];
  __shared__ double vbuf[256], pbuf[256];
  __shared__ double u0[256], u1[256], u2[256];  // LU factors of (T - lambda I), inverse iteration
  __shared__ double s_alpha, s_scale;
  const int D = a.D;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* M = a.use_smem ? sm : a.C;
  if (a.use_smem) {
    for (int i = tid; i < D * D; i += kThreads) M[i] = a.C[i];
    __syncthreads();
  }

  // ---------------------------------------------------------------- 1. tridiagonalise
  for (int j = 0; j + 2 < D; ++j) {
    const int L = D - j - 1;  // length of the column below the diagonal
    double part = 0.0;
    for (int i = tid; i < L; i += kThreads) {
      const double x = M[(j + 1 + i) * D + j];
      vbuf[i] = x;
      part += x * x;
    }
    const double nrm2 = block_sum(part, red);
    if (tid == 0) {
      const double nrm = sqrt(nrm2);
      const double x0 = vbuf[0];
      const double alpha = (x0 > 0.0) ? -nrm : nrm;  // avoid cancellation in v0 = x0 - alpha
      s_alpha = alpha;
      const double v0 = x0 - alpha;
      // ||v||^2 = ||x||^2 - x0^2 + v0^2
      const double vn2 = nrm2 - x0 * x0 + v0 * v0;
      s_scale = (vn2 > 0.0 && nrm > 0.0) ? 1.0 / sqrt(vn2) : 0.0;
      vbuf[0] = v0;
    }
    __syncthreads();
    const double sc = s_scale;
    for (int i = tid; i < L; i += kThreads) vbuf[i] *= sc;
    for (int i = tid; i < D; i += kThreads) a.V[static_cast<int64_t>(j) * D + i] = (i > j) ? vbuf[i - j - 1] : 0.0;
    __syncthreads();
    if (tid == 0) {
      d[j] = M[j * D + j];
      e[j] = (sc != 0.0) ? s_alpha : 0.0;
    }
    if (sc == 0.0) {  // column already zero below the subdiagonal: H = I
      __syncthreads();
      continue;
    }
    // p = 2 A' v  (A' = trailing L x L block), warp per row
    for (int r = warp; r < L; r += kWarps) {
      const double* row = M + (j + 1 + r) * D + (j + 1);
      double s = 0.0;
      for (int c = lane; c < L; c += 32) s += row[c] * vbuf[c];
      s = warp_sum(s);
      if (lane == 0) pbuf[r] = 2.0 * s;
    }
    __syncthreads();
    double vp = 0.0;
    for (int i = tid; i < L; i += kThreads) vp += vbuf[i] * pbuf[i];
    const double K = block_sum(vp, red);
    for (int i = tid; i < L; i += kThreads) pbuf[i] = pbuf[i] - K * vbuf[i];  // w = p - (v^T p) v
    __syncthreads();
    // A' -= v w^T + w v^T
    for (int64_t t = tid; t < static_cast<int64_t>(L) * L; t += kThreads) {
      const int r = static_cast<int>(t / L), c = static_cast<int>(t % L);
      double* pm = M + (j + 1 + r) * D + (j + 1 + c);
      *pm = *pm - vbuf[r] * pbuf[c] - pbuf[r] * vbuf[c];
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (D >= 2) {
      d[D - 2] = M[(D - 2) * D + (D - 2)];
      e[D - 2] = M[(D - 1) * D + (D - 2)];
    }
    d[D - 1] = M[(D - 1) * D + (D - 1)];
  }
  __syncthreads();
  for (int i = tid; i < D - 1; i += kThreads) e2[i] = e[i] * e[i];
  __syncthreads();

  // ---------------------------------------------------------------- 2. eigenvalues
  // Gershgorin bounds
  double gl = 0.0, gu = 0.0, tnorm = 0.0;
  if (tid == 0) {
    gl = DBL_MAX;
    gu = -DBL_MAX;
    for (int i = 0; i < D; ++i) {
      const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < D ? fabs(e[i]) : 0.0);
      gl = fmin(gl, d[i] - r);
      gu = fmax(gu, d[i] + r);
    }
    tnorm = fmax(fabs(gl), fabs(gu));
    red[0] = gl;
    red[1] = gu;
    red[2] = tnorm;
  }
  __syncthreads();
  gl = red[0];
  gu = red[1];
  tnorm = red[2];
  __syncthreads();
  const double pivmin = fmax(DBL_MIN, 1e-300 * tnorm) + DBL_MIN;
  const int kk = a.k < D ? a.k : D;
  // eigenvalue index (ascending) D-1-w for w = 0..kk-1 -> one warp each
  for (int w = warp; w < kk; w += kWarps) {
    const int target = D - 1 - w;  // want lambda with exactly `target` eigenvalues below
    double lo = gl - 1e-12 * tnorm - pivmin, hi = gu + 1e-12 * tnorm + pivmin;
    for (int it = 0; it < 64; ++it) {
      const double width = hi - lo;
      if (width <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + 4.0 * pivmin) break;
      const double x = lo + width * (lane + 1) / 33.0;
      const int cnt = sturm_count(d, e2, D, x, pivmin);
      // predicate: count(x) <= target  (x is at or below the wanted eigenvalue)
      const unsigned below = __ballot_sync(0xffffffffu, cnt <= target);
      // probes are increasing in x; find the last probe with cnt <= target
      const int nb = __popc(below);  // probes 0..nb-1 satisfy (monotone)
      const double nlo = (nb == 0) ? lo : lo + width * nb / 33.0;
      const double nhi = (nb == 32) ? hi : lo + width * (nb + 1) / 33.0;
      lo = nlo;
      hi = nhi;
    }
    if (lane == 0) lamv[w] = 0.5 * (lo + hi);
  }
  __syncthreads();

  // ---------------------------------------------------------------- 3. inverse iteration (warp 0, serial in lane 0)
  // clusters: consecutive eigenvalues within 1e-3 * ||T|| are re-orthogonalised
  const double clus = 1e-3 * tnorm;
  if (warp == 0) {
    for (int w = 0; w < kk; ++w) {
      double* xw = a.X + static_cast<int64_t>(w) * D;
      const double lam = lamv[w];
      // initial vector: deterministic pseudo-random
      for (int i = lane; i < D; i += 32) {
        unsigned h = (unsigned)(i * 2654435761u) ^ (unsigned)(w * 40503u + 17u);
        h ^= h >> 13;
        h *= 0x5bd1e995u;
        h ^= h >> 15;
        a.X[static_cast<int64_t>(w) * D + i] = 0.5 + (h & 0xffff) / 65536.0;
      }
      __syncwarp();
      for (int iter = 0; iter < 4; ++iter) {
        if (lane == 0) {
          // solve (T - lam I) y = x by Gaussian elimination with partial pivoting (tridiagonal)
          // store factors in pbuf/vbuf-like local arrays (use e2 as scratch? no: use local)
          double* x = a.X + static_cast<int64_t>(w) * D;
          const double eps_p = DBL_EPSILON * tnorm + pivmin;
          // factor
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
          // back substitution
          x[D - 1] /= u0[D - 1];
          if (D >= 2) x[D - 2] = (x[D - 2] - u1[D - 2] * x[D - 1]) / u0[D - 2];
          for (int i = D - 3; i >= 0; --i) x[i] = (x[i] - u1[i] * x[i + 1] - u2[i] * x[i + 2]) / u0[i];
        }
        __syncwarp();
        // re-orthogonalise against previous vectors of the same cluster (MGS), then normalise
        for (int p = 0; p < w; ++p) {
          if (fabs(lamv[p] - lam) > clus) continue;
          double s = 0.0;
          for (int i = lane; i < D; i += 32) s += a.X[static_cast<int64_t>(p) * D + i] * xw[i];
          s = warp_sum(s);
          for (int i = lane; i < D; i += 32) xw[i] -= s * a.X[static_cast<int64_t>(p) * D + i];
          __syncwarp();
        }
        double s = 0.0;
        for (int i = lane; i < D; i += 32) s += xw[i] * xw[i];
        s = warp_sum(s);
        const double inv = 1.0 / sqrt(s);
        for (int i = lane; i < D; i += 32) xw[i] *= inv;
        __syncwarp();
      }
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- 4. back-transform, sign, output
  const double lam1 = kk > 0 ? lamv[0] : 0.0;
  for (int w = warp; w < kk; w += kWarps) {
    double* y = a.X + static_cast<int64_t>(w) * D;
    for (int j = D - 3; j >= 0; --j) {
      const double* v = a.V + static_cast<int64_t>(j) * D;
      double s = 0.0;
      for (int i = lane; i < D; i += 32) s += v[i] * y[i];
      s = warp_sum(s);
      for (int i = lane; i < D; i += 32) y[i] -= 2.0 * s * v[i];
      __syncwarp();
    }
    double s = 0.0;
    for (int i = lane; i < D; i += 32) s += y[i] * y[i];
    s = warp_sum(s);
    const double inv = 1.0 / sqrt(s);
    // largest |coordinate|, lowest index on ties
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
  if (tid == 0) {
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
  EigArgs a{C, D, k, V, X, out64, out32, lam, n_dirs, 0};
  size_t smem = 0;
  if (static_cast<size_t>(D) * D * sizeof(double) <= 160 * 1024) {
    a.use_smem = 1;
    smem = static_cast<size_t>(D) * D * sizeof(double);
  }
  cudaError_t e = cudaFuncSetAttribute(eigen_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  count_launch();
  eigen_topk_kernel<<<1, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace prohd
