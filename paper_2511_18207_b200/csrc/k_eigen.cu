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
// Layout: ONE thread-block cluster of 8 (16 for D > 160) CTAs. The matrix is kept on chip:
// row r lives in CTA r % kCl (cyclic, so every CTA keeps work as the trailing block shrinks),
// <= 32 rows x 256 fp64 = 64 KB of shared memory per CTA (the D <= 512 variant: 16 CTAs x 32
// rows x 512 = 128 KB). Each Householder step exchanges p = 2 A v and the pre-update next column
// by direct stores into every CTA's shared memory (DSMEM) and needs ONE cluster barrier; every
// warp keeps the current column in registers and forms v and the updated next column itself.
// Latency-bound: ~(D-2) cluster barriers.
#include "internal.cuh"
#include "prohd_kernels.cuh"
#include "sm100.cuh"

#include <cooperative_groups.h>

#include <cfloat>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace prohd {
namespace {

constexpr int kCl = 8;       // CTAs per cluster
constexpr int kT = 256;      // threads per CTA
constexpr int kWarps = kT / 32;
constexpr int kMaxD = 256;     // the default variant's largest D; D <= 512 takes the MD = 512 variant
constexpr int kDeStride = 512;  // de = [d (512) | e (512)] for both variants
template <int MD>
constexpr int lu_stride() { return 6 * MD + MD / 8; }  // doubles of inverse-iteration scratch per warp

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 1/q for |q| >= DBL_MIN (normal): hardware approximation + 2 Newton steps (<= 1 ulp), a
// quarter of the latency of the IEEE division sequence on the serial chains below
__device__ __forceinline__ double rcp_normal(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  double e = fma(-q, r, 1.0);
  r = fma(r, e, r);
  e = fma(-q, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rcp_safe(double q) { return fabs(q) >= 0x1p-1000 ? rcp_normal(q) : 1.0 / q; }
// 1/sqrt(x) for normal x > 0: hardware approximation + 2 Newton steps (~1 ulp); off the IEEE sqrt
// and division sequences on the Householder step's serial chain. Tiny / zero x: the IEEE path.
__device__ __forceinline__ double rsqrt_nr(double x) {
  if (!(x >= 0x1p-1000)) return 1.0 / sqrt(x);
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double h = 0.5 * x;
  r = r * fma(-h * r, r, 1.5);
  r = r * fma(-h * r, r, 1.5);
  return r;
}

// 1/q for the Sturm count: hardware approximation + ONE Newton step (relative error ~2^-44: the
// count is that of T with the e2 perturbed by ~2^-44 relative, well inside what bisection to
// 2 eps needs; the q-form recurrence stays backward stable)
__device__ __forceinline__ double rcp_sturm(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  return fma(r, fma(-q, r, 1.0), r);
}
// Remote shared-memory stores that complete on the DESTINATION CTA's mbarrier (st.async, the
// async proxy): the receiver waits on its own barrier for the bytes, no release fence, no cluster
// barrier. Both addresses are shared::cluster addresses (mapa).
__device__ __forceinline__ void st_async_f64x2(uint32_t dst, double a0, double a1, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(dst),
               "d"(a0), "d"(a1), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void st_async_b64(uint32_t dst, unsigned long long v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(dst), "l"(v),
               "r"(mbar)
               : "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// acquire (cluster scope) wait on a local mbarrier fed by remote st.async; ~1 s watchdog
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  const long long t0 = clock64();
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(sm100::smem_u32(bar)), "r"(parity)
        : "memory");
    if (!ok && clock64() - t0 > 2000000000ll) __trap();
  } while (!ok);
}

// number of eigenvalues of T (d, e2 = e^2) strictly less than x (Sturm count); |q| >= pivmin
// (> DBL_MIN) at every division, so the reciprocal is taken on normal numbers
__device__ int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  if (q < 0) ++cnt;
  for (int i = 1; i < n; ++i) {
    q = d[i] - x - e2[i - 1] * rcp_sturm(q);
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
  int stop;       // dev timing only (option eig_stop): return after phase `stop` (0 = run all)
  double* de;     // [2][kDeStride]: diagonal d, then off-diagonal e of T (global hand-off)
};

// inverse iteration for eigenvalue `lam` of T (one warp; lane 0 runs the serial solve on the
// warp's shared-memory vector x; the result is copied to xout)
__device__ void inverse_iteration(const double* d, const double* e, int D, double lam, double tnorm, double pivmin,
                                  double* xout, double* x, double* u0, double* u1, double* u2, double* mlt,
                                  double* inv0, unsigned char* piv, const double* X, const int* prev, int nprev,
                                  int w, int lane) {
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
      // (T - lam I) y = x by Gaussian elimination with partial pivoting (tridiagonal, fill u2);
      // the factorisation (multipliers, row swaps, reciprocal pivots) is formed in the first
      // iteration and reused by the next two, which only run the substitutions
      if (iter == 0) {
        double dd = d[0] - lam, ee = (D > 1) ? e[0] : 0.0;
        for (int i = 0; i < D - 1; ++i) {
          const double sub = e[i];
          const double dn = d[i + 1] - lam;
          const double en = (i + 2 < D) ? e[i + 1] : 0.0;
          if (fabs(dd) >= fabs(sub)) {
            if (dd == 0.0) dd = eps_p;
            const double rd = rcp_safe(dd);
            const double m = sub * rd;
            u0[i] = dd;
            inv0[i] = rd;
            u1[i] = ee;
            u2[i] = 0.0;
            mlt[i] = m;
            piv[i] = 0;
            dd = dn - m * ee;
            ee = en;
          } else {
            const double m = dd * rcp_safe(sub);
            u0[i] = sub;
            inv0[i] = rcp_safe(sub);
            u1[i] = dn;
            u2[i] = en;
            mlt[i] = m;
            piv[i] = 1;
            dd = ee - m * dn;
            ee = -m * en;
          }
        }
        if (dd == 0.0) dd = eps_p;
        u0[D - 1] = dd;
        inv0[D - 1] = rcp_safe(dd);
      }
      // forward: the row operations of the elimination on the right-hand side
      double xn = x[0];
      for (int i = 0; i < D - 1; ++i) {
        const double xi1 = x[i + 1];
        if (piv[i] == 0) {
          x[i] = xn;
          xn = xi1 - mlt[i] * xn;
        } else {
          x[i] = xi1;
          xn = xn - mlt[i] * xi1;
        }
      }
      x[D - 1] = xn;
      // back substitution with the reciprocal pivots
      x[D - 1] *= inv0[D - 1];
      if (D >= 2) x[D - 2] = (x[D - 2] - u1[D - 2] * x[D - 1]) * inv0[D - 2];
      double x1 = D >= 2 ? x[D - 2] : 0.0, x2 = x[D - 1];  // x[i + 1], x[i + 2] in registers
      for (int i = D - 3; i >= 0; --i) {
        const double xi = (x[i] - u1[i] * x1 - u2[i] * x2) * inv0[i];
        x[i] = xi;
        x2 = x1;
        x1 = xi;
      }
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
  for (int i = lane; i < D; i += 32) xout[i] = x[i];
  __syncwarp();
}

// Householder tridiagonalisation T = Q^T C Q on one cluster of kCl CTAs (Golub & Van Loan
// 8.3.1). Row r of C lives in CTA r % kCl as a full row in shared memory. Column j of the
// current matrix is held in REGISTERS by every warp (lane l: rows l + 32 t), so a step needs no
// CTA barrier, and ONE cluster barrier (pc double-buffered on j & 1):
//   B. each warp forms the norm, alpha and v = (x - alpha e1)/||.|| from its copy of column j,
//      computes p_r = 2 sum_c M[r][c] v_c for its own rows r > j and scatters (p_r, the
//      PRE-update entry M[r][j+1]) as one 16-byte store into every CTA.  -> cluster barrier
//   C. K = v.p (from the full p), w = p - K v, M[r][c] -= v_r w_c + w_r v_c on own rows (v_r from
//      the row's own entry M[r][j]), and every warp forms the updated column j+1 in its registers
//      with the owner's expression M[r][j+1] - (v_r w_{j+1} + w_r v_{j+1}) (bit-identical).
// Writes d, e (de) and the Householder vectors (V rows 0 .. D-3).
template <int kCl, int MD>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kT, 1) eigen_reduce_cluster_kernel(EigArgs a) {
  constexpr int kRows = MD / kCl;  // rows per CTA (max)
    cg::cluster_group cl = cg::this_cluster();
  const int rank = static_cast<int>(cl.block_rank());
  extern __shared__ double dyn[];
  double* M = dyn;  // [kRows][D] own rows (row r -> M[(r/kCl)*D])
  __shared__ double2 pc2[2][MD];  // scattered (p_r, pre-update M[r][j+1]): [j & 1]
  __shared__ __align__(8) uint64_t pbar[2];          // complete_tx barriers of pc2[0], pc2[1]
  __shared__ unsigned long long tok[kWarps];          // per-step tokens of every warp of every CTA
  const int D = a.D;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nloc = (D - rank + kCl - 1) / kCl;  // rows r = rank + kCl*i, i < nloc
  for (int t = tid; t < nloc * D; t += kT) {
    const int i = t / D, c = t % D;
    M[i * D + c] = a.C[static_cast<int64_t>(rank + kCl * i) * D + c];
  }
  // column j of the current matrix, in registers and replicated in every warp: lane l holds rows
  // c = l + 32 t (t < 8). Column 0 is read from the ROWS (C[c][0]), the entries the row owners
  // hold: the register column and the owners' rows must agree bit for bit (the update uses v_r
  // from the row and v_c from the column; with C[0][c] instead, a 1-ulp asymmetry of the input
  // grew into O(||C||) errors of T, reproduced in a host emulation)
  constexpr int kTq = MD / 32;
  double x[kTq];
#pragma unroll
  for (int t = 0; t < kTq; ++t) {
    const int c = lane + 32 * t;
    x[t] = c < D ? a.C[static_cast<int64_t>(c) * D] : 0.0;
  }
  if (tid == 0) {
    sm100::mbar_init(&pbar[0], 1);
    sm100::mbar_init(&pbar[1], 1);
    sm100::fence_mbar_init();
  }
  __syncthreads();
  cl.sync();
  const uint32_t pbar_u32 = sm100::smem_u32(&pbar[0]), pc_u32 = sm100::smem_u32(&pc2[0][0]);
  const uint32_t tok_u32 = sm100::smem_u32(&tok[warp]);
  double* dg = a.de;
  double* eg = a.de + kDeStride;
  constexpr int kRW = kRows / kWarps;  // own rows per warp
  for (int j = 0; j + 2 < D; ++j) {
    double2* pc = pc2[j & 1];
    // B. every warp forms ||x||, alpha and the scale from its register copy of column j (rows
    // > j); v_c = (c == j+1 ? x0 - alpha : x_c) * sc
    double ss = 0.0, x0 = 0.0;
#pragma unroll
    for (int t = 0; t < kTq; ++t) {
      const int c = lane + 32 * t;
      const double xt = (c > j && c < D) ? x[t] : 0.0;
      ss = fma(xt, xt, ss);
      x0 = (c == j + 1) ? xt : x0;
    }
    const double nrm2 = warp_sum(ss);
    const double nrm = nrm2 > 0.0 ? nrm2 * rsqrt_nr(nrm2) : 0.0;
    x0 = __shfl_sync(0xffffffffu, x0, (j + 1) & 31);
    const double alpha = (x0 > 0.0) ? -nrm : nrm;
    const double v0 = x0 - alpha;
    const double vn2 = nrm2 - x0 * x0 + v0 * v0;
    // sc == 0: the column is already zero below the subdiagonal, H = I (v = 0, p = 0, K = 0:
    // the update below is then a no-op and the next column comes out unchanged)
    const double sc = (vn2 > 0.0 && nrm > 0.0) ? rsqrt_nr(vn2) : 0.0;
    double v[kTq];
#pragma unroll
    for (int t = 0; t < kTq; ++t) {
      const int c = lane + 32 * t;
      v[t] = (c > j && c < D) ? (c == j + 1 ? v0 : x[t]) * sc : 0.0;
    }
    // p_r = 2 M[r][j+1:] . v for own rows r > j (warp per row, the row dot products formed
    // together and reduced together)
    double ps[kRW];
#pragma unroll
    for (int q = 0; q < kRW; ++q) {
      const int i = warp + kWarps * q;
      const int r = rank + kCl * i;
      double s0 = 0.0;
      if (i < nloc && r > j) {
        const double* row = M + i * D;
#pragma unroll
        for (int t = 0; t < kTq; ++t) {
          const int c = lane + 32 * t;
          if (c > j && c < D) s0 = fma(row[c], v[t], s0);
        }
      }
      ps[q] = s0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int q = 0; q < kRW; ++q) ps[q] += __shfl_xor_sync(0xffffffffu, ps[q], o);
    // the exchange: one 16-byte st.async per row and target CTA, completing on the target's
    // barrier of this buffer, plus one 8-byte token per warp and target (so a step's barrier
    // completes only when EVERY warp of every CTA has finished the previous step, which makes the
    // double buffer safe without a cluster barrier). Expected per CTA and step: 16 (D - j - 1)
    // data bytes + 8 kCl kWarps token bytes.
    const int b = j & 1;
    if (tid == 0)
      sm100::mbar_arrive_expect_tx(&pbar[b], static_cast<uint32_t>(16 * (D - j - 1) + 8 * kCl * kWarps));
    const uint32_t rbar = mapa_u32(pbar_u32 + 8u * static_cast<uint32_t>(b), static_cast<uint32_t>(lane));
#pragma unroll
    for (int q = 0; q < kRW; ++q) {
      const int i = warp + kWarps * q;
      const int r = rank + kCl * i;
      if (i < nloc && r > j && lane < kCl)
        st_async_f64x2(mapa_u32(pc_u32 + 16u * static_cast<uint32_t>(b * MD + r), static_cast<uint32_t>(lane)),
                       2.0 * ps[q], M[i * D + j + 1], rbar);
    }
    if (lane < kCl) st_async_b64(mapa_u32(tok_u32, static_cast<uint32_t>(lane)), 0ull, rbar);
    // this step's global outputs (d_j, e_j, Householder vector j) while the exchange is in flight
    // d_j from the warp that owns (and last updated) row j: no cross-warp shared-memory hazard
    if (j % kCl == rank && warp == (j / kCl) % kWarps && lane == 0) dg[j] = M[(j / kCl) * D + j];
    if (rank == 0 && warp == 0) {
      if (lane == 0) eg[j] = (sc != 0.0) ? alpha : 0.0;
#pragma unroll
      for (int t = 0; t < kTq; ++t) {
        const int c = lane + 32 * t;
        if (c > j && c < D) a.V[static_cast<int64_t>(j) * D + c] = v[t];
      }
    }
    mbar_wait_acq_cluster(&pbar[b], static_cast<uint32_t>(j >> 1) & 1u);
    // C. K = v.p from the full p (same order in every warp and CTA), w = p - K v; M[r][c] -=
    // v_r w_c + w_r v_c on own rows; every warp forms the updated column j+1 (rows > j) in its
    // registers with the owner's expression, M[r][j+1] - (v_r w_{j+1} + w_r v_{j+1})
    double K = 0.0;
#pragma unroll
    for (int t = 0; t < kTq; ++t) {
      const int c = lane + 32 * t;
      if (c > j && c < D) K = fma(v[t], pc[c].x, K);
    }
    K = warp_sum(K);
    double w[kTq];
#pragma unroll
    for (int t = 0; t < kTq; ++t) {
      const int c = lane + 32 * t;
      w[t] = (c > j && c < D) ? pc[c].x - K * v[t] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kRW; ++q) {
      const int i = warp + kWarps * q;
      const int r = rank + kCl * i;
      if (i >= nloc || r <= j) continue;
      double* row = M + i * D;
      const double vr = (r == j + 1 ? v0 : row[j]) * sc;  // v_r from the row's own column-j entry
      const double wr = pc[r].x - K * vr;
#pragma unroll
      for (int t = 0; t < kTq; ++t) {
        const int c = lane + 32 * t;
        if (c > j && c < D) row[c] -= fma(vr, w[t], wr * v[t]);
      }
    }
    {
      const double vj = v0 * sc, wj = pc[j + 1].x - K * vj;
#pragma unroll
      for (int t = 0; t < kTq; ++t) {
        const int c = lane + 32 * t;
        x[t] = (c > j && c < D) ? pc[c].y - fma(v[t], wj, w[t] * vj) : 0.0;
      }
    }
  }
  cl.sync();  // every CTA's last exchange has landed before any CTA exits
  __syncthreads();  // the last step's row updates (other warps) before the 2x2 block
  // last 2x2 block
  if (D >= 2 && ((D - 2) % kCl) == rank && tid == 0) {
    const int i = (D - 2) / kCl;
    dg[D - 2] = M[i * D + (D - 2)];
  }
  if (((D - 1) % kCl) == rank && tid == 0) {
    const int i = (D - 1) / kCl;
    dg[D - 1] = M[i * D + (D - 1)];
    if (D >= 2) eg[D - 2] = M[i * D + (D - 2)];
  }
}

// Eigenvalues (bisection), eigenvectors of T (inverse iteration) and the back-transform,
// on the cluster, from d, e (de) and the Householder vectors (V).
template <int MD>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kT, 1) eigen_vectors_cluster_kernel(EigArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = static_cast<int>(cl.block_rank());
  extern __shared__ double dyn[];
  double* lu = dyn;  // per warp: u0, u1, u2, x, multipliers, 1/u0 (MD doubles each), swap flags
  __shared__ double d[MD], e[MD], e2[MD], lamv[MD];
  __shared__ int s_prev[kWarps][16];
  const int D = a.D;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < D; i += kT) {
    d[i] = a.de[i];
    e[i] = i < D - 1 ? a.de[kDeStride + i] : 0.0;
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
  // G warps per eigenvalue (32 G probes per multisection step; G = 4 for k <= 16 spreads the
  // 8 x 8 warps of the cluster over the eigenvalues), the G warps of a group in one CTA
  const int G = kk <= (kCl * kWarps) / 4 ? 4 : kk <= (kCl * kWarps) / 2 ? 2 : 1;
  const int gpc = kWarps / G;                 // groups per CTA
  const int grp = warp / G, gj = warp % G;    // group in this CTA, warp within the group
  const int P = 32 * G;                       // probes per step
  __shared__ int gnb[2][kWarps];              // per-step probe counts, double-buffered
  for (int base = 0; base < kk; base += kCl * gpc) {
    // every group runs the same number of outer iterations (named barriers inside)
    const int w = base + rank * gpc + grp;
    const bool live = w < kk;
    const int target = D - 1 - (live ? w : 0);  // the eigenvalue with exactly `target` eigenvalues below it
    double lo = gl - 1e-12 * tnorm - pivmin, hi = gu + 1e-12 * tnorm + pivmin;
    for (int it = 0; it < 64; ++it) {
      const double width = hi - lo;
      if (width <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + 4.0 * pivmin) break;  // uniform per group
      const double x = lo + width * (gj * 32 + lane + 1) / static_cast<double>(P + 1);
      const int cnt = sturm_count(d, e2, D, x, pivmin);
      const unsigned below = __ballot_sync(0xffffffffu, cnt <= target);
      if (G > 1) {
        if (lane == 0) gnb[it & 1][warp] = __popc(below);
        asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * G) : "memory");
      }
      int nb = __popc(below);  // monotone: probes 0..nb-1 are at or below the eigenvalue
      if (G > 1) {
        nb = 0;
        for (int q = 0; q < G; ++q) nb += gnb[it & 1][grp * G + q];
      }
      const double nlo = (nb == 0) ? lo : lo + width * nb / static_cast<double>(P + 1);
      const double nhi = (nb == P) ? hi : lo + width * (nb + 1) / static_cast<double>(P + 1);
      lo = nlo;
      hi = nhi;
    }
    if (live && gj == 0 && lane < kCl) *cl.map_shared_rank(&lamv[w], lane) = 0.5 * (lo + hi);
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
        double* u0 = lu + warp * lu_stride<MD>();
        int nprev = 0;
        for (int w = start; w < end; ++w) {
          inverse_iteration(d, e, D, lamv[w], tnorm, pivmin, a.X + static_cast<int64_t>(w) * D, u0 + 3 * MD, u0,
                            u0 + MD, u0 + 2 * MD, u0 + 4 * MD, u0 + 5 * MD,
                            reinterpret_cast<unsigned char*>(u0 + 6 * MD), a.X, s_prev[warp], nprev, w, lane);
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
    // y <- H_0 H_1 ... H_{D-3} y with y in registers (lane holds y[lane + 32 t]), H_j = I - 2 v_j v_j^T.
    // Reflectors are applied in PAIRS with one warp reduction: a = v_j.y, b = v_{j-1}.y and
    // c = v_{j-1}.v_j reduced together, then y -= 2 a v_j and y -= 2 (b - 2 a c) v_{j-1}
    // (= v_{j-1}.(H_j y)); the rows of the next two pairs are prefetched into registers, so the
    // global-memory latency of V is not on the chain.
    constexpr int kYT = MD / 32;
    double yr[kYT];
    double p0[kYT], p1[kYT], q0[kYT], q1[kYT], r0[kYT], r1[kYT];
    auto ldrow = [&](int j, double(&r)[kYT]) {
#pragma unroll
      for (int t = 0; t < kYT; ++t) {
        const int i = lane + 32 * t;
        r[t] = (j >= 0 && i > j && i < D) ? a.V[static_cast<int64_t>(j) * D + i] : 0.0;  // v_j[i], i > j
      }
    };
#pragma unroll
    for (int t = 0; t < kYT; ++t) {
      const int i = lane + 32 * t;
      yr[t] = i < D ? y[i] : 0.0;
    }
    const int J = D - 3;
    ldrow(J, p0);
    ldrow(J - 1, p1);
    ldrow(J - 2, q0);
    ldrow(J - 3, q1);
    for (int j = J; j >= 0; j -= 2) {
      ldrow(j - 4, r0);
      ldrow(j - 5, r1);
      double sa = 0.0, sb = 0.0, scc = 0.0;
#pragma unroll
      for (int t = 0; t < kYT; ++t) {
        sa = fma(p0[t], yr[t], sa);
        sb = fma(p1[t], yr[t], sb);
        scc = fma(p1[t], p0[t], scc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
        scc += __shfl_xor_sync(0xffffffffu, scc, o);
      }
      const double s2 = sb - 2.0 * sa * scc;
#pragma unroll
      for (int t = 0; t < kYT; ++t) {
        yr[t] = fma(-2.0 * sa, p0[t], yr[t]);
        yr[t] = fma(-2.0 * s2, p1[t], yr[t]);
        p0[t] = q0[t];
        p1[t] = q1[t];
        q0[t] = r0[t];
        q1[t] = r1[t];
      }
    }
#pragma unroll
    for (int t = 0; t < kYT; ++t) {
      const int i = lane + 32 * t;
      if (i < D) y[i] = yr[t];
    }
    __syncwarp();
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
  if (D > 2 * kMaxD) return cudaErrorInvalidValue;
  const int stop = opt(OPT_EIG_STOP) > 0 ? static_cast<int>(opt(OPT_EIG_STOP)) : 0;
  EigArgs a{C, D, k, V, X, out64, out32, lam, n_dirs, stop, V + static_cast<int64_t>(D) * D};
  cudaError_t e;
  if (D > kMaxD) {
    // 256 < D <= 512 (no BASELINE config): the same kernels instantiated for 512, the
    // tridiagonalisation on a 16-CTA cluster (32 rows x 512 fp64 = 128 KB per CTA)
    const size_t smem = sizeof(double) * static_cast<size_t>(512 / 16) * 512;
    if ((e = cudaFuncSetAttribute(eigen_reduce_cluster_kernel<16, 512>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                  1)) != cudaSuccess ||
        (e = cudaFuncSetAttribute(eigen_reduce_cluster_kernel<16, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem))) != cudaSuccess)
      return e;
    count_launch();
    eigen_reduce_cluster_kernel<16, 512><<<16, kT, smem, st>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const size_t smem3 = sizeof(double) * static_cast<size_t>(kWarps) * lu_stride<512>();
    if ((e = cudaFuncSetAttribute(eigen_vectors_cluster_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem3))) != cudaSuccess)
      return e;
    count_launch();
    eigen_vectors_cluster_kernel<512><<<kCl, kT, smem3, st>>>(a);
    return cudaGetLastError();
  }
  // tridiagonalisation on a 16-CTA cluster (non-portable size) where the device allows it, else on
  // 8 CTAs; with the st.async exchange 16 CTAs win at every D (D = 256: 0.455 vs 0.513 ms, D = 128:
  // 0.208 vs 0.221, D = 64: 0.102 vs 0.104); option eig_cl = 8 forces the portable size (A/B)
  bool wide = opt(OPT_EIG_CL) != 8;
  if (wide) {
    const size_t smem16 = sizeof(double) * static_cast<size_t>(kMaxD / 16) * kMaxD;
    wide = cudaFuncSetAttribute(eigen_reduce_cluster_kernel<16, kMaxD>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                1) == cudaSuccess &&
           cudaFuncSetAttribute(eigen_reduce_cluster_kernel<16, kMaxD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem16)) == cudaSuccess;
    if (wide) {
      count_launch();
      eigen_reduce_cluster_kernel<16, kMaxD><<<16, kT, smem16, st>>>(a);
      wide = cudaPeekAtLastError() == cudaSuccess;
      if (!wide) (void)cudaGetLastError();  // clear a launch refusal; fall back to 8 CTAs
    } else {
      (void)cudaGetLastError();
    }
  }
  if (!wide) {
    const size_t smem = sizeof(double) * static_cast<size_t>(kMaxD / kCl) * kMaxD;
    if ((e = cudaFuncSetAttribute(eigen_reduce_cluster_kernel<kCl, kMaxD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem))) != cudaSuccess)
      return e;
    count_launch();
    eigen_reduce_cluster_kernel<kCl, kMaxD><<<kCl, kT, smem, st>>>(a);
  }
  const size_t smem3 = sizeof(double) * static_cast<size_t>(kWarps) * lu_stride<kMaxD>();
  if ((e = cudaFuncSetAttribute(eigen_vectors_cluster_kernel<kMaxD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem3))) != cudaSuccess)
    return e;
  count_launch();
  eigen_vectors_cluster_kernel<kMaxD><<<kCl, kT, smem3, st>>>(a);
  return cudaGetLastError();
}

}  // namespace prohd
