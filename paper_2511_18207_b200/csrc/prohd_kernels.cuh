// prohd_kernels.cuh — launchers of the ProHD-specific kernels (K1 moments, K2
// eigen, K3 projection, K4 selection, K5 union/gather).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace prohd {

// ---------------------------------------------------------------- K1
// Gram pass (k_gram.cu): groups of <= 12 upper-triangle 32x32 tiles over <= 8 feature blocks
constexpr int kGramMaxFb = 32;      // D <= 1024
constexpr int kGramMaxGroups = 64;  // 8 diagonal + 2 x 28 off-diagonal 4x4-block squares at D = 1024
struct GramGroup {
  unsigned char ntiles, nfb, nslot, rep;  // nslot: staged slots (power of 2 >= nfb); rep: warps per tile
  unsigned char fb[8];    // feature blocks (32 features each) staged in slots 0..nfb-1
  unsigned char si[12];   // tile t = (fb[si[t]], fb[sj[t]]); si == sj: a diagonal tile (upper 8x8 blocks only)
  unsigned char sj[12];
  int rpg, cta0;          // the group's point ranges (CTAs cta0 .. cta0 + rpg - 1)
  int64_t per;            // points per range (multiple of 16)
  int load;               // DMMAs per k-step on the busiest SM sub-partition (plan_gram's cost model)
};
struct GramPlan {
  int ngroups = 0, nctas = 0;
  int64_t gpart_doubles = 0, spart_doubles = 0;
  int cs_blocks = 0;     // column-sum partial slots (colsum_kernel CTAs, or in-launch CTAs x row phases)
  int64_t cs_per = 0;    // rows per colsum CTA
  int cs_ctas = 0;       // > 0: the Gram launch carries this many column-sum CTAs after its nctas
  GramGroup grp[kGramMaxGroups];
};
bool plan_gram(int64_t nA, int64_t nB, int D, int num_sms, GramPlan& p);
cudaError_t launch_gram(const GramPlan& p, const float* A, int64_t nA, const float* B, int64_t nB, int D,
                        const double* s, double* Gpart, double* Spart, double* Gout, double* SA, double* SB,
                        cudaStream_t st);

// int8 tensor-core Gram (k_gram_i8.cu): exact-integer Ozaki slices on tcgen05 kind::i8 CTA pairs,
// D <= 256, D % 4 == 0. Writes G (D x D), S_A, S_B about its own fixed-point shift s'
// (overwrites s), and sets *overflow if a value fell outside the sampled range (then the caller
// reruns the fp64 DMMA Gram).
struct GramI8Plan {
  int D = 0, ngroups = 0, nctas = 0;
  int small = 0;  // 1: D <= 128 gram_i8s_kernel, nt0 + nt1 single CTAs (level sets); 2: D <= 64 gram_i8d_kernel
  int nt0 = 0, nt1 = 0;
  int64_t slab_doubles = 0, csum_count = 0;
};
bool plan_gram_i8(int64_t nA, int64_t nB, int D, int num_sms, GramI8Plan& p);
size_t gram_i8_ws_bytes(const GramI8Plan& p);
cudaError_t launch_gram_i8(const GramI8Plan& p, const float* A, int64_t nA, const float* B, int64_t nB,
                           uint8_t* ws, double* s, double* G, double* SA, double* SB, unsigned* overflow,
                           cudaStream_t st, const float* colmax_in = nullptr, const double* s_to = nullptr);
// sharded phase: per-feature max |x - s| of these rows (fp32, non-finite -> +inf) into colmax_out (device)
cudaError_t launch_colmax_i8(const GramI8Plan& p, const float* A, int64_t nA, const float* B, int64_t nB,
                             uint8_t* ws, const double* s, float* colmax_out, cudaStream_t st);

struct MomentsPlan {
  int nb = 0, npairs = 0, c_diag = 0, c_off = 0, nctas = 0, nslots = 0;
  bool gram = false;  // warp-specialised Gram pass (k_gram.cu); else the legacy 64x64-block kernel
  GramPlan gp;
  bool i8 = false;    // int8 tensor-core Gram (the default where supported, k_gram_i8.cu)
  GramI8Plan ip;
  int64_t gpart_doubles = 0, spart_doubles = 0;
  int64_t i8_bytes = 0;  // slabs, column-sum partials, scales (k_gram_i8.cu)
};
struct MomentsBufs {
  uint8_t* i8ws = nullptr;  // int8 Gram scratch (MomentsPlan::i8_bytes)
  unsigned* i8ovf = nullptr;  // int8 Gram range overflow flag
  double* s;      // [2D]: shift s (0 unless the offset is large), then D doubles of scratch
  double* Gpart;  // partial Grams
  double* Spart;  // partial column sums
  double* C;      // [D][D] -> covariance
  double* SA;     // [D]
  double* SB;     // [D]
  double* mu;     // [D] mean of A u B
  double* u0;     // [D] centroid axis (row 0 of U64)
  double* dnorm;  // ||mu_B - mu_A||
};
MomentsPlan plan_moments(int64_t nA, int64_t nB, int D, int num_sms);
cudaError_t launch_moments(const MomentsPlan& p, const float* A, int64_t nA, const float* B, int64_t nB, int D,
                           const MomentsBufs& b, cudaStream_t st);
// pieces of launch_moments (sharded path): shift s from the first <= 4096 rows of A and B;
// partial sums about b.s (-> b.SA, b.SB, b.C = G); finalize (mu, u0, C from the sums).
cudaError_t launch_shift(const float* A, int64_t nA, const float* B, int64_t nB, int D, double* s, cudaStream_t st);
// use_i8: the int8 tensor-core Gram when planned (it replaces b.s by its own shift s'; the
// sharded phase calls, whose shift is fixed by the caller, pass false), else the fp64 DMMA pass
cudaError_t launch_moments_partial(const MomentsPlan& p, const float* A, int64_t nA, const float* B, int64_t nB,
                                   int D, const MomentsBufs& b, cudaStream_t st, bool use_i8 = false);
cudaError_t launch_moments_finalize(int64_t nA, int64_t nB, int D, const MomentsBufs& b, cudaStream_t st);

// ---------------------------------------------------------------- K2
// Top-k eigenvectors of C (destroyed). Writes rows 1..k of out64/out32 ([k+1][D]),
// lam[0..k), and *n_dirs = 1 + number kept. V: D*D doubles, X: k*D doubles scratch.
cudaError_t launch_eigen_topk(double* C, int D, int k, double* V, double* X, double* out64, float* out32,
                              double* lam, int* n_dirs, cudaStream_t st);
// U32 = (float)U64 for rows [0, rows)
cudaError_t launch_dirs_to_f32(const double* U64, float* U32, int rows, int D, cudaStream_t st);

// ---------------------------------------------------------------- K3/K4/K5 (one point set)
constexpr int kRadixBins = 2048;
constexpr int kCompactBlocks = 128;  // K5 compaction CTAs
struct SelectBufs {
  float* P32;             // [L][n] fp32 projections, direction-major
  unsigned* maxnorm2;     // float bits of max ||x||^2 (atomicMax)
  unsigned* hist;         // [3 rounds][L][2][kRadixBins]
  unsigned* state;        // [L][2][4]: prefix, mask, remaining, unused
  int* cand;              // [L][2][cap]
  double* cval;           // [L][2][cap]
  unsigned* ccount;       // [L][2]
  int* lists;             // [L][2][m]
  unsigned* bitmap;       // [ceil(n/32)]
  long long* uidx;        // sorted unique union (capacity min(n, 2mL))
  unsigned* ucount;       // union size, then kCompactBlocks words of compaction scratch
  int* overflow;          // guard-band overflow flag
  int64_t cap;            // candidates per list
  int* sfail = nullptr;   // sampled K4 could not certify a list: rerun launch_select (nullptr: no sampled K4)
};
// first: reset the union bitmap/flags; last: compact the bitmap into the sorted union. Two calls
// (first=true,last=false then first=false,last=true) select with different m per direction group.
// K3 on the tensor cores (k_project_tc.cu): D % 4 == 0, D <= 256, 1 <= L <= 32
bool project_tc_supported(int64_t n, int D, int L);
double project_tc_eps_coef(int D);  // |pi32 - pi64| <= coef * ||x||
// fused pre-selection in K3's epilogue (sampled K4): state[lt * 4 + 0] = float bits of the
// threshold of list lt = 2 l + tail (top: pi >= thr, bottom: pi <= thr); every epilogue warp w
// (= 4 CTA + warp, 4 per CTA) appends (index, pi32) to its private slab sidx / sval
// [w][2L][capw] and stores its fill counts wcount[w][2L] (possibly > capw) at the end
struct ProjectFuse {
  const unsigned* state = nullptr;
  int* sidx = nullptr;
  float* sval = nullptr;
  unsigned* wcount = nullptr;
  int capw = 0;
  int ablate = 0;  // dev timing only (option k4_sampled 2 | 3): 1 no tests, 2 no appends
};
// row_stride (floats, 0 = D): rows of X at that pitch (the sampled K4 projects every (n/s)-th row)
cudaError_t launch_project_tc(const float* X, int64_t n, int D, const float* U32, int L, float* P32,
                              unsigned* maxnorm2, int num_sms, cudaStream_t st, const ProjectFuse* fuse = nullptr,
                              int64_t row_stride = 0);
// K3 dispatch (tensor-core kernel, else SIMT): P32 = direction-major projections, atomicMax of
// max ||x||^2 bits into *maxnorm2 (zeroed by the caller); *eps_coef: |pi32 - pi64| <= coef ||x||
cudaError_t launch_project(const float* X, int64_t n, int D, const float* U32, int L, float* P32,
                           unsigned* maxnorm2, cudaStream_t st, double* eps_coef);
cudaError_t launch_select(const float* X, int64_t n, int D, const double* U64, const float* U32, int L,
                          const int* n_dirs, int64_t m, const SelectBufs& b, cudaStream_t st, bool first = true,
                          bool last = true, double* eps_out = nullptr);
// K4 with a sampled threshold and K3's fused pre-selection (k_select.cu): the same candidate
// lists, union and bitmap as launch_select (first = last = true) for one direction group; *used
// = false (nothing launched) where it does not apply (option k4_sampled, n, m, K3 variant, or
// b.sfail == nullptr). A list it cannot certify sets *b.sfail: rerun launch_select.
bool select_sampled_plan(int64_t n, int D, int L, int64_t m, int* s_out, unsigned* r_out);
cudaError_t launch_select_sampled(const float* X, int64_t n, int D, const double* U64, const float* U32, int L,
                                  const int* n_dirs, int64_t m, const SelectBufs& b, cudaStream_t st,
                                  double* eps_out, bool* used);
// K4 fallback for lists whose guard band overflowed the candidate buffer (ccount > cap after
// launch_select / launch_local_candidates): exact streaming radix select on (fp64 projection,
// index), then the usual ranking into lists + bitmap (and the compaction if `compact`), or into
// cval_out / cidx_out for the sharded path. eps_coef: the value launch_select reported.
cudaError_t launch_select_fallback(const float* X, int64_t n, int D, const double* U64, int L, const int* n_dirs,
                                   int64_t m, const SelectBufs& b, double eps_coef, cudaStream_t st, bool compact,
                                   double* cval_out = nullptr, long long* cidx_out = nullptr,
                                   int64_t row_offset = 0);
struct StatusSrc {
  const unsigned* uc[2];
  const int* ovf[2];
  const unsigned* maxn[2];
  const int* ndirs;
  const unsigned* i8ovf;  // may be null
  const int* sfail[2];    // may be null
};
constexpr int kStatusWords = 10;
cudaError_t launch_pack_status(const StatusSrc& src, unsigned* out, cudaStream_t st);
struct EstResultDev {
  unsigned long long key[2];  // packed (d2 bits, ~row) of h(A_sel, .) and h(B_sel, .)
  double d2[2];               // fp64 witness distances
  long long a[2], b[2];       // witnesses as original indices
};
cudaError_t launch_pack_result(const unsigned long long* keys, const double* nn_d, const long long* nn_j,
                               const long long* uA, const long long* uB, bool map_cols, EstResultDev* out,
                               cudaStream_t st);
struct ExactResDev {           // directed_hd / hausdorff result, one device-to-host copy
  unsigned long long key[2];
  double d2[2];
  long long j[2];
  int bad;
  int _pad;
};
cudaError_t launch_pack_exact(const unsigned long long* keys, const double* nn_d, const long long* nn_j,
                              const int* bad, ExactResDev* out, cudaStream_t st);
cudaError_t launch_set_int(int* a, int v, cudaStream_t st);  // *a = v (stream-ordered, capturable)
cudaError_t launch_minus_one(const int* a, int* b, cudaStream_t st);  // *b = max(*a - 1, 0)
// Sharded selection: local top/bottom-m lists with their fp64 projection values and GLOBAL
// indices (row_offset + local row) -> cval_out/cidx_out [L][2][m] (index -1 = empty slot).
// If m >= n every local point is a candidate of every list.
cudaError_t launch_local_candidates(const float* X, int64_t n, int64_t row_offset, int D, const double* U64,
                                    const float* U32, int L, const int* n_dirs, int64_t m, const SelectBufs& b,
                                    double* cval_out, long long* cidx_out, cudaStream_t st, double* eps_out = nullptr);
// Merge G ranks' lists [G][L][2][m] into the global top/bottom-m per list (same total
// order) and the sorted unique union of their global indices (bitmap over n_total rows).
cudaError_t launch_merge_union(const double* cval, const long long* cidx, int G, int L, int64_t m, int64_t n_total,
                               unsigned* bitmap, long long* uidx, unsigned* ucount /* 1 + kCompactBlocks */,
                               const int* n_dirs,
                               cudaStream_t st);
// rows_out[i] = X_local[idx[lo + i] - row_offset] for i < cnt
cudaError_t launch_gather_offset(const float* X, int D, const long long* idx, int64_t lo, int64_t cnt,
                                 int64_t row_offset, float* rows_out, cudaStream_t st);
// Gather rows X[idx[i]] -> Y (row-major, stride D) for i < count (count on the device).
cudaError_t launch_gather(const float* X, int D, const long long* idx, const unsigned* count, int64_t cap,
                          float* Y, cudaStream_t st);
cudaError_t launch_iota(long long* idx, unsigned* count, int64_t n, cudaStream_t st);

// ---------------------------------------------------------------- f2 bounds
struct BoundsPlan {
  int nblk = 0;
  int64_t keys_words = 0, count_words = 0;
};
struct BoundsBufs {
  unsigned *keysA, *keysB, *sortA, *sortB, *tmp, *counts;  // [L][n] order-preserving keys, radix scratch
  unsigned long long* delta2;  // [L][2] fp64 bits: max delta^2 (origin, centred), error-inflated
  unsigned long long* hu;      // [2][L] fp64 bits: h_u(A,B) then h_u(B,A)
};
constexpr int kMeanParts = 296;
BoundsPlan plan_bounds(int64_t nA, int64_t nB, int L);
cudaError_t launch_union_mean(const float* A, int64_t nA, const float* B, int64_t nB, int D, double* part,
                              double* mu, cudaStream_t st);
cudaError_t launch_bounds(const float* A, int64_t nA, const float* B, int64_t nB, int D, const float* U32, int L,
                          const double* mu, const BoundsBufs& b, cudaStream_t st);

}  // namespace prohd
