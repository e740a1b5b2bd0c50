// prohd_shard.cu — phase calls of the row-sharded (multi-GPU) ProHD, SURVEY.md §8(b)/(e).
//
// The driver (paper_2511_18207_b200/dist.py) owns the process group; between these calls
// it runs the collectives (C1 SUM all-reduce of the moments, C2 all-gather of candidate
// lists, C3 all-gather of the selected rows, C4 MAX all-reduce of the subset-HD keys).
// Every arithmetic step runs in the same kernels as the single-GPU path:
//   prohd_shift            K1 shift kernel on the first rows (rank 0's shard)
//   prohd_local_moments    K1 partial sums of this rank's rows about the common shift
//   prohd_directions       K1 finalize + K2 eigen on the all-reduced moments (replicated)
//   prohd_local_candidates K3 + K4 on this rank's rows: local top/bottom-m with fp64 values
//   prohd_merge_union      merge of all ranks' lists by the same total order + K5 union
//   prohd_gather_owned     this rank's rows of the union, in union order
// Because the fp64 projection values and the (value, index) order are identical on every
// rank, the merged lists equal the single-GPU lists (oracle O12 / tests).
#include "api_common.cuh"
#include "prohd_kernels.cuh"
#include "prohd_steps.cuh"

#include <algorithm>
#include <cmath>
#include <vector>

namespace prohd {

struct ShardWs {
  float* stageA = nullptr;
  float* stageB = nullptr;
  MomentsBufs mom{};
  double* V = nullptr;
  double* Xe = nullptr;
  double* U64 = nullptr;
  float* U32 = nullptr;
  double* lam = nullptr;
  int* n_dirs = nullptr;
  SelectBufs sel{};
  unsigned* bitmap = nullptr;
  unsigned* ucount = nullptr;
};

static size_t carve_shard(Carver& c, ShardWs& w, int64_t nA, int64_t nB, int64_t n_total, int D, int k, int64_t m,
                          bool host_inputs, int num_sms) {
  const int L = k + 1;
  if (host_inputs) {
    w.stageA = c.take<float>(nA * D);
    w.stageB = c.take<float>(nB * D);
  }
  const MomentsPlan mp = plan_moments(nA, nB, D, num_sms);
  w.mom.s = c.take<double>(2 * static_cast<int64_t>(D));  // shift + scratch
  w.mom.Gpart = c.take<double>(mp.gpart_doubles);
  w.mom.Spart = c.take<double>(mp.spart_doubles);
  if (mp.i8) {
    w.mom.i8ws = c.take<uint8_t>(mp.i8_bytes);
    w.mom.i8ovf = c.take<unsigned>(1);
  }
  w.mom.C = c.take<double>(static_cast<int64_t>(D) * D);
  w.mom.SA = c.take<double>(D);
  w.mom.SB = c.take<double>(D);
  w.mom.mu = c.take<double>(D);
  w.mom.dnorm = c.take<double>(1);
  w.V = c.take<double>(static_cast<int64_t>(D) * D + 2 * 512);  // Householder vectors + d, e of T
  w.Xe = c.take<double>(static_cast<int64_t>(k > 0 ? k : 1) * D);
  w.U64 = c.take<double>(static_cast<int64_t>(L) * D);
  w.mom.u0 = w.U64;
  w.U32 = c.take<float>(static_cast<int64_t>(L) * D);
  w.lam = c.take<double>(k > 0 ? k : 1);
  w.n_dirs = c.take<int>(1);
  const int64_t nl = nA > nB ? nA : nB;
  SelectBufs& b = w.sel;
  b.cap = (nl < m + 65536) ? (nl > 0 ? nl : 1) : m + 65536;
  b.P32 = c.take<float>(static_cast<int64_t>(L) * (nl > 0 ? nl : 1));
  b.maxnorm2 = c.take<unsigned>(1);
  b.hist = c.take<unsigned>(static_cast<int64_t>(3) * L * 2 * kRadixBins);
  b.state = c.take<unsigned>(static_cast<int64_t>(L) * 2 * 4);
  b.cand = c.take<int>(static_cast<int64_t>(L) * 2 * b.cap);
  b.cval = c.take<double>(static_cast<int64_t>(L) * 2 * b.cap);
  b.ccount = c.take<unsigned>(static_cast<int64_t>(L) * 2);
  b.overflow = c.take<int>(1);
  w.bitmap = c.take<unsigned>((n_total + 31) / 32 + 1);
  w.ucount = c.take<unsigned>(1 + kCompactBlocks);  // count, then compaction scratch
  return c.off;
}

size_t shard_workspace_bytes(int64_t n_local_max, int64_t n_total_max, int D, int k, int64_t m, bool host_inputs) {
  Carver c{nullptr, 0, 0, true};
  ShardWs w;
  return carve_shard(c, w, n_local_max, n_local_max, n_total_max, D, k, m, host_inputs, 148);
}

}  // namespace prohd

static int shard_begin(prohd_ctx* ctx, ShardWs& w, int64_t nA, int64_t nB, int64_t n_total, int D, int k, int64_t m,
                       bool host_inputs) {
  Carver dry{nullptr, 0, 0, true};
  ShardWs tmp;
  const size_t need = carve_shard(dry, tmp, nA, nB, n_total, D, k, m, host_inputs, ctx->num_sms);
  if (ctx->ws == nullptr || ctx->ws_bytes < need)
    return fail(ctx, PROHD_E_WORKSPACE, "workspace too small: need %zu bytes, have %zu", need, ctx->ws_bytes);
  Carver c{ctx->ws, 0, ctx->ws_bytes, false};
  carve_shard(c, w, nA, nB, n_total, D, k, m, host_inputs, ctx->num_sms);
  return PROHD_OK;
}

// host shards are staged through the workspace; device shards must be 16-byte aligned
static int stage_local(prohd_ctx* ctx, ShardWs& w, const float*& A_local, int64_t nA_local, const float*& B_local,
                       int64_t nB_local, int D) {
  cudaStream_t st = ctx->stream;
  if (nA_local > 0 && !is_device_ptr(A_local)) {
    CK(cudaMemcpyAsync(w.stageA, A_local, sizeof(float) * nA_local * D, cudaMemcpyHostToDevice, st));
    A_local = w.stageA;
  }
  if (nB_local > 0 && !is_device_ptr(B_local)) {
    CK(cudaMemcpyAsync(w.stageB, B_local, sizeof(float) * nB_local * D, cudaMemcpyHostToDevice, st));
    B_local = w.stageB;
  }
  int rc;
  if ((rc = check_aligned(ctx, nA_local > 0 ? A_local : nullptr, D, "A_local")) ||
      (rc = check_aligned(ctx, nB_local > 0 ? B_local : nullptr, D, "B_local")))
    return rc;
  return PROHD_OK;
}

extern "C" {

size_t prohd_shard_workspace_bytes(int64_t n_local_max, int64_t n_total_max, int32_t D, int32_t k, int64_t m,
                                   uint32_t flags) {
  if (D < 1 || k < 0 || m < 1 || n_local_max < 0 || n_total_max < 1) return 0;
  return shard_workspace_bytes(n_local_max, n_total_max, D, k, m, (flags & PROHD_WS_HOST_INPUTS) != 0) + 256;
}

int prohd_shift(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D,
                double* shift_out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (shift_out == nullptr) return fail(ctx, PROHD_E_INVALID, "null shift_out");
  if ((rc = check_sets(ctx, A, nA, B, nB, D))) return rc;
  call_begin(ctx);
  const int64_t ca = nA < 4096 ? nA : 4096, cb = nB < 4096 ? nB : 4096;
  ShardWs w;
  const bool host_in = !(is_device_ptr(A) && is_device_ptr(B));
  if ((rc = shard_begin(ctx, w, ca, cb, 1, D, 0, 1, host_in))) return rc;
  bool hi;
  if ((rc = stage_inputs(ctx, A, ca, B, cb, D, w.stageA, w.stageB, hi))) return rc;
  CK(launch_shift(A, ca, B, cb, D, w.mom.s, ctx->stream));
  CK(cudaMemcpyAsync(shift_out, w.mom.s, sizeof(double) * D, cudaMemcpyDeviceToHost, ctx->stream));
  call_end(ctx);
  CK(cudaStreamSynchronize(ctx->stream));
  call_collect(ctx);
  return PROHD_OK;
}

int prohd_local_moments(prohd_ctx* ctx, const float* A_local, int64_t nA_local, const float* B_local,
                        int64_t nB_local, int32_t D, const double* shift, double* moments_out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (shift == nullptr || moments_out == nullptr) return fail(ctx, PROHD_E_INVALID, "null shift or moments_out");
  if (D < 1 || nA_local < 0 || nB_local < 0) return fail(ctx, PROHD_E_INVALID, "bad sizes");
  if ((nA_local > 0 && A_local == nullptr) || (nB_local > 0 && B_local == nullptr))
    return fail(ctx, PROHD_E_INVALID, "null input");
  call_begin(ctx);
  const bool host_in = (nA_local > 0 && !is_device_ptr(A_local)) || (nB_local > 0 && !is_device_ptr(B_local));
  ShardWs w;
  if ((rc = shard_begin(ctx, w, nA_local, nB_local, 1, D, 0, 1, host_in))) return rc;
  cudaStream_t st = ctx->stream;
  if ((rc = stage_local(ctx, w, A_local, nA_local, B_local, nB_local, D))) return rc;
  CK(cudaMemcpyAsync(w.mom.s, shift, sizeof(double) * D, cudaMemcpyHostToDevice, st));
  const int t0 = tmark(ctx);
  CK(cudaMemsetAsync(w.mom.SA, 0, sizeof(double) * D, st));
  CK(cudaMemsetAsync(w.mom.SB, 0, sizeof(double) * D, st));
  CK(cudaMemsetAsync(w.mom.C, 0, sizeof(double) * D * D, st));
  if (nA_local + nB_local > 0) {
    const MomentsPlan mp = plan_moments(nA_local, nB_local, D, ctx->num_sms);
    // the caller's shift is fixed across ranks (the moments are summed by an all-reduce), so the
    // phase call keeps the fp64 DMMA Gram (the int8 pass chooses its own fixed-point shift)
    CK(launch_moments_partial(mp, A_local, nA_local, B_local, nB_local, D, w.mom, st, false));
  }
  tspan(ctx, PH_MOMENTS, t0);
  CK(cudaMemcpyAsync(moments_out, w.mom.SA, sizeof(double) * D, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(moments_out + D, w.mom.SB, sizeof(double) * D, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(moments_out + 2 * D, w.mom.C, sizeof(double) * D * D, cudaMemcpyDeviceToDevice, st));
  call_end(ctx);
  CK(cudaStreamSynchronize(st));
  call_collect(ctx);
  return PROHD_OK;
}

// Sharded int8 moments, step 1: this rank's per-feature max |x - s| (the grid of the int8 Gram).
int prohd_local_colmax(prohd_ctx* ctx, const float* A_local, int64_t nA_local, const float* B_local,
                       int64_t nB_local, int32_t D, const double* shift, float* colmax_out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (shift == nullptr || colmax_out == nullptr) return fail(ctx, PROHD_E_INVALID, "null shift or colmax_out");
  if (D < 1 || nA_local < 0 || nB_local < 0) return fail(ctx, PROHD_E_INVALID, "bad sizes");
  if ((nA_local > 0 && A_local == nullptr) || (nB_local > 0 && B_local == nullptr))
    return fail(ctx, PROHD_E_INVALID, "null input");
  if (D > 256 || D % 4 != 0) return fail(ctx, PROHD_E_NOTIMPL, "the int8 Gram needs D <= 256, D %% 4 == 0");
  call_begin(ctx);
  const bool host_in = (nA_local > 0 && !is_device_ptr(A_local)) || (nB_local > 0 && !is_device_ptr(B_local));
  ShardWs w;
  if ((rc = shard_begin(ctx, w, nA_local, nB_local, 1, D, 0, 1, host_in))) return rc;
  cudaStream_t st = ctx->stream;
  if ((rc = stage_local(ctx, w, A_local, nA_local, B_local, nB_local, D))) return rc;
  CK(cudaMemcpyAsync(w.mom.s, shift, sizeof(double) * D, cudaMemcpyHostToDevice, st));
  GramI8Plan ip;
  if (nA_local + nB_local > 0 && w.mom.i8ws != nullptr && plan_gram_i8(nA_local, nB_local, D, ctx->num_sms, ip)) {
    const int t0 = tmark(ctx);
    CK(launch_colmax_i8(ip, A_local, nA_local, B_local, nB_local, w.mom.i8ws, w.mom.s, colmax_out, st));
    tspan(ctx, PH_MOMENTS, t0);
  } else {
    CK(cudaMemsetAsync(colmax_out, 0, sizeof(float) * D, st));  // no rows: the MAX identity
  }
  call_end(ctx);
  CK(cudaStreamSynchronize(st));
  call_collect(ctx);
  return PROHD_OK;
}

// Sharded int8 moments, step 2: prohd_local_moments on the int8 tensor cores with the grid of the
// all-reduced column maxima (identical on every rank), re-expressed about the caller's shift.
int prohd_local_moments_i8(prohd_ctx* ctx, const float* A_local, int64_t nA_local, const float* B_local,
                           int64_t nB_local, int32_t D, const double* shift, const float* colmax,
                           double* moments_out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (shift == nullptr || moments_out == nullptr || colmax == nullptr)
    return fail(ctx, PROHD_E_INVALID, "null shift, colmax or moments_out");
  if (D < 1 || nA_local < 0 || nB_local < 0) return fail(ctx, PROHD_E_INVALID, "bad sizes");
  if ((nA_local > 0 && A_local == nullptr) || (nB_local > 0 && B_local == nullptr))
    return fail(ctx, PROHD_E_INVALID, "null input");
  if (D > 256 || D % 4 != 0) return fail(ctx, PROHD_E_NOTIMPL, "the int8 Gram needs D <= 256, D %% 4 == 0");
  call_begin(ctx);
  const bool host_in = (nA_local > 0 && !is_device_ptr(A_local)) || (nB_local > 0 && !is_device_ptr(B_local));
  ShardWs w;
  if ((rc = shard_begin(ctx, w, nA_local, nB_local, 1, D, 0, 1, host_in))) return rc;
  cudaStream_t st = ctx->stream;
  if ((rc = stage_local(ctx, w, A_local, nA_local, B_local, nB_local, D))) return rc;
  // a non-finite global column max (non-finite input on some rank): the fp64 DMMA Gram, whose
  // sums carry the non-finite value to prohd_directions (PROHD_E_DATA there)
  std::vector<float> cm(D);
  CK(cudaMemcpyAsync(cm.data(), colmax, sizeof(float) * D, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(w.mom.s, shift, sizeof(double) * D, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(w.mom.s + D, shift, sizeof(double) * D, cudaMemcpyHostToDevice, st));  // target shift
  CK(cudaStreamSynchronize(st));
  bool finite = true;
  for (float v : cm) finite = finite && std::isfinite(v) && v < 3.0e38f;
  const int t0 = tmark(ctx);
  CK(cudaMemsetAsync(w.mom.SA, 0, sizeof(double) * D, st));
  CK(cudaMemsetAsync(w.mom.SB, 0, sizeof(double) * D, st));
  CK(cudaMemsetAsync(w.mom.C, 0, sizeof(double) * D * D, st));
  if (nA_local + nB_local > 0) {
    GramI8Plan ip;
    const bool i8 = finite && w.mom.i8ws != nullptr && w.mom.i8ovf != nullptr &&
                    plan_gram_i8(nA_local, nB_local, D, ctx->num_sms, ip);
    if (i8) {
      CK(cudaMemsetAsync(w.mom.i8ovf, 0, sizeof(unsigned), st));
      CK(launch_gram_i8(ip, A_local, nA_local, B_local, nB_local, w.mom.i8ws, w.mom.s, w.mom.C, w.mom.SA, w.mom.SB,
                        w.mom.i8ovf, st, colmax, w.mom.s + D));
    } else {
      const MomentsPlan mp = plan_moments(nA_local, nB_local, D, ctx->num_sms);
      CK(launch_moments_partial(mp, A_local, nA_local, B_local, nB_local, D, w.mom, st, false));
    }
  }
  tspan(ctx, PH_MOMENTS, t0);
  CK(cudaMemcpyAsync(moments_out, w.mom.SA, sizeof(double) * D, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(moments_out + D, w.mom.SB, sizeof(double) * D, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(moments_out + 2 * D, w.mom.C, sizeof(double) * D * D, cudaMemcpyDeviceToDevice, st));
  call_end(ctx);
  CK(cudaStreamSynchronize(st));
  call_collect(ctx);
  return PROHD_OK;
}

int prohd_directions(prohd_ctx* ctx, const double* moments, int64_t nA, int64_t nB, int32_t D, int32_t k,
                     const double* shift, double* dirs_out, int32_t* n_dirs_out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (moments == nullptr || shift == nullptr || dirs_out == nullptr || n_dirs_out == nullptr)
    return fail(ctx, PROHD_E_INVALID, "null pointer");
  if (nA < 1 || nB < 1 || D < 1) return fail(ctx, PROHD_E_INVALID, "bad sizes");
  if (k < 0 || k > D) return fail(ctx, PROHD_E_INVALID, "k must satisfy 0 <= k <= D");
  if (k > 0 && D > 512) return fail(ctx, PROHD_E_NOTIMPL, "the device eigen-solver supports D <= 512");
  call_begin(ctx);
  ShardWs w;
  if ((rc = shard_begin(ctx, w, 0, 0, 1, D, k, 1, false))) return rc;
  cudaStream_t st = ctx->stream;
  const int L = k + 1;
  CK(cudaMemcpyAsync(w.mom.s, shift, sizeof(double) * D, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(w.mom.SA, moments, sizeof(double) * D, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(w.mom.SB, moments + D, sizeof(double) * D, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(w.mom.C, moments + 2 * D, sizeof(double) * D * D, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemsetAsync(w.U64, 0, sizeof(double) * L * D, st));
  int t0 = tmark(ctx);
  CK(launch_moments_finalize(nA, nB, D, w.mom, st));
  tspan(ctx, PH_MOMENTS, t0);
  if (k > 0) {
    t0 = tmark(ctx);
    CK(launch_eigen_topk(w.mom.C, D, k, w.V, w.Xe, w.U64, w.U32, w.lam, w.n_dirs, st));
    tspan(ctx, PH_EIGEN, t0);
  } else {
    const int one = 1;
    CK(cudaMemcpyAsync(w.n_dirs, &one, sizeof(int), cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemcpyAsync(dirs_out, w.U64, sizeof(double) * L * D, cudaMemcpyDeviceToDevice, st));
  int nd = 0;
  CK(cudaMemcpyAsync(&nd, w.n_dirs, sizeof(int), cudaMemcpyDeviceToHost, st));
  call_end(ctx);
  CK(cudaStreamSynchronize(st));
  call_collect(ctx);
  *n_dirs_out = nd;
  return PROHD_OK;
}

int prohd_local_candidates(prohd_ctx* ctx, const float* X_local, int64_t n_local, int64_t row_offset, int32_t D,
                           const double* dirs, int32_t n_dirs, int64_t m, double* cand_val_out,
                           int64_t* cand_idx_out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (dirs == nullptr || cand_val_out == nullptr || cand_idx_out == nullptr)
    return fail(ctx, PROHD_E_INVALID, "null pointer");
  if (n_local < 0 || (n_local > 0 && X_local == nullptr) || D < 1 || n_dirs < 1 || m < 1 || row_offset < 0)
    return fail(ctx, PROHD_E_INVALID, "bad arguments");
  call_begin(ctx);
  const bool host_in = n_local > 0 && !is_device_ptr(X_local);
  ShardWs w;
  if ((rc = shard_begin(ctx, w, n_local, 0, 1, D, n_dirs - 1, m, host_in))) return rc;
  cudaStream_t st = ctx->stream;
  if (host_in) {
    CK(cudaMemcpyAsync(w.stageA, X_local, sizeof(float) * n_local * D, cudaMemcpyHostToDevice, st));
    X_local = w.stageA;
  }
  if ((rc = check_aligned(ctx, n_local > 0 ? X_local : nullptr, D, "X_local"))) return rc;
  CK(cudaMemcpyAsync(w.U64, dirs, sizeof(double) * n_dirs * D, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(w.n_dirs, &n_dirs, sizeof(int), cudaMemcpyHostToDevice, st));
  CK(launch_dirs_to_f32(w.U64, w.U32, n_dirs, D, st));
  const int t0 = tmark(ctx);
  double eps = 0.0;
  CK(launch_local_candidates(X_local, n_local, row_offset, D, w.U64, w.U32, n_dirs, w.n_dirs, m, w.sel,
                             cand_val_out, reinterpret_cast<long long*>(cand_idx_out), st, &eps));
  int ovf = 0;
  unsigned maxn = 0;
  if (n_local > 0) {
    CK(cudaMemcpyAsync(&ovf, w.sel.overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&maxn, w.sel.maxnorm2, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (ovf)  // guard band overflowed its buffer (massive ties): exact band select for those lists
      CK(launch_select_fallback(X_local, n_local, D, w.U64, n_dirs, w.n_dirs, m, w.sel, eps, st, false,
                                cand_val_out, reinterpret_cast<long long*>(cand_idx_out), row_offset));
  }
  tspan(ctx, PH_SELECT, t0);
  call_end(ctx);
  CK(cudaStreamSynchronize(st));
  call_collect(ctx);
  float f;
  std::memcpy(&f, &maxn, 4);
  if (!std::isfinite(f)) return fail(ctx, PROHD_E_DATA, "non-finite input coordinate (or squared norm overflow)");
  return PROHD_OK;
}

int prohd_merge_union(prohd_ctx* ctx, const double* cand_val, const int64_t* cand_idx, int32_t G, int32_t n_dirs,
                      int64_t m, int64_t n_total, int64_t* union_out, int64_t* count_out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (cand_val == nullptr || cand_idx == nullptr || union_out == nullptr || count_out == nullptr)
    return fail(ctx, PROHD_E_INVALID, "null pointer");
  if (G < 1 || n_dirs < 1 || m < 1 || n_total < 1) return fail(ctx, PROHD_E_INVALID, "bad sizes");
  call_begin(ctx);
  ShardWs w;
  if ((rc = shard_begin(ctx, w, 0, 0, n_total, 1, n_dirs - 1, 1, false))) return rc;
  cudaStream_t st = ctx->stream;
  const int t0 = tmark(ctx);
  if (2 * m >= n_total) {
    CK(launch_iota(reinterpret_cast<long long*>(union_out), w.ucount, n_total, st));
  } else {
    CK(cudaMemcpyAsync(w.n_dirs, &n_dirs, sizeof(int), cudaMemcpyHostToDevice, st));
    CK(launch_merge_union(cand_val, reinterpret_cast<const long long*>(cand_idx), G, n_dirs, m, n_total, w.bitmap,
                          reinterpret_cast<long long*>(union_out), w.ucount, w.n_dirs, st));
  }
  tspan(ctx, PH_SELECT, t0);
  unsigned cnt = 0;
  CK(cudaMemcpyAsync(&cnt, w.ucount, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  call_end(ctx);
  CK(cudaStreamSynchronize(st));
  call_collect(ctx);
  *count_out = cnt;
  return PROHD_OK;
}

int prohd_gather_owned(prohd_ctx* ctx, const float* X_local, int64_t n_local, int64_t row_offset, int32_t D,
                       const int64_t* union_idx, int64_t union_count, float* rows_out, int64_t* first_out,
                       int64_t* count_out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (union_idx == nullptr || first_out == nullptr || count_out == nullptr) return fail(ctx, PROHD_E_INVALID, "null");
  if (n_local < 0 || union_count < 0 || D < 1) return fail(ctx, PROHD_E_INVALID, "bad sizes");
  call_begin(ctx);
  cudaStream_t st = ctx->stream;
  std::vector<int64_t> u(static_cast<size_t>(union_count));
  if (union_count > 0)
    CK(cudaMemcpyAsync(u.data(), union_idx, sizeof(int64_t) * union_count, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const int64_t lo = std::lower_bound(u.begin(), u.end(), row_offset) - u.begin();
  const int64_t hi = std::lower_bound(u.begin(), u.end(), row_offset + n_local) - u.begin();
  if (hi > lo) {
    if (rows_out == nullptr || X_local == nullptr) return fail(ctx, PROHD_E_INVALID, "null rows_out / X_local");
    CK(launch_gather_offset(X_local, D, reinterpret_cast<const long long*>(union_idx), lo, hi - lo, row_offset,
                            rows_out, st));
  }
  call_end(ctx);
  CK(cudaStreamSynchronize(st));
  call_collect(ctx);
  *first_out = lo;
  *count_out = hi - lo;
  return PROHD_OK;
}

}  // extern "C"
