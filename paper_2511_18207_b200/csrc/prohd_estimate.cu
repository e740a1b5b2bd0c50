// prohd_estimate.cu — orchestration of ProHD Alg. 3 on the device.
//
//   step 1a  K1 moments: centroids + covariance of A u B            (Alg.1 l.1, Alg.2 l.1-2)
//   step 1b  u0 = normalised centroid difference (e1 rule) + K2 eigen (Alg.1 l.2, Alg.2 l.2)
//   step 2   K3 projections onto U = [u0 u1..uk]                     (Alg.1 l.3-4, Alg.2 l.5-7)
//   step 3   K4 top/bottom-m per direction, K5 union + gather        (Alg.1 l.5-9, Alg.2 l.8-11, Alg.3 l.4-5)
//   step 4   K0+K6+K7 exact HD on the subsets, both directions       (Alg.3 l.6-7)
// One host synchronisation (after step 3) reads the subset sizes to size the distance-kernel
// launches (one packed device-to-host copy of every status word); everything else is
// stream-ordered, and the result comes back in one packed copy.
#include "api_common.cuh"
#include "prohd_kernels.cuh"
#include "prohd_steps.cuh"

#include <vector>

namespace prohd {

struct EstWs {
  float* stageA = nullptr;
  float* stageB = nullptr;
  MomentsBufs mom{};
  double* V = nullptr;
  double* Xe = nullptr;
  double* U64 = nullptr;
  float* U32 = nullptr;
  double* lam = nullptr;
  int* n_dirs = nullptr;
  int* n_dirs1 = nullptr;  // n_dirs - 1 (principal directions only)
  SelectBufs sel[2]{};
  float* Xs[2] = {nullptr, nullptr};
  SetOps ops[2];
  SetOps full[2];  // certified mode: operands of the full sets (columns of the subset-full HD)
  float* rowmin = nullptr;
  float* colmin = nullptr;
  unsigned long long* keys = nullptr;
  double* nn_d = nullptr;
  long long* nn_j = nullptr;
  double* blk_d = nullptr;
  long long* blk_j = nullptr;
  int* bad = nullptr;
  double* centre = nullptr;  // [2D] common centre of the subset pair (K0)
  unsigned* status = nullptr;  // [kStatusWords] the mid-pipeline host read (pack_status_kernel)
  EstResultDev* res = nullptr;  // the final host read (pack_result_kernel)
  int64_t capU[2] = {0, 0};
};

static void carve_select(Carver& c, SelectBufs& b, int64_t n, int L, int64_t m) {
  b.cap = n < m + 65536 ? n : m + 65536;
  b.P32 = c.take<float>(static_cast<int64_t>(L) * n);
  b.maxnorm2 = c.take<unsigned>(1);
  b.hist = c.take<unsigned>(static_cast<int64_t>(3) * L * 2 * kRadixBins);
  b.state = c.take<unsigned>(static_cast<int64_t>(L) * 2 * 4);
  b.cand = c.take<int>(static_cast<int64_t>(L) * 2 * b.cap);
  b.cval = c.take<double>(static_cast<int64_t>(L) * 2 * b.cap);
  b.ccount = c.take<unsigned>(static_cast<int64_t>(L) * 2);
  b.lists = c.take<int>(static_cast<int64_t>(L) * 2 * m);
  b.bitmap = c.take<unsigned>((n + 31) / 32);
  const int64_t capU = n < 2 * m * L ? n : 2 * m * L;
  b.uidx = c.take<long long>(capU > n ? n : (2 * m >= n ? n : capU));
  b.ucount = c.take<unsigned>(1 + kCompactBlocks);  // count, then compaction scratch
  b.overflow = c.take<int>(1);
  b.sfail = c.take<int>(1);
}

static size_t carve_est(Carver& c, EstWs& w, int64_t nA, int64_t nB, int D, int k, int64_t m, bool host_inputs,
                        int num_sms, bool certified = false) {
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
  w.mom.u0 = w.U64;  // row 0 of U is the centroid axis
  w.U32 = c.take<float>(static_cast<int64_t>(L) * D);
  w.lam = c.take<double>(k > 0 ? k : 1);
  w.n_dirs = c.take<int>(1);
  w.n_dirs1 = c.take<int>(1);
  const int64_t n[2] = {nA, nB};
  for (int s = 0; s < 2; ++s) {
    carve_select(c, w.sel[s], n[s], L, m);
    w.capU[s] = (2 * m >= n[s]) ? n[s] : (n[s] < 2 * m * L ? n[s] : 2 * m * L);
    w.Xs[s] = c.take<float>(w.capU[s] * D);
    carve_set(c, w.ops[s], w.capU[s], D);
  }
  if (certified) {
    carve_set(c, w.full[0], nA, D);
    carve_set(c, w.full[1], nB, D);
  }
  w.rowmin = c.take<float>(w.capU[0] > w.capU[1] ? w.capU[0] : w.capU[1]);
  w.colmin = c.take<float>(w.capU[0] > w.capU[1] ? w.capU[0] : w.capU[1]);
  w.keys = c.take<unsigned long long>(2);
  w.nn_d = c.take<double>(2);
  w.nn_j = c.take<long long>(2);
  w.blk_d = c.take<double>(kNNBlocks);
  w.blk_j = c.take<long long>(kNNBlocks);
  w.bad = c.take<int>(1);
  w.centre = c.take<double>(2 * static_cast<int64_t>(D));
  w.status = c.take<unsigned>(kStatusWords);
  w.res = c.take<EstResultDev>(1);
  return c.off;
}

size_t estimate_workspace_bytes(int64_t nA, int64_t nB, int D, int k, int64_t m, bool host_inputs,
                                bool certified) {
  Carver c{nullptr, 0, 0, true};
  EstWs w;
  return carve_est(c, w, nA, nB, D, k, m, host_inputs, 148, certified);
}

}  // namespace prohd

int prohd_run(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D, int32_t k,
              int64_t m, const double* dirs_in, int32_t n_dirs_in, prohd_est* out, double* dirs_out,
              int64_t* idxA_out, int64_t* idxB_out, int mode, const int64_t* counts) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (out == nullptr) return fail(ctx, PROHD_E_INVALID, "null output");
  if ((rc = check_sets(ctx, A, nA, B, nB, D))) return rc;
  if (k < 0 || k > D) return fail(ctx, PROHD_E_INVALID, "k must satisfy 0 <= k <= D (k=%d, D=%d)", k, D);
  if (m < 1) return fail(ctx, PROHD_E_INVALID, "m must be >= 1 (m=%lld)", static_cast<long long>(m));
  if (dirs_in == nullptr && k > 0 && D > 512)
    return fail(ctx, PROHD_E_NOTIMPL, "the device eigen-solver supports D <= 512 (D=%d)", D);
  if (m > 0x7FFFFFFFLL) return fail(ctx, PROHD_E_INVALID, "m too large");
  const int L = k + 1;
  call_begin(ctx);
  const bool host_in = !(is_device_ptr(A) && is_device_ptr(B));
  Carver dry{nullptr, 0, 0, true};
  EstWs tmp;
  const bool certified = mode == 1;
  const size_t need = carve_est(dry, tmp, nA, nB, D, k, m, host_in, ctx->num_sms, certified);
  if (ctx->ws == nullptr || ctx->ws_bytes < need)
    return fail(ctx, PROHD_E_WORKSPACE, "workspace too small: need %zu bytes, have %zu", need, ctx->ws_bytes);
  Carver c{ctx->ws, 0, ctx->ws_bytes, false};
  EstWs w;
  carve_est(c, w, nA, nB, D, k, m, host_in, ctx->num_sms, certified);
  bool hi;
  if ((rc = stage_inputs(ctx, A, nA, B, nB, D, w.stageA, w.stageB, hi))) return rc;
  // the second stream of the selection chains, created outside any capture
  if (ctx->aux == nullptr) {
    CK(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
  }
  // CUDA-graph replay (api_common.cuh graphed()) of the two stream-ordered stretches of the call:
  // steps 1-3 up to the status read, and step 4 up to the result read. Used for the plain
  // estimate on device inputs without tracing; the work runs on the library's capture stream,
  // ordered after and before the caller's stream by events.
  const bool use_graph = dirs_in == nullptr && counts == nullptr && !certified && !host_in && !ctx->timing &&
                         opt(OPT_GRAPH) != 0;
  if (use_graph && (rc = ensure_gstream(ctx))) return rc;
  GraphStream swap_guard(ctx, use_graph);
  cudaStream_t st = ctx->stream;
  auto make_key = [&](int phase, int i8, int64_t uc0, int64_t uc1) {
    KeyBuf kk = graph_key(ctx, 100 + phase);
    kk.add(i8).add(A).add(B).add(nA).add(nB).add(m).add(uc0).add(uc1).add(D).add(k);
    return kk.b;
  };

  // ------------------------------------------------------------ step 1: directions
  // moments on the int8 tensor cores where planned (k_gram_i8.cu), else the fp64 DMMA Gram;
  // if the int8 pass saw a value outside its sampled fixed-point range (checked at the host
  // sync after the selection), steps 1-3 rerun with the DMMA Gram
  const MomentsPlan mp = dirs_in == nullptr ? plan_moments(nA, nB, D, ctx->num_sms) : MomentsPlan{};
  auto directions = [&](bool use_i8) -> int {
    if (dirs_in == nullptr) {
      int t0 = tmark(ctx);
      CK(launch_shift(A, nA, B, nB, D, w.mom.s, st));
      if (use_i8) CK(cudaMemsetAsync(w.mom.i8ovf, 0, sizeof(unsigned), st));
      CK(launch_moments_partial(mp, A, nA, B, nB, D, w.mom, st, use_i8));
      CK(launch_moments_finalize(nA, nB, D, w.mom, st));
      tspan(ctx, PH_MOMENTS, t0);
      if (k > 0) {
        t0 = tmark(ctx);
        CK(launch_eigen_topk(w.mom.C, D, k, w.V, w.Xe, w.U64, w.U32, w.lam, w.n_dirs, st));
        tspan(ctx, PH_EIGEN, t0);
      } else {
        CK(launch_set_int(w.n_dirs, 1, st));
      }
      CK(launch_dirs_to_f32(w.U64, w.U32, L, D, st));
    } else {
      CK(cudaMemcpyAsync(w.U64, dirs_in, sizeof(double) * n_dirs_in * D, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(w.n_dirs, &n_dirs_in, sizeof(int), cudaMemcpyHostToDevice, st));
      CK(launch_dirs_to_f32(w.U64, w.U32, L, D, st));
    }
    return PROHD_OK;
  };
  bool use_i8 = dirs_in == nullptr && mp.i8;

  // ------------------------------------------------------------ steps 2-3: projection, selection, union
  const float* X[2] = {A, B};
  const int64_t n[2] = {nA, nB};
  unsigned ucount[2];
  int ndirs = 0, ovf[2] = {0, 0};
  unsigned maxn[2];
  unsigned i8ovf = 0;
  double eps[2] = {0.0, 0.0};
  bool sampled[2] = {false, false};
  int64_t msel[2] = {m, m};
  int sfail[2] = {0, 0};
  auto enqueue_select = [&]() -> int {
    sampled[0] = sampled[1] = false;
    const int t_sel = tmark(ctx);
    // set B's chain runs on the context's second stream, set A's on the caller's: the low-occupancy
    // tail of one set's selection (collect, re-rank, compaction) overlaps the other's projection
    if (counts && L > 1) CK(launch_minus_one(w.n_dirs, w.n_dirs1, st));  // shared by both sets
    CK(cudaEventRecord(ctx->ev_fork, st));
    CK(cudaStreamWaitEvent(ctx->aux, ctx->ev_fork, 0));
    // the chains are enqueued by a helper so that an error in either still joins the aux stream
    // back into the caller's before returning (no kernel of this call is left unordered against
    // the caller's stream and workspace)
    auto enqueue_chains = [&]() -> cudaError_t {
      for (int s = 0; s < 2; ++s) {
        // projections run for every point (also when 2m >= n) so non-finite input is always detected
        cudaStream_t sst = s == 0 ? st : ctx->aux;
        SelectBufs& b = w.sel[s];
        const int64_t m0 = counts ? counts[2 * s] : m;      // centroid axis
        const int64_t m1 = counts ? counts[2 * s + 1] : m;  // principal directions
        const bool all = 2 * m0 >= n[s] || (L > 1 && 2 * m1 >= n[s]);
        cudaError_t e;
        if (all) {
          if ((e = launch_select(X[s], n[s], D, w.U64, w.U32, L, w.n_dirs, 1, b, sst)) != cudaSuccess) return e;
          if ((e = launch_iota(b.uidx, b.ucount, n[s], sst)) != cudaSuccess) return e;
        } else if (m0 == m1 || L == 1) {
          // sampled-threshold K4 where it applies (certification failures rerun the radix path
          // after the host sync below), else the radix K4
          bool used = false;
          if ((e = launch_select_sampled(X[s], n[s], D, w.U64, w.U32, L, w.n_dirs, m0, b, sst, &eps[s], &used)) !=
              cudaSuccess)
            return e;
          sampled[s] = used;
          msel[s] = m0;
          if (!used &&
              (e = launch_select(X[s], n[s], D, w.U64, w.U32, L, w.n_dirs, m0, b, sst, true, true, &eps[s])) !=
                  cudaSuccess)
            return e;
        } else {  // two direction groups with different per-tail counts, one shared union bitmap
          // the groups share the projection buffer, so each group's overflow fallback runs right
          // after it (device-side no-op unless a list overflowed)
          if ((e = launch_select(X[s], n[s], D, w.U64, w.U32, 1, w.n_dirs, m0, b, sst, true, false, &eps[s])) !=
              cudaSuccess)
            return e;
          if ((e = launch_select_fallback(X[s], n[s], D, w.U64, 1, w.n_dirs, m0, b, eps[s], sst, false)) != cudaSuccess)
            return e;
          if ((e = launch_select(X[s], n[s], D, w.U64 + D, w.U32 + D, L - 1, w.n_dirs1, m1, b, sst, false, true,
                                 &eps[s])) != cudaSuccess)
            return e;
          if ((e = launch_select_fallback(X[s], n[s], D, w.U64 + D, L - 1, w.n_dirs1, m1, b, eps[s], sst, true)) !=
              cudaSuccess)
            return e;
        }
      }
      return cudaSuccess;
    };
    const cudaError_t e_chain = enqueue_chains();
    CK(cudaEventRecord(ctx->ev_join, ctx->aux));
    CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
    CK(e_chain);
    tspan(ctx, PH_SELECT, t_sel);
    return PROHD_OK;
  };
  // every value the host needs after the selection, packed on the device (one D2H copy)
  auto pack_status = [&](bool with_sfail) -> int {
    StatusSrc src{{w.sel[0].ucount, w.sel[1].ucount}, {w.sel[0].overflow, w.sel[1].overflow},
                  {w.sel[0].maxnorm2, w.sel[1].maxnorm2}, w.n_dirs, use_i8 ? w.mom.i8ovf : nullptr,
                  {with_sfail && sampled[0] ? w.sel[0].sfail : nullptr,
                   with_sfail && sampled[1] ? w.sel[1].sfail : nullptr}};
    CK(launch_pack_status(src, w.status, st));
    return PROHD_OK;
  };
  auto read_status = [&]() -> int {
    unsigned h[kStatusWords];
    CK(cudaMemcpyAsync(h, w.status, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int q = 0; q < 2; ++q) {
      ucount[q] = h[q];
      ovf[q] = static_cast<int>(h[2 + q]);
      maxn[q] = h[4 + q];
      sfail[q] = static_cast<int>(h[8 + q]);
    }
    ndirs = static_cast<int>(h[6]);
    i8ovf = h[7];
    return PROHD_OK;
  };
  // steps 1-3 as one stream-ordered stretch (graph-captured when use_graph)
  auto steps123 = [&]() -> int {
    int r2;
    CK(cudaMemsetAsync(w.bad, 0, sizeof(int), st));
    CK(cudaMemsetAsync(w.U64, 0, sizeof(double) * L * D, st));
    if ((r2 = directions(use_i8))) return r2;
    if ((r2 = enqueue_select())) return r2;
    return pack_status(true);
  };
  auto select_and_read = [&]() -> int {
    if (use_graph) {
      struct {
        double eps[2];
        int64_t msel[2];
        bool sampled[2];
      } hv;
      std::memset(&hv, 0, sizeof hv);
      const int r2 = graphed(ctx, make_key(1, use_i8 ? 1 : 0, 0, 0), &hv, sizeof hv, [&]() -> int {
        const int r3 = steps123();
        for (int q = 0; q < 2; ++q) {
          hv.eps[q] = eps[q];
          hv.msel[q] = msel[q];
          hv.sampled[q] = sampled[q];
        }
        return r3;
      });
      if (r2) return r2;
      for (int q = 0; q < 2; ++q) {
        eps[q] = hv.eps[q];
        msel[q] = hv.msel[q];
        sampled[q] = hv.sampled[q];
      }
    } else {
      const int r2 = steps123();
      if (r2) return r2;
    }
    if ((rc = read_status())) return rc;
    if (sfail[0] || sfail[1]) {
      // a sampled threshold could not be certified for some list (ties or a sample far off the
      // tail): the radix K4 for that set, from the projections again
      for (int s = 0; s < 2; ++s)
        if (sfail[s])
          CK(launch_select(X[s], n[s], D, w.U64, w.U32, L, w.n_dirs, msel[s], w.sel[s], st, true, true, &eps[s]));
      if ((rc = pack_status(false))) return rc;
      if ((rc = read_status())) return rc;
    }
    return PROHD_OK;
  };
  if ((rc = select_and_read())) return rc;
  if (use_i8 && i8ovf) {  // a value outside the int8 Gram's range (non-finite input): rerun on the DMMA Gram
    use_i8 = false;
    if ((rc = select_and_read())) return rc;
  }
  for (int s = 0; s < 2; ++s) {
    float f;
    std::memcpy(&f, &maxn[s], 4);
    if (!std::isfinite(f)) return fail(ctx, PROHD_E_DATA, "non-finite input coordinate (or squared norm overflow)");
  }
  const bool two_groups = counts && L > 1 && counts[0] != counts[1];
  if ((ovf[0] || ovf[1]) && !two_groups) {
    // a guard band held more candidates than the buffer (massive ties at the m-th value): exact
    // streaming band select for the affected lists, then the union again (rare path)
    for (int s = 0; s < 2; ++s)
      if (ovf[s]) CK(launch_select_fallback(X[s], n[s], D, w.U64, L, w.n_dirs, m, w.sel[s], eps[s], st, true));
    unsigned uc2[2];
    CK(cudaMemcpyAsync(&uc2[0], w.sel[0].ucount, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&uc2[1], w.sel[1].ucount, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ucount[0] = uc2[0];
    ucount[1] = uc2[1];
  }
  if (ucount[0] < 1 || ucount[1] < 1 || ucount[0] > w.capU[0] || ucount[1] > w.capU[1])
    return fail(ctx, PROHD_E_INTERNAL, "bad union sizes %u %u", ucount[0], ucount[1]);

  // ------------------------------------------------------------ step 4: exact HD on the subsets
  auto step4 = [&]() -> int {
    int r2;
    const int t_sub = tmark(ctx);
    for (int s = 0; s < 2; ++s) CK(launch_gather(X[s], D, w.sel[s].uidx, w.sel[s].ucount, ucount[s], w.Xs[s], st));
    // one common centre for every operand of the subset HD: centre(A_sel, B_sel) (symmetric;
    // the sharded driver computes the same from the all-gathered subsets)
    CK(launch_centre(w.Xs[0], ucount[0], w.Xs[1], ucount[1], D, w.centre, st));
    if (!certified && (r2 = prep_pair(ctx, w.Xs[0], ucount[0], w.Xs[1], ucount[1], D, w.ops[0], w.ops[1], w.bad,
                                      w.centre)))
      return r2;
    ExactWs ew;
    ew.rowmin = w.rowmin;
    ew.colmin = w.colmin;
    ew.keys = w.keys;
    ew.nn_d = w.nn_d;
    ew.nn_j = w.nn_j;
    ew.blk_d = w.blk_d;
    ew.blk_j = w.blk_j;
    if (!certified) {
      if ((r2 = bidir_on_ops(ctx, w.ops[0], w.ops[1], D, ew))) return r2;  // Alg. 3 line 6, both directions
    } else {
      // certified mode (SPEC.md:279 subset-full): rows of each subset against the FULL other set
      // two pairs, each prepared together: (A_sel, B) and (B_sel, A)
      if ((r2 = prep_pair(ctx, w.Xs[0], ucount[0], B, nB, D, w.ops[0], w.full[1], w.bad, w.centre))) return r2;
      if ((r2 = prep_pair(ctx, w.Xs[1], ucount[1], A, nA, D, w.ops[1], w.full[0], w.bad, w.centre))) return r2;
      if ((r2 = directed_on_ops(ctx, w.ops[0], w.full[1], D, ew, 0))) return r2;
      if ((r2 = directed_on_ops(ctx, w.ops[1], w.full[0], D, ew, 1))) return r2;
    }
    tspan(ctx, PH_SUBSET, t_sub);
    // witnesses mapped to original indices on the device (one copy of the result below)
    CK(launch_pack_result(w.keys, w.nn_d, w.nn_j, w.sel[0].uidx, w.sel[1].uidx, !certified, w.res, st));
    return PROHD_OK;
  };
  if (use_graph)
    rc = graphed(ctx, make_key(2, use_i8 ? 1 : 0, ucount[0], ucount[1]), nullptr, 0, step4);
  else
    rc = step4();
  if (rc) return rc;
  EstResultDev res;
  CK(cudaMemcpyAsync(&res, w.res, sizeof res, cudaMemcpyDeviceToHost, st));
  if (idxA_out)
    CK(cudaMemcpyAsync(idxA_out, w.sel[0].uidx, sizeof(long long) * ucount[0], cudaMemcpyDeviceToHost, st));
  if (idxB_out)
    CK(cudaMemcpyAsync(idxB_out, w.sel[1].uidx, sizeof(long long) * ucount[1], cudaMemcpyDeviceToHost, st));
  if (dirs_out != nullptr)
    CK(cudaMemcpyAsync(dirs_out, w.U64, sizeof(double) * L * D, cudaMemcpyDeviceToHost, st));
  call_end(ctx);
  CK(cudaStreamSynchronize(st));
  call_collect(ctx);

  fill_directed(&out->ab, res.key[0], res.d2[0], res.b[0]);
  fill_directed(&out->ba, res.key[1], res.d2[1], res.b[1]);
  out->ab.a = res.a[0];  // original indices (a in the first argument, b in the second)
  out->ba.a = res.a[1];
  out->value = out->ab.dist2 >= out->ba.dist2 ? out->ab.dist : out->ba.dist;
  out->size_a = ucount[0];
  out->size_b = ucount[1];
  out->n_dirs = ndirs;
  out->_pad = 0;
  return PROHD_OK;
}

// Test hook (include/prohd.h prohd_covariance): step 1a of prohd_estimate alone.
extern "C" int prohd_covariance(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D,
                                double* mu_out, double* C_out, int32_t* path_out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (mu_out == nullptr || C_out == nullptr || path_out == nullptr) return fail(ctx, PROHD_E_INVALID, "null output");
  if ((rc = check_sets(ctx, A, nA, B, nB, D))) return rc;
  call_begin(ctx);
  const bool host_in = !(is_device_ptr(A) && is_device_ptr(B));
  Carver dry{nullptr, 0, 0, true};
  EstWs tmp;
  const size_t need = carve_est(dry, tmp, nA, nB, D, 0, 1, host_in, ctx->num_sms);
  if (ctx->ws == nullptr || ctx->ws_bytes < need)
    return fail(ctx, PROHD_E_WORKSPACE, "workspace too small: need %zu bytes, have %zu", need, ctx->ws_bytes);
  Carver c{ctx->ws, 0, ctx->ws_bytes, false};
  EstWs w;
  carve_est(c, w, nA, nB, D, 0, 1, host_in, ctx->num_sms);
  cudaStream_t st = ctx->stream;
  bool hi;
  if ((rc = stage_inputs(ctx, A, nA, B, nB, D, w.stageA, w.stageB, hi))) return rc;
  const MomentsPlan mp = plan_moments(nA, nB, D, ctx->num_sms);
  bool use_i8 = mp.i8;
  for (int attempt = 0; attempt < 2; ++attempt) {
    const int t0 = tmark(ctx);
    CK(launch_shift(A, nA, B, nB, D, w.mom.s, st));
    if (use_i8) CK(cudaMemsetAsync(w.mom.i8ovf, 0, sizeof(unsigned), st));
    CK(launch_moments_partial(mp, A, nA, B, nB, D, w.mom, st, use_i8));
    CK(launch_moments_finalize(nA, nB, D, w.mom, st));
    tspan(ctx, PH_MOMENTS, t0);
    unsigned ovf = 0;
    if (use_i8) CK(cudaMemcpyAsync(&ovf, w.mom.i8ovf, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!(use_i8 && ovf)) break;
    use_i8 = false;  // outside the int8 pass's sampled range: the fp64 DMMA Gram
  }
  CK(cudaMemcpyAsync(mu_out, w.mom.mu, sizeof(double) * D, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(C_out, w.mom.C, sizeof(double) * D * D, cudaMemcpyDeviceToHost, st));
  call_end(ctx);
  CK(cudaStreamSynchronize(st));
  call_collect(ctx);
  *path_out = use_i8 ? 1 : 0;
  return PROHD_OK;
}
