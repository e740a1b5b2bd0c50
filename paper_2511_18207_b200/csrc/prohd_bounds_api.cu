// prohd_bounds_api.cu — C ABI of the f2 bound report.
#include "api_common.cuh"
#include "prohd_kernels.cuh"

#include <cmath>
#include <cstring>

extern "C" int prohd_bounds(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D,
                            const double* dirs, int32_t n_dirs, double* per_dir_out, double* summary_out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (dirs == nullptr || per_dir_out == nullptr || summary_out == nullptr)
    return fail(ctx, PROHD_E_INVALID, "null pointer");
  if ((rc = check_sets(ctx, A, nA, B, nB, D))) return rc;
  if (n_dirs < 1 || n_dirs > 32) return fail(ctx, PROHD_E_INVALID, "n_dirs must be in [1, 32]");
  call_begin(ctx);
  const int L = n_dirs;
  const bool host_in = !(is_device_ptr(A) && is_device_ptr(B));
  const BoundsPlan bp = plan_bounds(nA, nB, L);
  const int64_t nmax = nA > nB ? nA : nB;
  auto carve = [&](Carver& c, float*& stA, float*& stB, double*& U64, float*& U32, double*& part, double*& mu,
                   BoundsBufs& b) {
    stA = stB = nullptr;
    if (host_in) {
      stA = c.take<float>(nA * D);
      stB = c.take<float>(nB * D);
    }
    U64 = c.take<double>(static_cast<int64_t>(L) * D);
    U32 = c.take<float>(static_cast<int64_t>(L) * D);
    part = c.take<double>(static_cast<int64_t>(2 * kMeanParts) * D);
    mu = c.take<double>(D);
    b.keysA = c.take<unsigned>(static_cast<int64_t>(L) * nA);
    b.keysB = c.take<unsigned>(static_cast<int64_t>(L) * nB);
    b.sortA = c.take<unsigned>(static_cast<int64_t>(L) * nA);
    b.sortB = c.take<unsigned>(static_cast<int64_t>(L) * nB);
    b.tmp = c.take<unsigned>(static_cast<int64_t>(L) * nmax);
    b.counts = c.take<unsigned>(bp.count_words);
    b.delta2 = c.take<unsigned long long>(2 * L);
    b.hu = c.take<unsigned long long>(2 * L);
    return c.off;
  };
  float *stA, *stB, *U32;
  double *U64, *part, *mu;
  BoundsBufs b{};
  Carver dry{nullptr, 0, 0, true};
  const size_t need = carve(dry, stA, stB, U64, U32, part, mu, b);
  if (ctx->ws == nullptr || ctx->ws_bytes < need)
    return fail(ctx, PROHD_E_WORKSPACE, "workspace too small: need %zu bytes, have %zu", need, ctx->ws_bytes);
  Carver c{ctx->ws, 0, ctx->ws_bytes, false};
  carve(c, stA, stB, U64, U32, part, mu, b);
  cudaStream_t st = ctx->stream;
  bool hi;
  if ((rc = stage_inputs(ctx, A, nA, B, nB, D, stA, stB, hi))) return rc;
  CK(cudaMemcpyAsync(U64, dirs, sizeof(double) * L * D, cudaMemcpyHostToDevice, st));
  CK(launch_dirs_to_f32(U64, U32, L, D, st));
  const int t0 = tmark(ctx);
  CK(launch_union_mean(A, nA, B, nB, D, part, mu, st));
  CK(launch_bounds(A, nA, B, nB, D, U32, L, mu, b, st));
  tspan(ctx, PH_SELECT, t0);
  unsigned long long d2[64], hu[64];
  CK(cudaMemcpyAsync(d2, b.delta2, sizeof(unsigned long long) * 2 * L, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hu, b.hu, sizeof(unsigned long long) * 2 * L, cudaMemcpyDeviceToHost, st));
  call_end(ctx);
  CK(cudaStreamSynchronize(st));
  call_collect(ctx);
  double HU = 0.0, mind = INFINITY;
  for (int l = 0; l < L; ++l) {
    double v[4];
    std::memcpy(&v[0], &d2[2 * l], 8);
    std::memcpy(&v[1], &d2[2 * l + 1], 8);
    std::memcpy(&v[2], &hu[l], 8);
    std::memcpy(&v[3], &hu[L + l], 8);
    v[0] = std::sqrt(v[0]);
    v[1] = std::sqrt(v[1]);
    if (!std::isfinite(v[0]) || !std::isfinite(v[1])) return fail(ctx, PROHD_E_DATA, "non-finite input");
    for (int q = 0; q < 4; ++q) per_dir_out[4 * l + q] = v[q];
    HU = std::fmax(HU, std::fmax(v[2], v[3]));
    mind = std::fmin(mind, std::fmin(v[0], v[1]));
  }
  summary_out[0] = HU;
  summary_out[1] = mind;
  summary_out[2] = HU + 2.0 * mind;  // Eq. (4): H_U <= H <= H_U + 2 min delta
  return PROHD_OK;
}
