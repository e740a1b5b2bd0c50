// prohd_api.cu — the C ABI declared in include/prohd.h.
//
// Orchestration only: argument validation, workspace carving, host->device
// staging of host inputs, TMA descriptor creation and the kernel launch
// sequence. Every arithmetic step of the path runs in the kernels (k_*.cu).
#include "../../include/prohd.h"
#include "api_common.cuh"
#include "prohd_kernels.cuh"
#include "prohd_steps.cuh"

#include <algorithm>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

// ================================================================== ABI
extern "C" {

const char* prohd_version(void) { return "prohd-b200 0.1 sm_100a"; }

static const char* const kOptNames[prohd::OPT_COUNT] = {
    "k6_variant", "k6_split3", "k6_bidir_2a", "k6_splits_2x", "k1_path", "k1_ctas",
    "k1_cs_sms",  "k1_beta_milli", "shift", "k3_simt", "eig_stop", "eig_cl", "k1_ablate",
    "k4_sampled", "k1_i8_ctas", "graph"};

int prohd_set_option(const char* name, int64_t value) {
  if (name == nullptr) return PROHD_E_INVALID;
  for (int i = 0; i < prohd::OPT_COUNT; ++i)
    if (std::strcmp(name, kOptNames[i]) == 0) {
      prohd::option_table()[i].store(value < 0 ? -1 : value);
      return PROHD_OK;
    }
  return PROHD_E_INVALID;
}

int prohd_get_option(const char* name, int64_t* value) {
  if (name == nullptr || value == nullptr) return PROHD_E_INVALID;
  for (int i = 0; i < prohd::OPT_COUNT; ++i)
    if (std::strcmp(name, kOptNames[i]) == 0) {
      *value = prohd::option_table()[i].load();
      return PROHD_OK;
    }
  return PROHD_E_INVALID;
}

int prohd_launch_count(int64_t* out) {
  if (out == nullptr) return PROHD_E_INVALID;
  *out = static_cast<int64_t>(prohd::launch_counter().load());
  return PROHD_OK;
}

int prohd_create(int device, void* cuda_stream, prohd_ctx** out) {
  if (out == nullptr) return PROHD_E_INVALID;
  *out = nullptr;
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return PROHD_E_CUDA;
  if (prop.major != 10 || prop.minor != 0) return PROHD_E_DEVICE;
  prohd_ctx* c = new prohd_ctx();
  c->device = device;
  c->stream = static_cast<cudaStream_t>(cuda_stream);
  c->num_sms = prop.multiProcessorCount;
  *out = c;
  return PROHD_OK;
}

int prohd_destroy(prohd_ctx* ctx) {
  if (ctx == nullptr) return PROHD_OK;
  for (cudaEvent_t e : ctx->ev) cudaEventDestroy(e);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  for (auto& g : ctx->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (ctx->gstream) cudaStreamDestroy(ctx->gstream);
  if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
  if (ctx->ev_out) cudaEventDestroy(ctx->ev_out);
  delete ctx;
  return PROHD_OK;
}

int prohd_enable_timing(prohd_ctx* ctx, int on) {
  if (ctx == nullptr) return PROHD_E_INVALID;
  if (on && ctx->ev.empty()) {
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return fail(ctx, PROHD_E_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
    ctx->ev.resize(128);
    for (auto& ev : ctx->ev) {
      e = cudaEventCreate(&ev);
      if (e != cudaSuccess) return fail(ctx, PROHD_E_CUDA, "cudaEventCreate: %s", cudaGetErrorString(e));
    }
  }
  ctx->timing = on != 0;
  return PROHD_OK;
}

int prohd_last_timings(const prohd_ctx* ctx, prohd_timings* out) {
  if (ctx == nullptr || out == nullptr) return PROHD_E_INVALID;
  *out = ctx->last;
  return PROHD_OK;
}

int prohd_set_stream(prohd_ctx* ctx, void* cuda_stream) {
  if (ctx == nullptr) return PROHD_E_INVALID;
  ctx->stream = static_cast<cudaStream_t>(cuda_stream);
  return PROHD_OK;
}

const char* prohd_last_error(const prohd_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

size_t prohd_workspace_bytes(int64_t nA, int64_t nB, int32_t D, int32_t k, int64_t m, uint32_t flags) {
  if (nA < 1 || nB < 1 || D < 1) return 0;
  Carver c{nullptr, 0, 0, true};
  ExactWs w;
  size_t exact = carve_exact(c, w, nA, nB, D, (flags & PROHD_WS_HOST_INPUTS) != 0);
  size_t est = estimate_workspace_bytes(nA, nB, D, k < 0 ? 0 : k, m < 1 ? 1 : m,
                                        (flags & PROHD_WS_HOST_INPUTS) != 0, (flags & PROHD_WS_CERTIFIED) != 0);
  return (exact > est ? exact : est) + 256;
}

int prohd_set_workspace(prohd_ctx* ctx, void* dptr, size_t bytes) {
  if (ctx == nullptr) return PROHD_E_INVALID;
  if (dptr != nullptr && (reinterpret_cast<uintptr_t>(dptr) & 255) != 0)
    return fail(ctx, PROHD_E_INVALID, "workspace must be 256-byte aligned");
  ctx->ws = static_cast<uint8_t*>(dptr);
  ctx->ws_bytes = dptr ? bytes : 0;
  return PROHD_OK;
}

// Common centre of the pair for K0 (translation invariance, no cancellation far from the
// origin): kCentreCols = centre(-, B) (the column set alone, so row shards of A on any
// number of GPUs prepare identical operands), kCentrePair = centre(A, B) (symmetric).
enum { kCentreCols = 0, kCentrePair = 1 };

static int exact_common(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D,
                        ExactWs& w, int centre_mode, const double* centre_in = nullptr) {
  int rc = enter(ctx);
  if (rc) return rc;
  if ((rc = check_sets(ctx, A, nA, B, nB, D))) return rc;
  call_begin(ctx);
  const bool host_in = !(is_device_ptr(A) && is_device_ptr(B));
  Carver dry{nullptr, 0, 0, true};
  ExactWs tmp;
  size_t need = carve_exact(dry, tmp, nA, nB, D, host_in);
  if (ctx->ws == nullptr || ctx->ws_bytes < need)
    return fail(ctx, PROHD_E_WORKSPACE, "workspace too small: need %zu bytes, have %zu", need, ctx->ws_bytes);
  Carver c{ctx->ws, 0, ctx->ws_bytes, false};
  carve_exact(c, w, nA, nB, D, host_in);
  bool hi;
  if ((rc = stage_inputs(ctx, A, nA, B, nB, D, w.stageA, w.stageB, hi))) return rc;
  CK(cudaMemsetAsync(w.bad, 0, sizeof(int), ctx->stream));
  if (centre_in != nullptr)
    CK(cudaMemcpyAsync(w.centre, centre_in, sizeof(double) * D, cudaMemcpyDefault, ctx->stream));
  else if (centre_mode == kCentrePair)
    CK(launch_centre(A, nA, B, nB, D, w.centre, ctx->stream));
  else
    CK(launch_centre(nullptr, 0, B, nB, D, w.centre, ctx->stream));
  if ((rc = prep_pair(ctx, A, nA, B, nB, D, w.A, w.B, w.bad, w.centre))) return rc;
  return PROHD_OK;
}

struct ExactHost {
  unsigned long long keys[2];
  double nn_d[2];
  long long nn_j[2];
  int bad;
};

// every result word in ONE device-to-host copy (pack_exact_kernel), then the single sync
static int fetch(prohd_ctx* ctx, const ExactWs& w, ExactHost& h, bool packed = false) {
  ExactResDev r;
  if (!packed)
    CK(launch_pack_exact(w.keys, w.nn_d, w.nn_j, w.bad, static_cast<ExactResDev*>(w.res), ctx->stream));
  CK(cudaMemcpyAsync(&r, w.res, sizeof r, cudaMemcpyDeviceToHost, ctx->stream));
  call_end(ctx);
  CK(cudaStreamSynchronize(ctx->stream));
  call_collect(ctx);
  for (int s = 0; s < 2; ++s) {
    h.keys[s] = r.key[s];
    h.nn_d[s] = r.d2[s];
    h.nn_j[s] = r.j[s];
  }
  h.bad = r.bad;
  if (h.bad) return fail(ctx, PROHD_E_DATA, "non-finite input coordinate (or squared norm overflow)");
  return PROHD_OK;
}

// directed_hd / hausdorff on device inputs without tracing: the whole enqueue (centre, K0, K6, K7,
// pack) replays a cached CUDA graph on the library's capture stream (api_common.cuh graphed(),
// prohd_estimate.cu); the host then reads one packed result.
static int exact_run(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D, bool bidir,
                     ExactHost& h) {
  int rc = enter(ctx);
  if (rc) return rc;
  if ((rc = check_sets(ctx, A, nA, B, nB, D))) return rc;
  const bool dev_in = is_device_ptr(A) && is_device_ptr(B);
  const bool use_graph = dev_in && !ctx->timing && opt(OPT_GRAPH) != 0;
  if (use_graph && (rc = ensure_gstream(ctx))) return rc;
  GraphStream gs(ctx, use_graph);
  ExactWs w;
  auto work = [&]() -> int {
    int r2 = exact_common(ctx, A, nA, B, nB, D, w, bidir ? kCentrePair : kCentreCols);
    if (r2) return r2;
    if ((r2 = bidir ? bidir_on_ops(ctx, w.A, w.B, D, w) : directed_on_ops(ctx, w.A, w.B, D, w, 0))) return r2;
    CK(launch_pack_exact(w.keys, w.nn_d, w.nn_j, w.bad, static_cast<ExactResDev*>(w.res), ctx->stream));
    return PROHD_OK;
  };
  if (use_graph) {
    KeyBuf kk = graph_key(ctx, bidir ? 2 : 1);
    kk.add(A).add(B).add(nA).add(nB).add(D);
    // exact_common's carve fills w inside the capture; on a replay it is not run, so carve here too
    Carver c{ctx->ws, 0, ctx->ws_bytes, false};
    if (ctx->ws != nullptr) {
      Carver dry{nullptr, 0, 0, true};
      ExactWs tmp;
      if (carve_exact(dry, tmp, nA, nB, D, false) <= ctx->ws_bytes) carve_exact(c, w, nA, nB, D, false);
    }
    call_begin(ctx);
    rc = graphed(ctx, kk.b, nullptr, 0, work);
  } else {
    rc = work();
  }
  if (rc) return rc;
  return fetch(ctx, w, h, true);
}

int directed_hd(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D,
                prohd_directed* out) {
  if (out == nullptr) return fail(ctx, PROHD_E_INVALID, "null output");
  ExactHost h;
  int rc = exact_run(ctx, A, nA, B, nB, D, false, h);
  if (rc) return rc;
  fill_directed(out, h.keys[0], h.nn_d[0], h.nn_j[0]);
  return PROHD_OK;
}

int hausdorff(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D, prohd_hd* out) {
  if (out == nullptr) return fail(ctx, PROHD_E_INVALID, "null output");
  ExactHost h;
  int rc = exact_run(ctx, A, nA, B, nB, D, true, h);  // one fused sweep for both directions
  if (rc) return rc;
  fill_directed(&out->ab, h.keys[0], h.nn_d[0], h.nn_j[0]);
  fill_directed(&out->ba, h.keys[1], h.nn_d[1], h.nn_j[1]);
  out->value = out->ab.dist2 >= out->ba.dist2 ? out->ab.dist : out->ba.dist;
  return PROHD_OK;
}

int hausdorff_minima(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D,
                     float* rowmin_dev, float* colmin_dev, prohd_hd* out) {
  if (out == nullptr || rowmin_dev == nullptr || colmin_dev == nullptr || !is_device_ptr(rowmin_dev) ||
      !is_device_ptr(colmin_dev))
    return fail(ctx, PROHD_E_INVALID, "null output or host minima pointers");
  ExactWs w;
  int rc = exact_common(ctx, A, nA, B, nB, D, w, kCentrePair);
  if (rc) return rc;
  if ((rc = bidir_on_ops(ctx, w.A, w.B, D, w))) return rc;
  CK(cudaMemcpyAsync(rowmin_dev, w.rowmin, sizeof(float) * nA, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(colmin_dev, w.colmin, sizeof(float) * nB, cudaMemcpyDeviceToDevice, ctx->stream));
  ExactHost h;
  if ((rc = fetch(ctx, w, h))) return rc;
  fill_directed(&out->ab, h.keys[0], h.nn_d[0], h.nn_j[0]);
  fill_directed(&out->ba, h.keys[1], h.nn_d[1], h.nn_j[1]);
  out->value = out->ab.dist2 >= out->ba.dist2 ? out->ab.dist : out->ba.dist;
  return PROHD_OK;
}

int directed_hd_rowmin(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D,
                       float* rowmin_dev) {
  if (rowmin_dev == nullptr || !is_device_ptr(rowmin_dev))
    return fail(ctx, PROHD_E_INVALID, "rowmin_dev must be a device pointer");
  ExactWs w;
  int rc = exact_common(ctx, A, nA, B, nB, D, w, kCentreCols);
  if (rc) return rc;
  if ((rc = run_dist(ctx, w.A, w.B, D, rowmin_dev))) return rc;
  ExactHost h{};
  CK(cudaMemcpyAsync(&h.bad, w.bad, sizeof h.bad, cudaMemcpyDeviceToHost, ctx->stream));
  call_end(ctx);
  CK(cudaStreamSynchronize(ctx->stream));
  call_collect(ctx);
  if (h.bad) return fail(ctx, PROHD_E_DATA, "non-finite input coordinate");
  return PROHD_OK;
}

int directed_hd_local(prohd_ctx* ctx, const float* A_local, int64_t nA_local, int64_t row_offset,
                      const float* B, int64_t nB, int32_t D, const double* centre, uint64_t* key_out) {
  if (key_out == nullptr) return fail(ctx, PROHD_E_INVALID, "null key_out");
  if (row_offset < 0) return fail(ctx, PROHD_E_INVALID, "negative row_offset");
  if (row_offset + nA_local > 0x7FFFFF00LL) return fail(ctx, PROHD_E_INVALID, "global row too large");
  ExactWs w;
  int rc = exact_common(ctx, A_local, nA_local, B, nB, D, w, kCentreCols, centre);
  if (rc) return rc;
  if ((rc = run_dist(ctx, w.A, w.B, D, w.rowmin))) return rc;
  CK(launch_rowmax_key(w.rowmin, nA_local, row_offset, &w.keys[0], ctx->stream));
  ExactHost h{};
  CK(cudaMemcpyAsync(h.keys, w.keys, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&h.bad, w.bad, sizeof h.bad, cudaMemcpyDeviceToHost, ctx->stream));
  call_end(ctx);
  CK(cudaStreamSynchronize(ctx->stream));
  call_collect(ctx);
  if (h.bad) return fail(ctx, PROHD_E_DATA, "non-finite input coordinate");
  *key_out = h.keys[0];
  return PROHD_OK;
}

int prohd_centre(prohd_ctx* ctx, const float* X, int64_t nX, const float* Y, int64_t nY, int32_t D,
                 double* centre_out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (centre_out == nullptr) return fail(ctx, PROHD_E_INVALID, "null centre_out");
  if (D < 1 || nX < 0 || nY < 0 || nX + nY < 1) return fail(ctx, PROHD_E_INVALID, "bad sizes");
  if ((nX > 0 && X == nullptr) || (nY > 0 && Y == nullptr)) return fail(ctx, PROHD_E_INVALID, "null input");
  const int64_t cx = nX < 4096 ? nX : 4096, cy = nY < 4096 ? nY : 4096;
  if ((cx > 0 && !is_device_ptr(X)) || (cy > 0 && !is_device_ptr(Y)))
    return fail(ctx, PROHD_E_INVALID, "prohd_centre takes device inputs");
  Carver dry{nullptr, 0, 0, true};
  dry.take<double>(2 * static_cast<int64_t>(D));
  if (ctx->ws == nullptr || ctx->ws_bytes < dry.off)
    return fail(ctx, PROHD_E_WORKSPACE, "workspace too small: need %zu bytes, have %zu", dry.off, ctx->ws_bytes);
  Carver c{ctx->ws, 0, ctx->ws_bytes, false};
  double* cbuf = c.take<double>(2 * static_cast<int64_t>(D));
  call_begin(ctx);
  CK(launch_centre(X, cx, Y, cy, D, cbuf, ctx->stream));
  CK(cudaMemcpyAsync(centre_out, cbuf, sizeof(double) * D, cudaMemcpyDefault, ctx->stream));
  call_end(ctx);
  CK(cudaStreamSynchronize(ctx->stream));
  call_collect(ctx);
  return PROHD_OK;
}

int prohd_project(prohd_ctx* ctx, const float* X, int64_t n, int32_t D, const double* dirs, int32_t L,
                  float* proj_out, double* eps_out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (X == nullptr || dirs == nullptr || proj_out == nullptr || eps_out == nullptr)
    return fail(ctx, PROHD_E_INVALID, "null pointer");
  if (n < 1 || D < 1 || L < 1 || L > 32) return fail(ctx, PROHD_E_INVALID, "bad sizes");
  if (!is_device_ptr(X) || !is_device_ptr(dirs) || !is_device_ptr(proj_out))
    return fail(ctx, PROHD_E_INVALID, "prohd_project takes device pointers");
  if ((rc = check_aligned(ctx, X, D, "X"))) return rc;
  Carver dry{nullptr, 0, 0, true};
  dry.take<float>(static_cast<int64_t>(L) * D);
  dry.take<unsigned>(1);
  if (ctx->ws == nullptr || ctx->ws_bytes < dry.off)
    return fail(ctx, PROHD_E_WORKSPACE, "workspace too small: need %zu bytes, have %zu", dry.off, ctx->ws_bytes);
  Carver c{ctx->ws, 0, ctx->ws_bytes, false};
  float* U32 = c.take<float>(static_cast<int64_t>(L) * D);
  unsigned* mx = c.take<unsigned>(1);
  double coef = 0.0;
  unsigned mxh = 0;
  call_begin(ctx);
  CK(cudaMemsetAsync(mx, 0, sizeof(unsigned), ctx->stream));
  CK(launch_dirs_to_f32(dirs, U32, L, D, ctx->stream));
  CK(launch_project(X, n, D, U32, L, proj_out, mx, ctx->stream, &coef));
  CK(cudaMemcpyAsync(&mxh, mx, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
  call_end(ctx);
  CK(cudaStreamSynchronize(ctx->stream));
  call_collect(ctx);
  float m2;
  memcpy(&m2, &mxh, sizeof(m2));
  *eps_out = coef * std::sqrt(static_cast<double>(m2)) * 1.0625;
  return PROHD_OK;
}

int directed_hd_witness(prohd_ctx* ctx, const float* a, const float* B, int64_t nB, int32_t D,
                        prohd_directed* out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (a == nullptr || out == nullptr) return fail(ctx, PROHD_E_INVALID, "null pointer");
  if ((rc = check_sets(ctx, a, 1, B, nB, D))) return rc;
  Carver dry{nullptr, 0, 0, true};
  ExactWs tmp;
  const bool host_in = !(is_device_ptr(a) && is_device_ptr(B));
  size_t need = carve_exact(dry, tmp, 1, nB, D, host_in);
  if (ctx->ws == nullptr || ctx->ws_bytes < need)
    return fail(ctx, PROHD_E_WORKSPACE, "workspace too small: need %zu bytes, have %zu", need, ctx->ws_bytes);
  Carver c{ctx->ws, 0, ctx->ws_bytes, false};
  ExactWs w;
  carve_exact(c, w, 1, nB, D, host_in);
  bool hi;
  if ((rc = stage_inputs(ctx, a, 1, B, nB, D, w.stageA, w.stageB, hi))) return rc;
  CK(launch_nn64(a, B, nB, D, w.blk_d, w.blk_j, kNNBlocks, &w.nn_d[0], &w.nn_j[0], ctx->stream));
  double d;
  long long j;
  CK(cudaMemcpyAsync(&d, w.nn_d, sizeof d, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&j, w.nn_j, sizeof j, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  out->b = j;
  out->dist2 = d;
  out->dist = std::sqrt(d);
  out->dist2_tc = NAN;
  return PROHD_OK;
}

int prohd_estimate(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D, int32_t k,
                   int64_t m, prohd_est* out, double* dirs_out, int64_t* idxA_out, int64_t* idxB_out) {
  return prohd_run(ctx, A, nA, B, nB, D, k, m, nullptr, 0, out, dirs_out, idxA_out, idxB_out);
}

int prohd_estimate_certified(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D,
                             int32_t k, int64_t m, prohd_est* out, double* dirs_out, int64_t* idxA_out,
                             int64_t* idxB_out) {
  return prohd_run(ctx, A, nA, B, nB, D, k, m, nullptr, 0, out, dirs_out, idxA_out, idxB_out, 1);
}

int prohd_estimate_alpha(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D,
                         double alpha, prohd_est* out, double* dirs_out, int64_t* idxA_out, int64_t* idxB_out) {
  if (!(alpha > 0.0 && alpha < 1.0)) return fail(ctx, PROHD_E_INVALID, "alpha must be in (0, 1)");
  if (D < 1 || nA < 1 || nB < 1) return fail(ctx, PROHD_E_INVALID, "bad sizes");
  int k = static_cast<int>(std::floor(std::sqrt(static_cast<double>(D))));  // Alg. 3 l.1: m = floor(sqrt D)
  if (k < 1) k = 1;
  if (k > D) k = D;
  const double ap = alpha / k;  // alpha' = alpha / m
  int64_t cnt[4];
  const int64_t n[2] = {nA, nB};
  for (int s = 0; s < 2; ++s) {  // k_X = max{1, floor(alpha n_X)}
    cnt[2 * s] = std::max<int64_t>(1, static_cast<int64_t>(std::floor(alpha * n[s])));
    cnt[2 * s + 1] = std::max<int64_t>(1, static_cast<int64_t>(std::floor(ap * n[s])));
  }
  const int64_t m = std::max(std::max(cnt[0], cnt[1]), std::max(cnt[2], cnt[3]));
  return prohd_run(ctx, A, nA, B, nB, D, k, m, nullptr, 0, out, dirs_out, idxA_out, idxB_out, 0, cnt);
}

int hausdorff_subsets(prohd_ctx* ctx, const float* A, int64_t nA, const int64_t* idxA, int64_t kA, const float* B,
                      int64_t nB, const int64_t* idxB, int64_t kB, int32_t D, prohd_hd* out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (out == nullptr || idxA == nullptr || idxB == nullptr) return fail(ctx, PROHD_E_INVALID, "null pointer");
  if ((rc = check_sets(ctx, A, nA, B, nB, D))) return rc;
  if (kA < 1 || kB < 1 || kA > nA || kB > nB) return fail(ctx, PROHD_E_INVALID, "bad subset sizes");
  // host copies of the index lists: validated, and used to map witnesses back
  std::vector<int64_t> ia(kA), ib(kB);
  CK(cudaMemcpy(ia.data(), idxA, sizeof(int64_t) * kA, cudaMemcpyDefault));
  CK(cudaMemcpy(ib.data(), idxB, sizeof(int64_t) * kB, cudaMemcpyDefault));
  for (int64_t v : ia)
    if (v < 0 || v >= nA) return fail(ctx, PROHD_E_INVALID, "idxA entry out of range");
  for (int64_t v : ib)
    if (v < 0 || v >= nB) return fail(ctx, PROHD_E_INVALID, "idxB entry out of range");
  call_begin(ctx);
  const bool host_in = !(is_device_ptr(A) && is_device_ptr(B));
  // workspace: staged inputs (if host) + gathered subsets + their operands + exact-HD scratch
  Carver dry{nullptr, 0, 0, true};
  float* stA = nullptr;
  float* stB = nullptr;
  auto carve = [&](Carver& c, ExactWs& w, float*& xa, float*& xb, long long*& dia, long long*& dib) {
    if (host_in) {
      stA = c.take<float>(nA * D);
      stB = c.take<float>(nB * D);
    }
    xa = c.take<float>(kA * D);
    xb = c.take<float>(kB * D);
    dia = c.take<long long>(kA);
    dib = c.take<long long>(kB);
    return carve_exact(c, w, kA, kB, D, false);
  };
  ExactWs tmp;
  float *xa, *xb;
  long long *dia, *dib;
  const size_t need = carve(dry, tmp, xa, xb, dia, dib);
  if (ctx->ws == nullptr || ctx->ws_bytes < need)
    return fail(ctx, PROHD_E_WORKSPACE, "workspace too small: need %zu bytes, have %zu", need, ctx->ws_bytes);
  Carver c{ctx->ws, 0, ctx->ws_bytes, false};
  ExactWs w;
  carve(c, w, xa, xb, dia, dib);
  cudaStream_t st = ctx->stream;
  bool hi;
  if ((rc = stage_inputs(ctx, A, nA, B, nB, D, stA, stB, hi))) return rc;
  CK(cudaMemcpyAsync(dia, ia.data(), sizeof(int64_t) * kA, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dib, ib.data(), sizeof(int64_t) * kB, cudaMemcpyHostToDevice, st));
  CK(launch_gather_offset(A, D, dia, 0, kA, 0, xa, st));
  CK(launch_gather_offset(B, D, dib, 0, kB, 0, xb, st));
  CK(cudaMemsetAsync(w.bad, 0, sizeof(int), st));
  CK(launch_centre(xa, kA, xb, kB, D, w.centre, st));
  if ((rc = prep_pair(ctx, xa, kA, xb, kB, D, w.A, w.B, w.bad, w.centre))) return rc;
  if ((rc = bidir_on_ops(ctx, w.A, w.B, D, w))) return rc;
  ExactHost h;
  if ((rc = fetch(ctx, w, h))) return rc;
  fill_directed(&out->ab, h.keys[0], h.nn_d[0], h.nn_j[0]);
  fill_directed(&out->ba, h.keys[1], h.nn_d[1], h.nn_j[1]);
  out->ab.a = ia[out->ab.a];
  out->ab.b = ib[out->ab.b];
  out->ba.a = ib[out->ba.a];
  out->ba.b = ia[out->ba.b];
  out->value = out->ab.dist2 >= out->ba.dist2 ? out->ab.dist : out->ba.dist;
  return PROHD_OK;
}

int prohd_estimate_with_dirs(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D,
                             int32_t n_dirs, int64_t m, const double* dirs, prohd_est* out, int64_t* idxA_out,
                             int64_t* idxB_out) {
  if (dirs == nullptr || n_dirs < 1) return fail(ctx, PROHD_E_INVALID, "dirs must be non-null with n_dirs >= 1");
  return prohd_run(ctx, A, nA, B, nB, D, n_dirs - 1, m, dirs, n_dirs, out, nullptr, idxA_out, idxB_out);
}

}  // extern "C"
