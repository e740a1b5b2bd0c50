// api_common.cuh — host-side helpers shared by the C-ABI translation units:
// context struct, error reporting, workspace carving, input staging, operand
// preparation and the distance-kernel driver.
#pragma once
#include "../../include/prohd.h"
#include "internal.cuh"

#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace prohd {
enum Phase { PH_TOTAL, PH_H2D, PH_PREP, PH_DIST, PH_REDUCE, PH_MOMENTS, PH_EIGEN, PH_SELECT, PH_SUBSET, PH_COUNT };
}

struct prohd_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint8_t* ws = nullptr;
  size_t ws_bytes = 0;
  int num_sms = 148;
  std::string err;
  // tracing (prohd_enable_timing): CUDA events recorded on `stream` around phases
  bool timing = false;
  std::vector<cudaEvent_t> ev;
  int nev = 0;
  struct Mark {
    int phase, e0, e1;
  };
  std::vector<Mark> marks;
  int t_total = -1;
  long long launches0 = 0;
  prohd_timings last{};
  // second stream for independent per-set work (the two sets' selection chains overlap)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // CUDA-graph replay of prohd_estimate's stream-ordered phases (prohd_estimate.cu): the
  // library's own capture stream (the caller's may be the legacy default stream, which cannot
  // be captured), joined to the caller's stream by events, and a small cache of instantiated
  // graphs keyed by every argument the enqueued work depends on
  cudaStream_t gstream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  struct GraphEntry {
    std::vector<uint8_t> key;
    cudaGraphExec_t exec = nullptr;
    long long launches = 0;          // kernels in the graph (added to the launch counter per replay)
    std::vector<uint8_t> host;       // host-side values the enqueue computed (restored on replay)
  };
  std::vector<GraphEntry> graphs;
};

namespace prohd {

// ------------------------------------------------------------------ TMA descriptors
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

inline bool make_tmap_2d(CUtensorMap* map, const float* base, int64_t rows, int Dp, int box_rows, char* err,
                  size_t errlen, int box_inner = kBK, int64_t row_stride = 0) {
  PFN_encodeTiled enc = get_encode();
  if (enc == nullptr) {
    snprintf(err, errlen, "cuTensorMapEncodeTiled unavailable");
    return false;
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(Dp), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_stride > 0 ? row_stride : Dp) * 4};  // bytes, % 16 == 0
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   box_inner * 4 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(err, errlen, "cuTensorMapEncodeTiled failed (%d) rows=%lld Dp=%d box=%d", static_cast<int>(r),
             static_cast<long long>(rows), Dp, box_rows);
    return false;
  }
  return true;
}

// ------------------------------------------------------------------ workspace carving
struct Carver {
  uint8_t* base;
  size_t off = 0;
  size_t cap;
  bool dry;  // size-only pass
  template <typename T>
  T* take(int64_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = dry ? nullptr : reinterpret_cast<T*>(base + off);
    off += static_cast<size_t>(count) * sizeof(T);
    return p;
  }
};

// Operands of one point set for the distance kernel (K0 output).
struct SetOps {
  const float* x = nullptr;     // device copy of the fp32 input (D stride)
  void* H = nullptr;            // split hi (fp16 of the scaled coordinates, or fp32 RN-TF32)
  void* L = nullptr;            // split lo
  float* norms = nullptr;       // ||y||^2, padded to kBN with +inf
  float* scale = nullptr;       // per-row power-of-two scale (F16), padded to kBN
  PrepStats* stats = nullptr;   // max |y|, min ||y||^2 of the set
  int64_t n = 0;
  bool f16 = true;
};

struct ExactWs {
  float* stageA = nullptr;
  float* stageB = nullptr;
  SetOps A, B;
  float* rowmin = nullptr;
  float* colmin = nullptr;
  unsigned long long* keys = nullptr;  // [2]
  double* nn_d = nullptr;              // [2]
  long long* nn_j = nullptr;           // [2]
  double* blk_d = nullptr;
  long long* blk_j = nullptr;
  int* bad = nullptr;
  double* centre = nullptr;  // [2D]: the pair's common centre (K0), then scratch
  void* res = nullptr;       // ExactResDev: the packed result (prohd_api.cu)
};

inline void carve_set(Carver& c, SetOps& s, int64_t n, int D) {
  const int Dp = k6_stride_f32(D);  // room for either format (fp16 uses half)
  s.n = n;
  s.H = c.take<float>(n * Dp);
  s.L = c.take<float>(n * Dp);
  s.norms = c.take<float>(round_up(n, kBN));
  s.scale = c.take<float>(round_up(n, kBN));
  s.stats = c.take<PrepStats>(1);
}

inline size_t carve_exact(Carver& c, ExactWs& w, int64_t nA, int64_t nB, int D, bool host_inputs) {
  if (host_inputs) {
    w.stageA = c.take<float>(nA * D);
    w.stageB = c.take<float>(nB * D);
  }
  carve_set(c, w.A, nA, D);
  carve_set(c, w.B, nB, D);
  w.rowmin = c.take<float>(nA > nB ? nA : nB);
  w.colmin = c.take<float>(nA > nB ? nA : nB);
  w.keys = c.take<unsigned long long>(2);
  w.nn_d = c.take<double>(2);
  w.nn_j = c.take<long long>(2);
  w.blk_d = c.take<double>(kNNBlocks);
  w.blk_j = c.take<long long>(kNNBlocks);
  w.bad = c.take<int>(1);
  w.centre = c.take<double>(2 * static_cast<int64_t>(D));
  w.res = c.take<uint8_t>(64);
  return c.off;
}

}  // namespace prohd

using namespace prohd;

// ------------------------------------------------------------------ tracing
inline int tmark(prohd_ctx* ctx) {
  if (!ctx->timing) return -1;
  if (ctx->nev >= static_cast<int>(ctx->ev.size())) return -1;
  cudaEventRecord(ctx->ev[ctx->nev], ctx->stream);
  return ctx->nev++;
}
inline void tspan(prohd_ctx* ctx, int phase, int e0) {
  if (e0 < 0) return;
  const int e1 = tmark(ctx);
  if (e1 >= 0) ctx->marks.push_back({phase, e0, e1});
}
// call at the start of an ABI call (after enter)
inline void call_begin(prohd_ctx* ctx) {
  ctx->nev = 0;
  ctx->marks.clear();
  ctx->last = prohd_timings{};
  ctx->launches0 = launch_counter().load();
  ctx->t_total = tmark(ctx);
}
// call right before the final stream synchronisation
inline void call_end(prohd_ctx* ctx) { tspan(ctx, PH_TOTAL, ctx->t_total); }
// call after the final synchronisation
inline void call_collect(prohd_ctx* ctx) {
  prohd_timings& t = ctx->last;
  t.kernel_launches = static_cast<int32_t>(launch_counter().load() - ctx->launches0);
  if (!ctx->timing) return;
  double acc[PH_COUNT] = {0};
  for (const auto& mk : ctx->marks) {
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, ctx->ev[mk.e0], ctx->ev[mk.e1]) == cudaSuccess) acc[mk.phase] += ms;
    if (mk.phase == PH_DIST) t.dist_launches++;
  }
  t.total_ms = acc[PH_TOTAL];
  t.h2d_ms = acc[PH_H2D];
  t.prep_ms = acc[PH_PREP];
  t.dist_ms = acc[PH_DIST];
  t.reduce_ms = acc[PH_REDUCE];
  t.moments_ms = acc[PH_MOMENTS];
  t.eigen_ms = acc[PH_EIGEN];
  t.select_ms = acc[PH_SELECT];
  t.subset_ms = acc[PH_SUBSET];
}


// ------------------------------------------------------------------ helpers
inline int fail(prohd_ctx* ctx, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  return code;
}

#define CK(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) return fail(ctx, PROHD_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

inline bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

inline int enter(prohd_ctx* ctx) {
  if (ctx == nullptr) return PROHD_E_INVALID;
  ctx->err.clear();
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return fail(ctx, PROHD_E_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
  return PROHD_OK;
}

inline int check_sets(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D) {
  if (A == nullptr || B == nullptr) return fail(ctx, PROHD_E_INVALID, "null input pointer");
  if (nA < 1 || nB < 1) return fail(ctx, PROHD_E_INVALID, "empty point cloud (nA=%lld nB=%lld)", (long long)nA,
                                    (long long)nB);
  if (D < 1) return fail(ctx, PROHD_E_INVALID, "D must be >= 1 (got %d)", D);
  if (nA > 0x7FFFFF00LL || nB > 0x7FFFFF00LL) return fail(ctx, PROHD_E_INVALID, "n too large for 32-bit row keys");
  return PROHD_OK;
}

// Device inputs with D % 4 == 0 feed 16-byte vector loads, cp.async / bulk copies and TMA
// (K1, K3, K4), which need 16-byte aligned bases (row strides 4D are then multiples of 16).
// torch allocations are 256-byte aligned; a pointer offset by a partial row is rejected
// here with PROHD_E_INVALID instead of faulting inside a kernel (prohd.h "Alignment").
inline int check_aligned(prohd_ctx* ctx, const void* p, int32_t D, const char* what) {
  if (p != nullptr && D % 4 == 0 && (reinterpret_cast<uintptr_t>(p) & 15u) != 0)
    return fail(ctx, PROHD_E_INVALID, "%s must be 16-byte aligned when D %% 4 == 0", what);
  return PROHD_OK;
}

// Make device copies of A/B available (staging host inputs through the workspace).
inline int stage_inputs(prohd_ctx* ctx, const float*& A, int64_t nA, const float*& B, int64_t nB, int32_t D,
                        float* stA, float* stB, bool& host_inputs) {
  const bool dA = is_device_ptr(A), dB = is_device_ptr(B);
  host_inputs = !(dA && dB);
  const int t0 = tmark(ctx);
  if (!dA) {
    if (stA == nullptr) return fail(ctx, PROHD_E_WORKSPACE, "host inputs need a PROHD_WS_HOST_INPUTS workspace");
    CK(cudaMemcpyAsync(stA, A, sizeof(float) * nA * D, cudaMemcpyHostToDevice, ctx->stream));
    A = stA;
  }
  if (!dB) {
    if (stB == nullptr) return fail(ctx, PROHD_E_WORKSPACE, "host inputs need a PROHD_WS_HOST_INPUTS workspace");
    CK(cudaMemcpyAsync(stB, B, sizeof(float) * nB * D, cudaMemcpyHostToDevice, ctx->stream));
    B = stB;
  }
  if (host_inputs) tspan(ctx, PH_H2D, t0);
  int rc = check_aligned(ctx, A, D, "A");
  if (rc == PROHD_OK) rc = check_aligned(ctx, B, D, "B");
  return rc;
}

// K0 for the two sets of a pair (the sets a K6 sweep will meet): stats of both first (the F16
// scale mode depends on both), then the split arrays of each. The sets' operands may be used in
// either role (row or column) against each other.
inline int prep_pair(prohd_ctx* ctx, const float* X, int64_t nX, const float* Y, int64_t nY, int D, SetOps& sx,
                     SetOps& sy, int* bad, const double* centre) {
  const bool f16 = !k6_split3();
  SetOps* ops[2] = {&sx, &sy};
  const float* src[2] = {X, Y};
  const int64_t n[2] = {nX, nY};
  const int t0 = tmark(ctx);
  for (int i = 0; i < 2; ++i) {
    ops[i]->x = src[i];
    ops[i]->n = n[i];
    ops[i]->f16 = f16;
    CK(cudaMemsetAsync(&ops[i]->stats->maxabs, 0, sizeof(unsigned), ctx->stream));
    CK(cudaMemsetAsync(&ops[i]->stats->minnorm2, 0x7F, sizeof(unsigned), ctx->stream));  // 3.39e38
    CK(launch_prep_stats(src[i], nullptr, n[i], D, round_up(n[i], kBN), centre, ops[i]->norms, ops[i]->stats, bad,
                         ctx->stream));
  }
  for (int i = 0; i < 2; ++i)
    CK(launch_prep_write(src[i], nullptr, n[i], D, round_up(n[i], kBN), centre, ops[i]->stats, ops[1 - i]->stats,
                         f16, ops[i]->H, ops[i]->L, ops[i]->scale, ctx->stream));
  tspan(ctx, PH_PREP, t0);
  return PROHD_OK;
}

// rows of `R` against columns of `C` -> rowmin (device)
inline int run_dist(prohd_ctx* ctx, const SetOps& R, const SetOps& C, int D, float* rowmin,
                    float* colmin = nullptr) {
  CUtensorMap maps[4];
  char err[256];
  // 64-byte TMA box rows (SWIZZLE_64B) over the split arrays, described as fp32 columns
  const int cols = R.f16 ? k6_stride_f16(D) / 2 : k6_stride_f32(D);
  if (!make_tmap_2d(&maps[0], reinterpret_cast<const float*>(R.H), R.n, cols, kBM, err, sizeof err, 16) ||
      !make_tmap_2d(&maps[1], reinterpret_cast<const float*>(R.L), R.n, cols, kBM, err, sizeof err, 16) ||
      !make_tmap_2d(&maps[2], reinterpret_cast<const float*>(C.H), C.n, cols, kBN, err, sizeof err, 16) ||
      !make_tmap_2d(&maps[3], reinterpret_cast<const float*>(C.L), C.n, cols, kBN, err, sizeof err, 16))
    return fail(ctx, PROHD_E_CUDA, "%s", err);
  CUtensorMap bhalf[2];
  const bool pair = k6_uses_pair(D, R.f16, colmin != nullptr, R.n, C.n);
  if (pair && (!make_tmap_2d(&bhalf[0], reinterpret_cast<const float*>(C.H), C.n, cols, kBM, err, sizeof err, 16) ||
               !make_tmap_2d(&bhalf[1], reinterpret_cast<const float*>(C.L), C.n, cols, kBM, err, sizeof err, 16)))
    return fail(ctx, PROHD_E_CUDA, "%s", err);
  DistArgs a;
  a.maps = maps;
  a.maps_bhalf = pair ? bhalf : nullptr;
  a.nA = R.n;
  a.nB = C.n;
  a.D = D;
  a.f16 = R.f16;
  a.na = R.norms;
  a.nb = C.norms;
  a.sa = R.scale;
  a.sb = C.scale;
  a.sta = R.stats;
  a.stb = C.stats;
  a.rowmin = rowmin;
  a.num_sms = ctx->num_sms;
  a.colmin = colmin;
  const int t0 = tmark(ctx);
  CK(launch_dist_rowmin(a, ctx->stream));
  tspan(ctx, PH_DIST, t0);
  return PROHD_OK;
}

// h(R, C) on prepared operands; result lands in w.keys[slot], w.nn_d[slot], w.nn_j[slot].
inline int directed_on_ops(prohd_ctx* ctx, const SetOps& R, const SetOps& C, int D, ExactWs& w, int slot) {
  int rc = run_dist(ctx, R, C, D, w.rowmin);
  if (rc) return rc;
  const int t0 = tmark(ctx);
  CK(launch_rowmax_key(w.rowmin, R.n, 0, &w.keys[slot], ctx->stream));
  CK(launch_nn64_from_key(R.x, 0, R.n, &w.keys[slot], C.x, C.n, D, w.blk_d, w.blk_j, kNNBlocks, &w.nn_d[slot],
                          &w.nn_j[slot], ctx->stream));
  tspan(ctx, PH_REDUCE, t0);
  return PROHD_OK;
}

// h(R, C) and h(C, R): slot 0 is R -> C, slot 1 is C -> R. For D >= 128 from ONE fused
// bidirectional sweep (row and column minima, 65536 x 262144 at D = 256:
// 31.5 ms against 50.4 ms for two directed sweeps); below that two directed sweeps are faster (the
// column-minimum epilogue outweighs the halved MMA work: D = 64 14.7 vs 16.4 ms, D = 16 26.5 vs
// 50.1 ms). Either way both operands come from the same K0 preparation (common centre).
inline int bidir_on_ops(prohd_ctx* ctx, const SetOps& R, const SetOps& C, int D, ExactWs& w) {
  int rc = D >= 128 ? run_dist(ctx, R, C, D, w.rowmin, w.colmin) : run_dist(ctx, R, C, D, w.rowmin);
  if (rc) return rc;
  if (D < 128 && (rc = run_dist(ctx, C, R, D, w.colmin))) return rc;
  const int t0 = tmark(ctx);
  CK(launch_rowmax_key(w.rowmin, R.n, 0, &w.keys[0], ctx->stream));
  CK(launch_rowmax_key(w.colmin, C.n, 0, &w.keys[1], ctx->stream));
  CK(launch_nn64_from_key(R.x, 0, R.n, &w.keys[0], C.x, C.n, D, w.blk_d, w.blk_j, kNNBlocks, &w.nn_d[0],
                          &w.nn_j[0], ctx->stream));
  CK(launch_nn64_from_key(C.x, 0, C.n, &w.keys[1], R.x, R.n, D, w.blk_d, w.blk_j, kNNBlocks, &w.nn_d[1],
                          &w.nn_j[1], ctx->stream));
  tspan(ctx, PH_REDUCE, t0);
  return PROHD_OK;
}

// Enqueue `work` (stream-ordered launches on ctx->stream and ctx->aux only: no host reads, no
// host-memory copies) through a cached CUDA graph: the first call with this key captures and
// instantiates it (the launch counter counts its kernels once, at capture), later calls replay it
// (count_launch(n) per replay). `host` is a byte image of the host-side values the enqueue
// computes (saved at capture, restored on replay). A capture the runtime refuses falls back to
// running `work` eagerly; an error inside `work` is returned as is.
template <class F>
int graphed(prohd_ctx* ctx, const std::vector<uint8_t>& key, void* host, size_t host_bytes, F&& work) {
  for (auto& g : ctx->graphs)
    if (g.key == key) {
      if (host_bytes) std::memcpy(host, g.host.data(), host_bytes);
      count_launch(static_cast<int>(g.launches));
      CK(cudaGraphLaunch(g.exec, ctx->stream));
      return PROHD_OK;
    }
  const long long l0 = launch_counter().load();
  if (cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return work();
  }
  const int rc = work();
  cudaGraph_t graph = nullptr;
  const cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
  if (e != cudaSuccess || graph == nullptr) {  // capture invalidated: run eagerly
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    ctx->err.clear();
    launch_counter().store(l0);
    return work();
  }
  if (rc != PROHD_OK) {
    cudaGraphDestroy(graph);
    return rc;
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) {
    cudaGetLastError();
    launch_counter().store(l0);
    return work();
  }
  prohd_ctx::GraphEntry ent;
  ent.key = key;
  ent.exec = exec;
  ent.launches = launch_counter().load() - l0;
  ent.host.assign(static_cast<const uint8_t*>(host), static_cast<const uint8_t*>(host) + host_bytes);
  if (ctx->graphs.size() >= 8) {  // small FIFO cache
    cudaGraphExecDestroy(ctx->graphs.front().exec);
    ctx->graphs.erase(ctx->graphs.begin());
  }
  ctx->graphs.push_back(std::move(ent));
  CK(cudaGraphLaunch(exec, ctx->stream));
  return PROHD_OK;
}

// The library's capture stream for graphed() work: created on first use; while a GraphStream is
// alive ctx->stream is the capture stream, ordered after the caller's stream (event) and the
// caller's stream ordered after it again on destruction.
inline int ensure_gstream(prohd_ctx* ctx) {
  if (ctx->gstream != nullptr) return PROHD_OK;
  CK(cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming));
  return PROHD_OK;
}
struct GraphStream {
  prohd_ctx* c;
  cudaStream_t orig;
  bool on;
  GraphStream(prohd_ctx* c_, bool on_) : c(c_), orig(c_->stream), on(on_ && c_->gstream != nullptr) {
    if (!on) return;
    cudaEventRecord(c->ev_in, orig);
    cudaStreamWaitEvent(c->gstream, c->ev_in, 0);
    c->stream = c->gstream;
  }
  ~GraphStream() {
    if (!on) return;
    cudaEventRecord(c->ev_out, c->gstream);
    cudaStreamWaitEvent(orig, c->ev_out, 0);
    c->stream = orig;
  }
};
// Graph-cache key: the raw bytes of every argument the enqueued work depends on, plus the option
// table and the workspace (pointer, size).
struct KeyBuf {
  std::vector<uint8_t> b;
  template <typename T>
  KeyBuf& add(const T& v) {
    const uint8_t* p = reinterpret_cast<const uint8_t*>(&v);
    b.insert(b.end(), p, p + sizeof(T));
    return *this;
  }
};
inline KeyBuf graph_key(prohd_ctx* ctx, int tag) {
  KeyBuf k;
  k.add(tag).add(ctx->ws).add(ctx->ws_bytes).add(ctx->num_sms);
  for (int i = 0; i < OPT_COUNT; ++i) k.add(opt(static_cast<OptId>(i)));
  return k;
}

inline void fill_directed(prohd_directed* o, unsigned long long key, double d2, long long j) {
  o->a = static_cast<int64_t>(0xFFFFFFFFu - static_cast<uint32_t>(key & 0xFFFFFFFFull));
  o->b = j;
  o->dist2 = d2;
  o->dist = std::sqrt(d2);
  uint32_t fb = static_cast<uint32_t>(key >> 32);
  float f;
  std::memcpy(&f, &fb, 4);
  o->dist2_tc = f;
}

