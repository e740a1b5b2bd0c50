// internal.cuh — launchers shared between the kernel files and the C-ABI layer.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>

namespace prohd {

// Process-wide count of kernel launches issued by this library (for tracing).
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> c{0};
  return c;
}
inline void count_launch(int n = 1) { launch_counter().fetch_add(n, std::memory_order_relaxed); }

// Variant options (prohd_set_option, include/prohd.h). Each forces another device variant of
// the SAME computation for A/B measurement; -1 = unset (the measured-best default). They are set
// explicitly through the ABI (never read from the environment), process-wide.
enum OptId {
  OPT_K6_VARIANT,    // 1 single A block, 2 two-SM pair (directed), 3 two A blocks per CTA
  OPT_K6_SPLIT3,     // 1: literal 3xTF32 (three TF32 MMAs on fp32 hi/lo)
  OPT_K6_BIDIR_2A,   // fused bidirectional sweep on 0 the single-block, 1 the two-A, 2 the CTA-pair kernel (default)
  OPT_K6_SPLITS_2X,  // 1: the old fill-twice column-split rule
  OPT_K1_PATH,       // 0 fp64 DMMA Gram, 1 int8 tcgen05 Gram, 2 legacy 64x64-tile moments kernel
  OPT_K1_CTAS,       // legacy moments kernel: resident CTAs per SM (3 or 4)
  OPT_K1_CS_SMS,     // DMMA Gram: column-sum SMs inside the launch (0 = separate pass)
  OPT_K1_BETA_MILLI, // DMMA Gram: CTA allocation by (load + beta/1000)
  OPT_SHIFT,         // 0 never / 1 always shift the Gram
  OPT_K3_SIMT,       // 1: SIMT projection kernel instead of tcgen05
  OPT_EIG_STOP,      // stop K2 after stage 1|2|3 (timing prefixes)
  OPT_EIG_CL,        // 8: portable 8-CTA tridiagonalisation cluster
  OPT_K1_ABLATE,     // int8 Gram timing ablations (wrong results): 1 no slicing work, 2 no MMAs
  OPT_K4_SAMPLED,    // 0 radix K4 over all projections, 1 sampled-threshold K4 wherever it applies
  OPT_K1_I8_CTAS,    // int8 Gram: cap on the CTA count (tests: mid-sweep drains at small sizes)
  OPT_GRAPH,         // 0: prohd_estimate launches eagerly (no CUDA-graph replay)
  OPT_COUNT
};
inline std::atomic<long long>* option_table() {
  static std::atomic<long long> t[OPT_COUNT] = {};
  static bool init = [] {
    for (auto& v : t) v.store(-1);
    return true;
  }();
  (void)init;
  return t;
}
inline long long opt(OptId id) { return option_table()[id].load(std::memory_order_relaxed); }

constexpr int kBM = 128;  // rows of the row operand per CTA tile (UMMA M)
constexpr int kBN = 256;  // columns (points of the column operand) per tile (UMMA N)
constexpr int kBK = 32;   // fp32 K elements per pipeline chunk (one 128-B swizzle row)

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int pad_dim(int D) { return static_cast<int>(round_up(D, 4)); }  // 16-B TMA row stride

// K0 (k_prep.cu): the K6 operands of one point set. y = x - c (fp64, c the pair's common centre,
// nullptr = none); three-term split arrays H (hi) and L (lo), row stride k6_stride_*(D) elements,
// zero padded:
//   F16  (default):          hi = fp16_rn(s y), lo = fp16_rn(s y - hi), s = scale[i] (power of two)
//   TF32 (option k6_split3): hi = rn_tf32(y), lo = fp32(y - hi), scale[i] = 1
// norms[i] = ||y_i||^2 (fp32 from fp64) for i < n, +inf for n <= i < n_pad. *bad = 1 if any x or
// norm is not finite. The stats pass must run on BOTH sets of a pair before either write pass
// (the F16 scale mode depends on both).
struct PrepStats {
  unsigned maxabs;    // float bits of max_i,f |y_if| (0 = none yet)
  unsigned minnorm2;  // float bits of min_i ||y_i||^2 (+inf = none yet)
};
inline int k6_stride_f16(int D) { return static_cast<int>(round_up(D, 8)); }  // halfs: 16-B row stride
inline int k6_stride_f32(int D) { return static_cast<int>(round_up(D, 4)); }  // floats
// power-of-two scale putting max |y| into (2^13, 2^14] (1 for 0 / non-finite; clamped to 2^+-60)
__host__ __device__ inline float prep_scale_for(float M) {
  if (!(M > 0.0f) || !(M < 3.0e38f)) return 1.0f;
  int e = 0;
  (void)frexpf(M, &e);  // M = m 2^e, m in [0.5, 1)
  int k = 14 - e;
  k = k < -60 ? -60 : (k > 60 ? 60 : k);
  return ldexpf(1.0f, k);
}
// F16 scale mode of a pair: ONE scale per set (s_X from the set's max |y|) unless some row is so
// small against the pair's largest coordinate M that the fp16 subnormal floor (2^-25 / s_X per
// coordinate, <= 2^-38 M) could cost more than 3e-6 of the pair's ||a||^2 + ||b||^2:
// rows need sqrt(||a||^2+||b||^2) >= 2^-37 sqrt(2D) M / 3e-6 = 2.43e-6 sqrt(2D) M. Otherwise one
// scale per ROW (every row at the top of the fp16 range; K6's epilogue then rescales per column).
__device__ __forceinline__ bool prep_mode_perrow(const PrepStats* a, const PrepStats* b, int D) {
  const float M = fmaxf(__uint_as_float(a->maxabs), __uint_as_float(b->maxabs));
  const float mn2 = fminf(__uint_as_float(a->minnorm2), __uint_as_float(b->minnorm2));
  return !(sqrtf(mn2) >= 2.43e-6f * sqrtf(2.0f * static_cast<float>(D)) * M);
}
cudaError_t launch_prep_stats(const float* X, const long long* idx, int64_t n, int D, int64_t n_pad,
                              const double* centre, float* norms, PrepStats* st, int* bad, cudaStream_t stream);
cudaError_t launch_prep_write(const float* X, const long long* idx, int64_t n, int D, int64_t n_pad,
                              const double* centre, const PrepStats* self, const PrepStats* other, bool f16, void* H,
                              void* L, float* scale, cudaStream_t stream);
// option k6_split3 = 1: the north star's literal 3xTF32 form (fp32 hi/lo, three TF32 MMAs)
// instead of the default three fp16 MMAs on scaled fp16 hi/lo.
bool k6_split3();
// Common centre of a pair (X, Y): fp64 mean of the first min(nX, 4096) rows of X and the
// first min(nY, 4096) rows of Y (either count may be 0), summed per set and then added,
// so centre(X, Y) == centre(Y, X) bit for bit. c: 2D doubles (the second half is scratch).
cudaError_t launch_centre(const float* X, int64_t nX, const float* Y, int64_t nY, int D, double* c,
                          cudaStream_t st);

struct DistArgs {
  const CUtensorMap* maps;  // [A_H, A_L, B_H, B_L]: 64-B box rows (32 fp16 or 16 fp32 features)
  int64_t nA, nB;
  int D;
  bool f16;                 // operand format (K0): F16 (scaled fp16) or TF32
  const float* na;          // row-operand norms
  const float* nb;          // column-operand norms, padded to a multiple of kBN with +inf
  const float* sa;          // row-operand scales (K0), n_pad
  const float* sb;          // column-operand scales, padded to a multiple of kBN
  const PrepStats* sta;     // stats of both sets (F16 scale mode)
  const PrepStats* stb;
  float* rowmin;            // out: min_j d2(i, j), clamped >= 0
  int num_sms;
  float* colmin = nullptr;  // optional out (fused bidirectional pass): min_i d2(i, j), clamped >= 0
  const CUtensorMap* maps_bhalf = nullptr;  // [B_H, B_L] with 128-row boxes (CTA-pair kernel), or null
};
// K6: fused split-precision tcgen05 distance + row-min kernel.
cudaError_t launch_dist_rowmin(const DistArgs& a, cudaStream_t st);
// whether launch_dist_rowmin runs the CTA-pair kernel for this sweep (it then needs maps_bhalf)
bool k6_uses_pair(int D, bool f16, bool bidir, int64_t nA, int64_t nB);

// K7a: packed max key over rows: (bits(d2) << 32) | (0xFFFFFFFF - (row + row_offset)).
cudaError_t launch_rowmax_key(const float* rowmin, int64_t n, int64_t row_offset, unsigned long long* key,
                              cudaStream_t st);
// K7b: fp64 nearest neighbour of point `a` (D floats, device) in B (device, stride D):
//   writes {d2 (double), j (int64)} to out2 (device, 16 bytes). `scratch` holds
//   2 * nblocks entries. Lowest j on exact ties.
cudaError_t launch_nn64(const float* a, const float* B, int64_t nB, int D, double* blk_d, long long* blk_j,
                        int nblocks, double* out_d, long long* out_j, cudaStream_t st);
// helper: a = X + row * D where row is decoded from the key on the device
cudaError_t launch_nn64_from_key(const float* X, int64_t x_offset, int64_t nX, const unsigned long long* key,
                                 const float* B, int64_t nB, int D, double* blk_d, long long* blk_j, int nblocks,
                                 double* out_d, long long* out_j, cudaStream_t st);
constexpr int kNNBlocks = 592;  // 4 x 148 SMs

// TMA descriptor for a row-major fp32 matrix [rows x Dp], box {box_inner, box_rows}, SWIZZLE_128B for
// box_inner = 32 (128-B rows) and SWIZZLE_64B for box_inner = 16; row_stride in floats (0 = Dp).
bool make_tmap_2d(CUtensorMap* map, const float* base, int64_t rows, int Dp, int box_rows, char* err, size_t errlen,
                  int box_inner, int64_t row_stride);

}  // namespace prohd
