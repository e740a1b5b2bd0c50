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
  OPT_K6_BIDIR_2A,   // 1: fused bidirectional sweep on the two-A kernel
  OPT_K6_SPLITS_2X,  // 1: the old fill-twice column-split rule
  OPT_K1_PATH,       // 0 fp64 DMMA Gram, 1 int8 tcgen05 Gram, 2 legacy 64x64-tile moments kernel
  OPT_K1_CTAS,       // legacy moments kernel: resident CTAs per SM (3 or 4)
  OPT_K1_CS_SMS,     // DMMA Gram: column-sum SMs inside the launch (0 = separate pass)
  OPT_K1_BETA_MILLI, // DMMA Gram: CTA allocation by (load + beta/1000)
  OPT_SHIFT,         // 0 never / 1 always shift the Gram
  OPT_K3_SIMT,       // 1: SIMT projection kernel instead of tcgen05
  OPT_EIG_STOP,      // stop K2 after stage 1|2|3 (timing prefixes)
  OPT_EIG_CL,        // 8: portable 8-CTA tridiagonalisation cluster
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

// K0: split points, translated by a common centre c (fp64, D; nullptr = none), into the K6
// operands: y = x - c in fp64, hi = fp32(y) rounded to nearest TF32 (low 13 mantissa bits
// zero), lo = fp32(y - hi), pr[f] = bf16 pair (hi_f, lo_f) and pc[f] = (lo_f, hi_f) (element
// 2f at the lower address), and ||y||^2 accumulated in fp64. hi/pr/pc rows have stride Dp
// (zero padded); norms[i] = ||y_i||^2 for i < n and +inf for n <= i < n_pad. *bad = 1 if any
// x or norm is not finite.
cudaError_t launch_prep(const float* X, int64_t n, int D, int Dp, int64_t n_pad, const double* centre, float* hi,
                        uint32_t* pr, uint32_t* pc, float* norms, int* bad, cudaStream_t st);
// option k6_split3 = 1: the north star's literal 3xTF32 form (hi.hi + hi.lo + lo.hi, three TF32
// MMAs); K0 then writes lo (fp32) into pr and pc instead of the bf16 pairs. Default: off.
bool k6_split3();
// Common centre of a pair (X, Y): fp64 mean of the first min(nX, 4096) rows of X and the
// first min(nY, 4096) rows of Y (either count may be 0), summed per set and then added,
// so centre(X, Y) == centre(Y, X) bit for bit. c: 2D doubles (the second half is scratch).
cudaError_t launch_centre(const float* X, int64_t nX, const float* Y, int64_t nY, int D, double* c,
                          cudaStream_t st);

struct DistArgs {
  const CUtensorMap* maps;  // [A_hi, A_pr, B_hi, B_pc]
  int64_t nA, nB;
  int D;
  const float* na;  // row-operand norms
  const float* nb;  // column-operand norms, padded to a multiple of kBN with +inf
  float* rowmin;    // out: min_j d2(i, j), clamped >= 0
  int num_sms;
  float* colmin = nullptr;  // optional out (fused bidirectional pass): min_i d2(i, j), clamped >= 0
};
// K6: fused 3xTF32 tcgen05 distance + row-min kernel.
cudaError_t launch_dist_rowmin(const DistArgs& a, cudaStream_t st);
// rows per TMA box of the column operand for the selected K6 variant (256: 1-SM, 128: 2-SM pair)
int dist_b_box_rows(int D, bool bidir);
// fp32 features per TMA box row of the selected K6 variant (32: SWIZZLE_128B; 16: SWIZZLE_64B)
int dist_box_inner(int D, bool bidir);

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
// box_inner = 32 (128-B rows) and SWIZZLE_64B for box_inner = 16.
bool make_tmap_2d(CUtensorMap* map, const float* base, int64_t rows, int Dp, int box_rows, char* err, size_t errlen,
                  int box_inner);

}  // namespace prohd
