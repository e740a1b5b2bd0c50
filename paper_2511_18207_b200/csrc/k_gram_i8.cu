// k_gram_i8.cu — K1 on the int8 tensor cores: the Gram G = sum_p x_p x_p^T of A u B,
// exact-integer products (Ozaki-style slicing), for data taken about the origin.
//
// PAPER.md Alg. 2 lines 1-2; see k_gram.cu for the fp64 DMMA variant and the
// shift policy (this path runs when the shift kernel dropped the shift, s = 0).
//
// Each fp32 value of feature f is written in fixed point relative to its column's
// magnitude bound 2^E_f (E_f > log2 max_p |x_pf|) as 7 signed 7-bit digits,
//     x = sign * sum_t d_t 2^(E_f - 7(t+1)),  d_t in [0, 127],  t = 0..6  (49 bits),
// exact whenever x has no bits below 2^(E_f - 49) (else rounded to nearest, |err| <=
// 2^(E_f - 50)). Slice t of x is the int8 sign*d_t. Then
//     x_i x_j = 2^(E_i + E_j - 14) sum_{t,u} s_t(x_i) s_u(x_j) 2^(-7(t+u)),
// and sum_p s_t(x_pi) s_u(x_pj) is an exact int8 x int8 -> int32 tensor-core product.
// Pairs with t + u <= 7 are kept (34 pairs; the dropped ones are < 2^-62 of
// max_p|x_pi| max_p|x_pj| per point); pairs with the same d = t + u share one int32 TMEM
// accumulator (8 accumulators x 64 columns = all 512 TMEM columns). With <= 8 pairs per d
// and |s_t s_u| <= 127^2 an accumulator grows by < 2^17 per point, so it is drained to
// fp64 every 8192 points (< 2^30), exact. The epilogue combines the 8 accumulators in fp64
// with their power-of-two weights.
//
// Kernels:
//   colmax_kernel  per-feature max|x| (atomicMax on the bits) and fp64 column sums of A and
//                  of B (per-CTA partials, fixed-order reduce): one read of the data.
//   slice_kernel   the 7 int8 slice planes, feature-major: S[t][f][p] (p over A then B, rows
//                  padded to Np = 64k points), through a shared-memory transpose.
//   gram_i8_kernel tiles of 128 I-features x 64 J-features (every tile holding an i <= j
//                  pair), CTA = (tile, point range), warp-specialised like K6: warp 0 TMA
//                  (SWIZZLE_64B boxes of 64 points x 64 features, 7 slices of the I and J
//                  blocks, 84 KB per stage, 2 stages), warp 1 TMEM + tcgen05.mma.kind::i8
//                  (M=128, N=64, K=32), warps 2-5 drain the accumulators to fp64.
#include "internal.cuh"
#include "prohd_kernels.cuh"
#include "sm100.cuh"

namespace prohd {
namespace {

constexpr int kSl = 7;           // slices (7 bits each)
constexpr int kPts = 64;         // points per pipeline stage (one 64-B swizzle row)
constexpr int kFI = 128;         // I-block features (UMMA M)
constexpr int kFJ = 64;          // J-block features (UMMA N)
constexpr int kNAcc = 8;         // accumulators d = t + u = 0..7
constexpr int kFlush = 8192;     // points between drains (exactness bound above)
constexpr int kStagesI8 = 2;
constexpr uint32_t kBox = kPts * 64;                       // 4 KB: one TMA box (64 rows x 64 B)
constexpr uint32_t kStageI8 = kSl * (kFI / 64 + 1) * kBox;  // 7 x 3 boxes = 84 KB
constexpr size_t kSmemI8 = static_cast<size_t>(kStagesI8) * kStageI8 + 1024 + 256;

// ------------------------------------------------------------------ colmax + column sums
__global__ void __launch_bounds__(256) colmax_kernel(const float* __restrict__ A, int64_t nA,
                                                     const float* __restrict__ B, int64_t nB, int D,
                                                     unsigned* __restrict__ maxbits, double* __restrict__ Spart) {
  // thread = (feature f = blockIdx.y * 32 + lane, warp w): rows w, w + 8, ... of each CTA chunk
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int f = blockIdx.y * 32 + lane;
  const int64_t N = nA + nB;
  unsigned m = 0u;
  double sa = 0.0, sb = 0.0;
  if (f < D) {
    for (int64_t p = static_cast<int64_t>(blockIdx.x) * 8 + w; p < N; p += static_cast<int64_t>(gridDim.x) * 8) {
      const float x = p < nA ? __ldg(A + p * D + f) : __ldg(B + (p - nA) * D + f);
      m = max(m, __float_as_uint(x) & 0x7FFFFFFFu);  // |x| bits; inf/nan order above every finite
      if (p < nA)
        sa += static_cast<double>(x);
      else
        sb += static_cast<double>(x);
    }
  }
  __shared__ unsigned sm[8][32];
  __shared__ double s1[8][32], s2[8][32];
  sm[w][lane] = m;
  s1[w][lane] = sa;
  s2[w][lane] = sb;
  __syncthreads();
  if (w == 0 && f < D) {
    unsigned mm = 0u;
    double a = 0.0, b = 0.0;
    for (int q = 0; q < 8; ++q) {
      mm = max(mm, sm[q][lane]);
      a += s1[q][lane];
      b += s2[q][lane];
    }
    atomicMax(maxbits + f, mm);
    Spart[(static_cast<int64_t>(blockIdx.x) * 2 + 0) * D + f] = a;
    Spart[(static_cast<int64_t>(blockIdx.x) * 2 + 1) * D + f] = b;
  }
}

__global__ void __launch_bounds__(256) colsum_reduce_kernel(const double* __restrict__ Spart, int nparts, int D,
                                                            double* __restrict__ SA, double* __restrict__ SB) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < D; f += gridDim.x * blockDim.x) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < nparts; ++q) {
      a += Spart[(static_cast<int64_t>(q) * 2 + 0) * D + f];
      b += Spart[(static_cast<int64_t>(q) * 2 + 1) * D + f];
    }
    SA[f] = a;
    SB[f] = b;
  }
}

// E_f with max|x_f| < 2^E_f (0 for an all-zero column)
__device__ __forceinline__ int col_exp(unsigned mb) {
  const int e = static_cast<int>((mb >> 23) & 0xFFu);
  return e == 0 ? (mb == 0u ? 0 : -125) : e - 126;  // normal: |x| < 2^(e - 127 + 1)
}

// ------------------------------------------------------------------ slicing
constexpr int kSlT = 64;        // tile: 64 points x 64 features
constexpr int kSlRow = 68;      // smem row stride in bytes (17 words: conflict-free packed stores)
__global__ void __launch_bounds__(256) slice_kernel(const float* __restrict__ A, int64_t nA,
                                                    const float* __restrict__ B, int64_t nB, int D, int Df,
                                                    int64_t Np, const unsigned* __restrict__ maxbits,
                                                    int8_t* __restrict__ S) {
  __shared__ __align__(16) uint32_t sm[kSl * kSlT * kSlRow / 4];  // [t][f][68 B]
  const int tid = threadIdx.x;
  const int fl = tid & 63, pg = tid >> 6;  // feature, group of 16 points
  const int f = blockIdx.y * kSlT + fl;
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * kSlT + pg * 16;
  const int64_t N = nA + nB;
  const int E = f < D ? col_exp(__ldg(maxbits + f)) : 0;
  uint32_t word[kSl];
#pragma unroll
  for (int t = 0; t < kSl; ++t) word[t] = 0u;
#pragma unroll 4
  for (int q = 0; q < 16; ++q) {
    const int64_t p = p0 + q;
    float x = 0.0f;
    if (f < D && p < N) x = p < nA ? __ldg(A + p * D + f) : __ldg(B + (p - nA) * D + f);
    const unsigned u = __float_as_uint(x);
    const unsigned ef = (u >> 23) & 0xFFu;
    const unsigned long long mant = ef == 0u ? (u & 0x7FFFFFu) : ((u & 0x7FFFFFu) | 0x800000u);
    const int e = ef == 0u ? -126 : static_cast<int>(ef) - 127;  // x = mant * 2^(e - 23)
    const int sh = e - E + 26;  // y = |x| * 2^(49 - E) = mant * 2^sh
    unsigned long long y;
    if (sh >= 0)
      y = mant << sh;
    else if (sh > -40)
      y = (mant + (1ull << (-sh - 1))) >> (-sh);
    else
      y = 0ull;
    const bool neg = (u >> 31) != 0u;
#pragma unroll
    for (int t = 0; t < kSl; ++t) {
      int dgt = static_cast<int>((y >> (7 * (kSl - 1 - t))) & 127ull);
      if (neg) dgt = -dgt;
      word[t] |= (static_cast<uint32_t>(dgt) & 0xFFu) << (8 * (q & 3));
    }
    if ((q & 3) == 3) {
#pragma unroll
      for (int t = 0; t < kSl; ++t) {
        sm[(t * kSlT + fl) * (kSlRow / 4) + pg * 4 + (q >> 2)] = word[t];
        word[t] = 0u;
      }
    }
  }
  __syncthreads();
  // write out: per (t, f) row, 64 bytes = 4 x 16 B
  for (int q = tid; q < kSl * kSlT * 4; q += 256) {
    const int t = q / (kSlT * 4), r = (q / 4) % kSlT, c = q % 4;
    const uint32_t* src = sm + (t * kSlT + r) * (kSlRow / 4) + c * 4;
    const uint4 v = make_uint4(src[0], src[1], src[2], src[3]);
    const int ff = blockIdx.y * kSlT + r;
    int8_t* dst = S + (static_cast<int64_t>(t) * Df + ff) * Np + static_cast<int64_t>(blockIdx.x) * kSlT + c * 16;
    *reinterpret_cast<uint4*>(dst) = v;
  }
}

// ------------------------------------------------------------------ int8 tensor-core Gram
struct GramI8Sched {
  int ntiles, nranges;
  int64_t per;        // points per range (multiple of kPts)
  int64_t N, Np;
  int D, Df;
  int tI[16], tJ[16];  // tile -> (I block of 128, J block of 64)
};

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// K-major operand staged by TMA with SWIZZLE_64B: rows of 64 B, 8-row (512 B) atoms.
__device__ __forceinline__ uint64_t smem_desc_k_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;          // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(512u >> 4) << 32;   // SBO: 8 rows x 64 B
  d |= static_cast<uint64_t>(1u) << 46;          // version (sm_100)
  d |= static_cast<uint64_t>(4u) << 61;          // SWIZZLE_64B
  return d;
}
// instruction descriptor, kind::i8: D s32, A and B signed int8, K-major, N >> 3, M >> 4
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t M, uint32_t N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// 32 lanes x 32 bit, 32 consecutive columns (as int32)
__device__ __forceinline__ void tmem_ld32i(uint32_t taddr, int (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

__global__ void __launch_bounds__(192, 1)
    gram_i8_kernel(const __grid_constant__ CUtensorMap tS, GramI8Sched s, const unsigned* __restrict__ maxbits,
                   double* __restrict__ Gpart) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStagesI8 * kStageI8);
  uint64_t* empty = full + kStagesI8;
  uint64_t* tfull = empty + kStagesI8;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x % s.ntiles, range = blockIdx.x / s.ntiles;
  const int I = s.tI[tile], J = s.tJ[tile];
  const int64_t q0 = static_cast<int64_t>(range) * s.per;
  const int64_t q1 = q0 + s.per < s.Np ? q0 + s.per : s.Np;
  const int nst = q1 > q0 ? static_cast<int>((q1 - q0) / kPts) : 0;  // stages of 64 points
  const int st_per_flush = kFlush / kPts;
  const int nflush = (nst + st_per_flush - 1) / st_per_flush;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStagesI8; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) tma_prefetch(&tS);
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // -------------------------------------------------------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int c = 0; c < nst; ++c) {
        mbar_wait(&empty[stage], phase ^ 1u);
        uint8_t* st = smem + stage * kStageI8;
        mbar_arrive_expect_tx(&full[stage], kStageI8);
        const int x = static_cast<int>(q0 + static_cast<int64_t>(c) * kPts);
        for (int t = 0; t < kSl; ++t) {
          // I block (2 boxes of 64 rows) then J block (1 box); slice t rows start at t * Df
          uint8_t* dst = st + t * 3 * kBox;
          tma_load_2d(dst, &tS, x, t * s.Df + I * kFI, &full[stage]);
          tma_load_2d(dst + kBox, &tS, x, t * s.Df + I * kFI + 64, &full[stage]);
          tma_load_2d(dst + 2 * kBox, &tS, x, t * s.Df + J * kFJ, &full[stage]);
        }
        if (++stage == kStagesI8) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // -------------------------------------------------------------- MMA issuer
      constexpr uint32_t idesc = idesc_i8(kFI, kFJ);
      int stage = 0;
      uint32_t phase = 0, fphase = 0;
      for (int fl = 0; fl < nflush; ++fl) {
        mbar_wait(tempty, fphase ^ 1u);  // the epilogue drained the previous flush
        tc_fence_after();
        const int c0 = fl * st_per_flush;
        const int c1 = min(nst, c0 + st_per_flush);
        for (int c = c0; c < c1; ++c) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sbase = smem_u32(smem + stage * kStageI8);
          for (int kk = 0; kk < kPts / 32; ++kk) {
            const uint32_t off = static_cast<uint32_t>(kk * 32);  // 32 int8 = 32 B along K
            for (int t = 0; t < kSl; ++t) {
              const uint64_t da = smem_desc_k_sw64(sbase + t * 3 * kBox + off);
              for (int u = 0; u < kSl && t + u < kNAcc; ++u) {
                const uint64_t db = smem_desc_k_sw64(sbase + u * 3 * kBox + 2 * kBox + off);
                const int d = t + u;
                // the first product into accumulator d after a drain overwrites it
                const bool first = (c == c0) && (kk == 0) && (t == (d < kSl ? 0 : d - (kSl - 1)));
                mma_i8(tmem_base + static_cast<uint32_t>(d * kFJ), da, db, idesc, first ? 0u : 1u);
              }
            }
          }
          mma_commit(&empty[stage]);
          if (++stage == kStagesI8) {
            stage = 0;
            phase ^= 1u;
          }
        }
        mma_commit(tfull);
        fphase ^= 1u;
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2-5)
    const int qd = warp & 3;  // TMEM lane quarter
    const int il = qd * 32 + lane;  // I-feature within the block
    const uint32_t lane_addr = static_cast<uint32_t>(qd * 32) << 16;
    double run[kFJ];
#pragma unroll
    for (int c = 0; c < kFJ; ++c) run[c] = 0.0;
    uint32_t fphase = 0;
    for (int fl = 0; fl < nflush; ++fl) {
      mbar_wait(tfull, fphase);
      tc_fence_after();
      for (int d = 0; d < kNAcc; ++d) {
        const double wgt = ldexp(1.0, -7 * d);
#pragma unroll
        for (int h = 0; h < kFJ / 32; ++h) {
          int v[32];
          tmem_ld32i(tmem_base + lane_addr + static_cast<uint32_t>(d * kFJ + h * 32), v);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c) run[h * 32 + c] = fma(static_cast<double>(v[c]), wgt, run[h * 32 + c]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
      fphase ^= 1u;
    }
    // G[i][j] partial = 2^(E_i + E_j - 14) * run[j]
    const int fi = I * kFI + il;
    const int Ei = fi < s.D ? col_exp(__ldg(maxbits + fi)) : 0;
    double* out = Gpart + (static_cast<int64_t>(blockIdx.x) * kFI + il) * kFJ;
#pragma unroll
    for (int c = 0; c < kFJ; ++c) {
      const int fj = J * kFJ + c;
      const int Ej = fj < s.D ? col_exp(__ldg(maxbits + fj)) : 0;
      out[c] = ldexp(run[c], Ei + Ej - 14);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

// G (full symmetric) from the per-CTA tile partials; ranges summed in order.
__global__ void __launch_bounds__(256) gram_i8_reduce_kernel(const double* __restrict__ Gpart, GramI8Sched s,
                                                             double* __restrict__ G) {
  const int64_t total = static_cast<int64_t>(s.ntiles) * kFI * kFJ;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int tile = static_cast<int>(e / (kFI * kFJ));
    const int il = static_cast<int>((e / kFJ) % kFI), jc = static_cast<int>(e % kFJ);
    const int i = s.tI[tile] * kFI + il, j = s.tJ[tile] * kFJ + jc;
    if (i > j || j >= s.D) continue;  // each i <= j pair lives in exactly one tile
    double acc = 0.0;
    for (int r = 0; r < s.nranges; ++r)
      acc += Gpart[((static_cast<int64_t>(r) * s.ntiles + tile) * kFI + il) * kFJ + jc];
    G[static_cast<int64_t>(i) * s.D + j] = acc;
    G[static_cast<int64_t>(j) * s.D + i] = acc;
  }
}

}  // namespace

bool plan_gram_i8(int64_t nA, int64_t nB, int D, int num_sms, GramI8Plan& p) {
  if (D > 256 || D < 1) return false;
  p.D = D;
  p.Df = static_cast<int>(round_up(D, 128));
  p.N = nA + nB;
  p.Np = round_up(p.N > 0 ? p.N : 1, kPts);
  p.ntiles = 0;
  for (int I = 0; I < p.Df / kFI; ++I)
    for (int J = 0; J < p.Df / kFJ; ++J)
      if ((J + 1) * kFJ > I * kFI && J * kFJ < D && I * kFI < D) {
        p.tI[p.ntiles] = I;
        p.tJ[p.ntiles] = J;
        ++p.ntiles;
      }
  const int sms = num_sms > 0 ? num_sms : 148;
  int nr = sms / p.ntiles;
  if (nr < 1) nr = 1;
  const int64_t stages = p.Np / kPts;
  if (nr > stages) nr = static_cast<int>(stages);
  p.per = (stages + nr - 1) / nr * kPts;
  p.nranges = static_cast<int>((p.Np + p.per - 1) / p.per);
  p.nctas = p.ntiles * p.nranges;
  p.cm_ctas = 2 * sms;
  p.slice_bytes = static_cast<int64_t>(kSl) * p.Df * p.Np;
  p.gpart_doubles = static_cast<int64_t>(p.nctas) * kFI * kFJ;
  p.spart_doubles = static_cast<int64_t>(p.cm_ctas) * 2 * D;
  return true;
}

cudaError_t launch_gram_i8(const GramI8Plan& p, const float* A, int64_t nA, const float* B, int64_t nB,
                           unsigned* maxbits, double* Spart, int8_t* S, double* Gpart, double* G, double* SA,
                           double* SB, cudaStream_t st) {
  const int D = p.D;
  cudaError_t e;
  if ((e = cudaMemsetAsync(maxbits, 0, sizeof(unsigned) * D, st)) != cudaSuccess) return e;
  count_launch();
  colmax_kernel<<<dim3(p.cm_ctas, (D + 31) / 32), 256, 0, st>>>(A, nA, B, nB, D, maxbits, Spart);
  count_launch();
  colsum_reduce_kernel<<<(D + 255) / 256, 256, 0, st>>>(Spart, p.cm_ctas, D, SA, SB);
  // padded features (D .. Df) of every plane must read as zero slices
  if (p.Df > D) {
    for (int t = 0; t < kSl; ++t)
      if ((e = cudaMemsetAsync(S + (static_cast<int64_t>(t) * p.Df + D) * p.Np, 0,
                               static_cast<size_t>(p.Df - D) * p.Np, st)) != cudaSuccess)
        return e;
  }
  count_launch();
  slice_kernel<<<dim3(static_cast<unsigned>(p.Np / kSlT), (D + kSlT - 1) / kSlT), 256, 0, st>>>(
      A, nA, B, nB, D, p.Df, p.Np, maxbits, S);
  CUtensorMap map;
  {
    typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncFn enc = nullptr;
    if (enc == nullptr) {
      cudaDriverEntryPointQueryResult q;
      void* fn = nullptr;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess || fn == nullptr)
        return cudaErrorUnknown;
      enc = reinterpret_cast<EncFn>(fn);
    }
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(p.Np), static_cast<cuuint64_t>(kSl) * p.Df};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(p.Np)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kPts), 64u};
    const cuuint32_t estr[2] = {1u, 1u};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, S, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  GramI8Sched s{};
  s.ntiles = p.ntiles;
  s.nranges = p.nranges;
  s.per = p.per;
  s.N = p.N;
  s.Np = p.Np;
  s.D = D;
  s.Df = p.Df;
  for (int t = 0; t < p.ntiles; ++t) {
    s.tI[t] = p.tI[t];
    s.tJ[t] = p.tJ[t];
  }
  if ((e = cudaFuncSetAttribute(gram_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmemI8))) != cudaSuccess)
    return e;
  count_launch();
  gram_i8_kernel<<<p.nctas, 192, kSmemI8, st>>>(map, s, maxbits, Gpart);
  count_launch();
  gram_i8_reduce_kernel<<<148, 256, 0, st>>>(Gpart, s, G);
  return cudaGetLastError();
}

}  // namespace prohd
