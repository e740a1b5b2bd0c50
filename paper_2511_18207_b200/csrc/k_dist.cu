// k_dist.cu — K6: fused 3xTF32 tcgen05 distance + row-minimum kernel.
//
// Computes, for every row a_i of the row operand A and all columns b_j of B,
//     v_ij = ||b_j||^2 - 2 a_i . b_j        (a_i . b_j on tcgen05, 3xTF32)
//     rowmin_i = max(0, ||a_i||^2 + min_j v_ij)
// which is min_j ||a_i - b_j||^2 (Eq. (1), inner min). The
// n_A x n_B distance matrix never leaves TMEM/registers.
//
// Split products (SURVEY.md §8(a) "shared fused distance kernel"): with x = hi + lo,
// hi = x rounded to nearest TF32 (11 significant bits, K0) and lo = x - hi (|lo| <= 2^-11 |x|),
//   a.b ~= hi_a.hi_b                      one kind::tf32 MMA per 8 features
//        + [hi_a lo_a].[lo_b hi_b]        one kind::f16 MMA (bf16) per 8 features,
// the second over interleaved bf16 pairs (K doubled) so that a single instruction forms both
// correction terms hi_a.lo_b + lo_a.hi_b. Both accumulate into one fp32 TMEM accumulator.
// Error per product a_i b_i (hi.hi and the bf16 products are exact; bf16 unit roundoff
// u = 2^-8, applied to hi and to lo in each correction term):
//   |hi_a lo_b - bf16(hi_a) bf16(lo_b)| <= (2u + u^2)|hi_a||lo_b| <= (2^-7 + 2^-16)(1 + 2^-11) 2^-11 |a_i||b_i|
// twice, plus the dropped lo_a.lo_b <= 2^-22 |a_i||b_i|: in all <= 7.9e-6 |a_i||b_i| (an
// exhaustive emulation over all 2^23 mantissas of a_i = b_i gives at most 5.9e-6). So
// |a.b - dot| <= 7.9e-6 ||a|| ||b|| and |d2 - d2_exact| <= 7.9e-6 (||a||^2 + ||b||^2) plus the
// fp32 accumulation (<= ~1.9e-6 of the same norms for D/8 accumulator updates at D = 256 in the
// aligned worst case), inside the 1e-5 budget of BASELINE.json (Q17); the centring of K0 shrinks
// the norms further. (With truncated hi, |lo| < 2^-10 |x|, the worst case was 1.22e-5 of the
// product: tests/test_gpu_exact.py::test_split_worst_case_mantissas.)
// Against 3xTF32 (three TF32 MMAs) the tensor time per pair drops from 6D/P_tf32 to
// 2D/P_tf32 + 4D/P_bf16 (P_bf16 ~ 2 P_tf32): ~1.5x.
//
// Structure (persistent, 1 CTA per SM, warp-specialised; 320 threads for the single-block and
// two-A kernels, 192 for the opt-in 2-SM pair):
//   warp 0      TMA producer: per K-chunk it loads the A and B hi / pair tiles into a smem
//               ring (single block: 32 fp32 = one 128-B swizzle row, [128 x 32] A and [256 x 32]
//               B, 2 stages of 96 KB; two-A: 16-feature SWIZZLE_64B stages x3).
//   warp 1      TMEM allocator (512 columns) and MMA issuer: all 32 lanes run the issue loop and
//               an elect.sync predicate inside the tcgen05.mma / commit asm picks the issuing
//               lane (kElect; the fused bidirectional sweep below D = 192 keeps a lane-0 issuer).
//               tcgen05.mma.cta_group::1 M=128, N=256: per 8 features one kind::tf32 MMA (K=8)
//               and one kind::f16 bf16 MMA (K=16 over the pairs); commit -> smem slot free,
//               commit -> accumulator full.
//   warps 2-9   epilogue (8 warps): tcgen05.ld 32x32b.x32 (one TMEM lane = one row per thread;
//               two warps per lane quarter, each one 128-column half of the tile in the single-
//               block kernel, one accumulator per group of 4 warps in the two-A kernel),
//               v = fma(-2, acc, ||b||^2), running min in a register across all B tiles of the
//               unit; the single-block accumulator is double buffered so the epilogue of tile t
//               overlaps the MMAs of t+1.
// Work unit = (128-row block of A, contiguous range of B tiles). With one range
// the row minimum is stored; with several (small n_A) it is combined with an
// integer atomicMin on the float bits (valid since d2 >= 0).
#include "internal.cuh"
#include "sm100.cuh"

#include <cstdio>
#include <cstdlib>

namespace prohd {
namespace {

constexpr int kStages = 2;
constexpr int kThreads = 192;   // 2-SM kernel: TMA, MMA, 4 epilogue warps
constexpr int kThreads1 = 320;  // single-block kernel: TMA, MMA, 8 epilogue warps (two column halves)
constexpr uint32_t kATile = kBM * kBK * 4;                  // 16 KB
constexpr uint32_t kBTile = kBN * kBK * 4;                  // 32 KB
constexpr uint32_t kStageBytes = 2 * kATile + 2 * kBTile;   // 96 KB
constexpr uint32_t kTmemCols = 512;
constexpr size_t kSmemBytes = static_cast<size_t>(kStages) * kStageBytes + 1024 + 256;

struct Sched {
  int split3;  // k6_split3(): three TF32 MMAs (hi.hi, hi.lo, lo.hi) on fp32 lo tiles
  int64_t nA, nB;
  int nrb, nt, nsplit, tps, nk, ks_last;  // nk, ks_last: 32-feature chunks
  int nk1, ks_last1;                      // 16-feature chunks (two-A-block variant)
  int atomic_out;
};

// butterfly reduce-scatter: lane L ends with min over the warp's 32 lanes of v[L] in v[0]
__device__ __forceinline__ void warp_colmin32(float (&v)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = up ? v[i] : v[i + s];
      const float keep = up ? v[i + s] : v[i];
      const float recv = __shfl_xor_sync(0xffffffffu, send, s);
      v[i] = fminf(keep, recv);
    }
  }
}

// kBidir: the same sweep also produces column minima
// colmin[j] = min_i ||a_i - b_j||^2 (the B->A direction). Per 32-column chunk each warp
// reduces its 32 rows with a butterfly reduce-scatter, the 4 warps combine in shared
// memory, and the last warp of the tile flushes the 256 minima with global atomicMin.
template <bool kBidir, bool kElect>
__global__ void __launch_bounds__(kThreads1, 1)
    dist_rowmin_kernel(const __grid_constant__ CUtensorMap tAh, const __grid_constant__ CUtensorMap tAl,
                       const __grid_constant__ CUtensorMap tBh, const __grid_constant__ CUtensorMap tBl, Sched s,
                       const float* __restrict__ na, const float* __restrict__ nb, float* __restrict__ rowmin,
                       float* __restrict__ colmin) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ unsigned colbuf[2][kBN];  // kBidir: per-accumulator column minima (float bits)
  __shared__ __align__(16) float nbuf[2][kBN];  // column norms of the tile in each accumulator
  __shared__ unsigned tilecnt[2];
  __shared__ float rbuf[kBM];  // row minima of the second column half, combined at the unit's end

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (kBidir) {
    for (int i = threadIdx.x; i < 2 * kBN; i += blockDim.x) (&colbuf[0][0])[i] = 0x7F800000u;
    if (threadIdx.x < 2) tilecnt[threadIdx.x] = 0u;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tAh);
    tma_prefetch(&tAl);
    tma_prefetch(&tBh);
    tma_prefetch(&tBl);
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int units = s.nrb * s.nsplit;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int rb = u / s.nsplit, sp = u % s.nsplit;
        const int t0 = sp * s.tps;
        const int t1 = min(s.nt, t0 + s.tps);
        for (int t = t0; t < t1; ++t) {
          for (int c = 0; c < s.nk; ++c) {
            mbar_wait(&empty[stage], phase ^ 1u);
            uint8_t* st = smem + stage * kStageBytes;
            mbar_arrive_expect_tx(&full[stage], kStageBytes);
            tma_load_2d(st, &tAh, c * kBK, rb * kBM, &full[stage]);
            tma_load_2d(st + kATile, &tAl, c * kBK, rb * kBM, &full[stage]);
            tma_load_2d(st + 2 * kATile, &tBh, c * kBK, t * kBN, &full[stage]);
            tma_load_2d(st + 2 * kATile + kBTile, &tBl, c * kBK, t * kBN, &full[stage]);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // kElect: warp-wide issue with an elected lane (sm100.cuh mma_*_w); else lane 0 issues
    // (measured faster for the fused bidirectional sweep at D = 128, §7.1)
    auto mtf32 = [](uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t ac) {
      if constexpr (kElect) mma_tf32_w(d, a, b, id, ac); else mma_tf32(d, a, b, id, ac);
    };
    auto mbf16 = [](uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t ac) {
      if constexpr (kElect) mma_bf16_w(d, a, b, id, ac); else mma_bf16(d, a, b, id, ac);
    };
    auto mcommit = [](uint64_t* bar) {
      if constexpr (kElect) mma_commit_w(bar); else mma_commit(bar);
    };
    if (kElect || lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = idesc_tf32(kBM, kBN);
      constexpr uint32_t idesc16 = idesc_bf16(kBM, kBN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int sp = u % s.nsplit;
        const int t0 = sp * s.tps;
        const int t1 = min(s.nt, t0 + s.tps);
        for (int t = t0; t < t1; ++t) {
          mbar_wait(&tempty[acc], aphase ^ 1u);
          tc_fence_after();
          const uint32_t d = tmem_base + static_cast<uint32_t>(acc * kBN);
          for (int c = 0; c < s.nk; ++c) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t ah = smem_u32(smem + stage * kStageBytes);
            const uint32_t al = ah + kATile;
            const uint32_t bh = ah + 2 * kATile;
            const uint32_t bl = bh + kBTile;
            const int ks = (c == s.nk - 1) ? s.ks_last : (kBK / 8);
            for (int kk = 0; kk < ks; ++kk) {
              const uint32_t off = static_cast<uint32_t>(kk * 32);  // 8 tf32 = 32 B along K
              const uint64_t dah = smem_desc_k_sw128(ah + off);
              const uint64_t dal = smem_desc_k_sw128(al + off);
              const uint64_t dbh = smem_desc_k_sw128(bh + off);
              const uint64_t dbl = smem_desc_k_sw128(bl + off);
              mtf32(d, dah, dbh, idesc, (c | kk) != 0 ? 1u : 0u);  // hi_a . hi_b
              if (s.split3) {
                mtf32(d, dah, dbl, idesc, 1u);  // hi_a . lo_b
                mtf32(d, dal, dbh, idesc, 1u);  // lo_a . hi_b
              } else {
                mbf16(d, dal, dbl, idesc16, 1u);  // [hi lo]_a . [lo hi]_b
              }
            }
            mcommit(&empty[stage]);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1u;
            }
          }
          mcommit(&tfull[acc]);
          acc ^= 1;
          if (acc == 0) aphase ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- epilogue
    // 8 warps: warps 2-5 take columns 0-127 of each tile, warps 6-9 columns 128-255, each for
    // its TMEM lane quarter (warp % 4); the two halves' row minima meet in shared memory at the
    // end of the unit
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;
    const int row_local = q * 32 + lane;
    const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
    const int e = (warp - 2) * 32 + lane;  // 0..255: one column norm each
    int acc = 0;
    uint32_t aphase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int rb = u / s.nsplit, sp = u % s.nsplit;
      const int t0 = sp * s.tps;
      const int t1 = min(s.nt, t0 + s.tps);
      float rmin = __int_as_float(0x7f800000);
      const int64_t row = static_cast<int64_t>(rb) * kBM + row_local;
      // kBidir: this row's ||a||^2, or +inf for rows past nA (excluded from column minima)
      const float narow = kBidir ? (row < s.nA ? __ldg(na + row) : __int_as_float(0x7f800000)) : 0.0f;
      for (int t = t0; t < t1; ++t) {
        // the tile's column norms: loaded before the accumulator wait, staged in shared memory,
        // read back as broadcasts
        {
          const float n1 = __ldg(nb + static_cast<int64_t>(t) * kBN + e);
          mbar_wait(&tfull[acc], aphase);
          nbuf[acc][e] = n1;
          asm volatile("bar.sync 1, 256;" ::: "memory");  // the 8 epilogue warps
        }
        tc_fence_after();
        const uint32_t taddr = tmem_base + lane_addr + static_cast<uint32_t>(acc * kBN);
        const float4* nbp = reinterpret_cast<const float4*>(nbuf[acc]);
        // two 32-column chunks per TMEM wait; the 32 values of a chunk reduce as a tree
        auto chunk = [&](float (&v)[32], int cc) {
          float m[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 n4 = nbp[cc * 8 + i];
            v[4 * i + 0] = fmaf(-2.0f, v[4 * i + 0], n4.x);
            v[4 * i + 1] = fmaf(-2.0f, v[4 * i + 1], n4.y);
            v[4 * i + 2] = fmaf(-2.0f, v[4 * i + 2], n4.z);
            v[4 * i + 3] = fmaf(-2.0f, v[4 * i + 3], n4.w);
            m[i] = fminf(fminf(v[4 * i + 0], v[4 * i + 1]), fminf(v[4 * i + 2], v[4 * i + 3]));
          }
          rmin = fminf(rmin, fminf(fminf(fminf(m[0], m[1]), fminf(m[2], m[3])),
                                   fminf(fminf(m[4], m[5]), fminf(m[6], m[7]))));
          if (kBidir) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i] + narow, 0.0f);
            warp_colmin32(v, lane);
            atomicMin(&colbuf[acc][cc * 32 + lane], __float_as_uint(v[0]));
          }
        };
#pragma unroll 1
        for (int cc = half * 4; cc < half * 4 + 4; cc += 2) {
          float v0[32], v1[32];
          tmem_ld32(taddr + cc * 32, v0);
          tmem_ld32(taddr + (cc + 1) * 32, v1);
          tmem_wait_ld();
          chunk(v0, cc);
          chunk(v1, cc + 1);
        }
        tc_fence_before();
        __syncwarp();
        if (kBidir) {
          __threadfence_block();
          unsigned old = 0;
          if (lane == 0) old = atomicAdd(&tilecnt[acc], 1u);
          old = __shfl_sync(0xffffffffu, old, 0);
          if (old == 7u) {  // last of the 8 epilogue warps: flush the tile's column minima
            __threadfence_block();
            for (int j = lane; j < kBN; j += 32) {
              const unsigned val = atomicExch(&colbuf[acc][j], 0x7F800000u);
              const int64_t col = static_cast<int64_t>(t) * kBN + j;
              if (col < s.nB) atomicMin(reinterpret_cast<unsigned*>(colmin) + col, val);
            }
            if (lane == 0) tilecnt[acc] = 0u;
            __threadfence_block();
          }
          __syncwarp();
        }
        if (lane == 0) mbar_arrive(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) aphase ^= 1u;
      }
      if (half == 1) rbuf[row_local] = rmin;
      asm volatile("bar.sync 2, 256;" ::: "memory");
      if (half == 0 && row < s.nA) {
        const float d2 = fmaxf(fminf(rmin, rbuf[row_local]) + __ldg(na + row), 0.0f);
        if (s.atomic_out)
          atomicMin(reinterpret_cast<int*>(rowmin + row), __float_as_int(d2));
        else
          rowmin[row] = d2;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// ============================================================================
// 2-SM variant (cta_group::2): a CTA pair computes a 256-row block of A against
// 256-column tiles of B with one M=256, N=256 MMA per K-step. Each CTA stages its
// own 128 rows of A and its 128-column half of the B tile (64 KB per stage with
// hi+lo, 3 stages), so per SM the operand traffic per pair drops from 24 B to
// 16 B and the tensor core reads half as much of each SM's shared memory.
// Barriers: full[] lives in the leader (rank 0) and counts both CTAs' TMA bytes
// (2-SM TMA); empty[] and tfull[] exist in both CTAs and are signalled by the
// leader's multicast tcgen05.commit; tempty[] lives in the leader and counts the
// 8 epilogue warps of the pair.
// ============================================================================
constexpr int kStages2 = 3;
constexpr uint32_t kHalf = 128 * kBK * 4;     // 16 KB: 128 rows x 32 fp32
constexpr uint32_t kStage2Bytes = 4 * kHalf;  // A_hi, A_lo, B_hi, B_lo halves
constexpr size_t kSmem2 = static_cast<size_t>(kStages2) * kStage2Bytes + 1024 + 256;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    dist_rowmin_2sm_kernel(const __grid_constant__ CUtensorMap tAh, const __grid_constant__ CUtensorMap tAl,
                           const __grid_constant__ CUtensorMap tBh, const __grid_constant__ CUtensorMap tBl, Sched s,
                           const float* __restrict__ na, const float* __restrict__ nb, float* __restrict__ rowmin) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages2 * kStage2Bytes);
  uint64_t* empty = full + kStages2;
  uint64_t* tfull = empty + kStages2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ __align__(16) float nbuf[2][kBN];  // column norms of the tile in each accumulator

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = static_cast<int>(cluster_id_x());
  const int ncl = static_cast<int>(nclusters_x());
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages2; ++i) {
      mbar_init(&full[i], 2);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tAh);
    tma_prefetch(&tAl);
    tma_prefetch(&tBh);
    tma_prefetch(&tBl);
  }
  if (warp == 1) tmem_alloc_2sm<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int units = s.nrb * s.nsplit;  // nrb counts 256-row blocks here

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cid; u < units; u += ncl) {
        const int pb = u / s.nsplit, sp = u % s.nsplit;
        const int t0 = sp * s.tps;
        const int t1 = min(s.nt, t0 + s.tps);
        const int arow = pb * 256 + static_cast<int>(rank) * 128;
        for (int t = t0; t < t1; ++t) {
          const int brow = t * kBN + static_cast<int>(rank) * 128;
          for (int c = 0; c < s.nk; ++c) {
            mbar_wait(&empty[stage], phase ^ 1u);
            const uint32_t fl = mapa(smem_u32(&full[stage]), 0);
            if (leader)
              mbar_arrive_expect_tx(&full[stage], 2 * kStage2Bytes);
            else
              mbar_arrive_cluster(fl);
            uint8_t* st = smem + stage * kStage2Bytes;
            tma_load_2d_2sm(st, &tAh, c * kBK, arow, fl);
            tma_load_2d_2sm(st + kHalf, &tAl, c * kBK, arow, fl);
            tma_load_2d_2sm(st + 2 * kHalf, &tBh, c * kBK, brow, fl);
            tma_load_2d_2sm(st + 3 * kHalf, &tBl, c * kBK, brow, fl);
            if (++stage == kStages2) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = idesc_tf32(256, kBN);
      constexpr uint32_t idesc16 = idesc_bf16(256, kBN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      for (int u = cid; u < units; u += ncl) {
        const int sp = u % s.nsplit;
        const int t0 = sp * s.tps;
        const int t1 = min(s.nt, t0 + s.tps);
        for (int t = t0; t < t1; ++t) {
          mbar_wait(&tempty[acc], aphase ^ 1u);
          tc_fence_after();
          const uint32_t d = tmem_base + static_cast<uint32_t>(acc * kBN);
          for (int c = 0; c < s.nk; ++c) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t ah = smem_u32(smem + stage * kStage2Bytes);
            const uint32_t al = ah + kHalf;
            const uint32_t bh = ah + 2 * kHalf;
            const uint32_t bl = ah + 3 * kHalf;
            const int ks = (c == s.nk - 1) ? s.ks_last : (kBK / 8);
            for (int kk = 0; kk < ks; ++kk) {
              const uint32_t off = static_cast<uint32_t>(kk * 32);
              const uint64_t dah = smem_desc_k_sw128(ah + off);
              const uint64_t dal = smem_desc_k_sw128(al + off);
              const uint64_t dbh = smem_desc_k_sw128(bh + off);
              const uint64_t dbl = smem_desc_k_sw128(bl + off);
              mma_tf32_2sm(d, dah, dbh, idesc, (c | kk) != 0 ? 1u : 0u);  // hi_a . hi_b
              if (s.split3) {
                mma_tf32_2sm(d, dah, dbl, idesc, 1u);
                mma_tf32_2sm(d, dal, dbh, idesc, 1u);
              } else {
                mma_bf16_2sm(d, dal, dbl, idesc16, 1u);  // [hi lo]_a . [lo hi]_b
              }
            }
            mma_commit_2sm_mc(&empty[stage], 0x3);
            if (++stage == kStages2) {
              stage = 0;
              phase ^= 1u;
            }
          }
          mma_commit_2sm_mc(&tfull[acc], 0x3);
          acc ^= 1;
          if (acc == 0) aphase ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    const int row_local = q * 32 + lane;
    const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t te[2] = {mapa(smem_u32(&tempty[0]), 0), mapa(smem_u32(&tempty[1]), 0)};
    int acc = 0;
    uint32_t aphase = 0;
    for (int u = cid; u < units; u += ncl) {
      const int pb = u / s.nsplit, sp = u % s.nsplit;
      const int t0 = sp * s.tps;
      const int t1 = min(s.nt, t0 + s.tps);
      float rmin = __int_as_float(0x7f800000);
      for (int t = t0; t < t1; ++t) {
        // the tile's column norms: loaded before the accumulator wait, staged in shared memory
        // (one 16-B piece per thread per accumulator buffer), read back as broadcasts
        {
          const int e = q * 32 + lane;  // 0..127: two floats each
          const float2 n2 = __ldg(reinterpret_cast<const float2*>(nb + static_cast<int64_t>(t) * kBN) + e);
          mbar_wait(&tfull[acc], aphase);
          reinterpret_cast<float2*>(nbuf[acc])[e] = n2;
          asm volatile("bar.sync 1, 128;" ::: "memory");  // the 4 epilogue warps
        }
        tc_fence_after();
        const uint32_t taddr = tmem_base + lane_addr + static_cast<uint32_t>(acc * kBN);
        const float4* nbp = reinterpret_cast<const float4*>(nbuf[acc]);
#pragma unroll 1
        for (int cc = 0; cc < kBN / 32; ++cc) {
          float v[32];
          tmem_ld32(taddr + cc * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 n4 = nbp[cc * 8 + i];
            rmin = fminf(rmin, fmaf(-2.0f, v[4 * i + 0], n4.x));
            rmin = fminf(rmin, fmaf(-2.0f, v[4 * i + 1], n4.y));
            rmin = fminf(rmin, fmaf(-2.0f, v[4 * i + 2], n4.z));
            rmin = fminf(rmin, fmaf(-2.0f, v[4 * i + 3], n4.w));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(te[acc]);
        acc ^= 1;
        if (acc == 0) aphase ^= 1u;
      }
      const int64_t row = static_cast<int64_t>(pb) * 256 + static_cast<int64_t>(rank) * 128 + row_local;
      if (row < s.nA) {
        const float d2 = fmaxf(rmin + __ldg(na + row), 0.0f);
        if (s.atomic_out)
          atomicMin(reinterpret_cast<int*>(rowmin + row), __float_as_int(d2));
        else
          rowmin[row] = d2;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm<kTmemCols>(tmem_base);
  }
}


// ============================================================================
// Two-A-block variant (directed sweep only): one CTA computes TWO 128-row blocks of A against
// each 256-column tile of B, one fp32 accumulator each (all 512 TMEM columns, so the epilogue of
// a tile is not overlapped with the next tile's MMAs). Stages of 16 features (SWIZZLE_64B rows):
// A1 and A2 hi/pr 4 x 8 KB + B hi/pc 2 x 16 KB = 64 KB, three in flight. Per pair and feature the
// operand stream drops from 96 KB / (128 x 256 x 32) to 64 KB / (256 x 256 x 16): 2/3.
// ============================================================================
constexpr int kBK2 = 16;
constexpr int kThreadsA2 = 320;  // TMA, MMA, 8 epilogue warps
constexpr int kStagesA2 = 3;
constexpr uint32_t kA2Tile = 128 * kBK2 * 4;                    // 8 KB
constexpr uint32_t kB2Tile = kBN * kBK2 * 4;                    // 16 KB
constexpr uint32_t kStageA2Bytes = 4 * kA2Tile + 2 * kB2Tile;   // 64 KB
constexpr size_t kSmemA2 = static_cast<size_t>(kStagesA2) * kStageA2Bytes + 1024 + 256;

// kBidir: column minima too (as the single-block kernel), combined over the tile's 256 rows
template <bool kBidir>
__global__ void __launch_bounds__(kThreadsA2, 1)
    dist_rowmin_2a_kernel(const __grid_constant__ CUtensorMap tAh, const __grid_constant__ CUtensorMap tAl,
                          const __grid_constant__ CUtensorMap tBh, const __grid_constant__ CUtensorMap tBl, Sched s,
                          const float* __restrict__ na, const float* __restrict__ nb, float* __restrict__ rowmin,
                          float* __restrict__ colmin) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStagesA2 * kStageA2Bytes);
  uint64_t* empty = full + kStagesA2;
  uint64_t* tfull = empty + kStagesA2;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  __shared__ __align__(16) float nbuf[2][kBN];  // column norms, double-buffered by tile parity
  __shared__ unsigned colbuf[2][kBN];            // kBidir: the tile's column minima (float bits)
  __shared__ unsigned tilecnt[2];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (kBidir) {
    for (int i = threadIdx.x; i < 2 * kBN; i += blockDim.x) (&colbuf[0][0])[i] = 0x7F800000u;
    if (threadIdx.x < 2) tilecnt[threadIdx.x] = 0u;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStagesA2; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tempty[0], 8);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tAh);
    tma_prefetch(&tAl);
    tma_prefetch(&tBh);
    tma_prefetch(&tBl);
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int units = s.nrb * s.nsplit;  // nrb counts 256-row block pairs here

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int pb = u / s.nsplit, sp = u % s.nsplit;
        const int t0 = sp * s.tps;
        const int t1 = min(s.nt, t0 + s.tps);
        for (int t = t0; t < t1; ++t) {
          for (int c = 0; c < s.nk1; ++c) {
            mbar_wait(&empty[stage], phase ^ 1u);
            uint8_t* st = smem + stage * kStageA2Bytes;
            mbar_arrive_expect_tx(&full[stage], kStageA2Bytes);
            tma_load_2d(st, &tAh, c * kBK2, pb * 256, &full[stage]);
            tma_load_2d(st + kA2Tile, &tAl, c * kBK2, pb * 256, &full[stage]);
            tma_load_2d(st + 2 * kA2Tile, &tAh, c * kBK2, pb * 256 + 128, &full[stage]);
            tma_load_2d(st + 3 * kA2Tile, &tAl, c * kBK2, pb * 256 + 128, &full[stage]);
            tma_load_2d(st + 4 * kA2Tile, &tBh, c * kBK2, t * kBN, &full[stage]);
            tma_load_2d(st + 4 * kA2Tile + kB2Tile, &tBl, c * kBK2, t * kBN, &full[stage]);
            if (++stage == kStagesA2) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    {
      // ------------------------------------------------------------ MMA issuer (warp-wide, elected lane issues)
      constexpr uint32_t idesc = idesc_tf32(kBM, kBN);
      constexpr uint32_t idesc16 = idesc_bf16(kBM, kBN);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t tph = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int sp = u % s.nsplit;
        const int t0 = sp * s.tps;
        const int t1 = min(s.nt, t0 + s.tps);
        for (int t = t0; t < t1; ++t) {
          mbar_wait(&tempty[0], tph ^ 1u);  // the epilogue has drained both accumulators
          tc_fence_after();
          const uint32_t d0 = tmem_base, d1 = tmem_base + static_cast<uint32_t>(kBN);
          for (int c = 0; c < s.nk1; ++c) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t a1h = smem_u32(smem + stage * kStageA2Bytes);
            const uint32_t a1l = a1h + kA2Tile, a2h = a1h + 2 * kA2Tile, a2l = a1h + 3 * kA2Tile;
            const uint32_t bh = a1h + 4 * kA2Tile, bl = bh + kB2Tile;
            const int ks = (c == s.nk1 - 1) ? s.ks_last1 : (kBK2 / 8);
            for (int kk = 0; kk < ks; ++kk) {
              const uint32_t off = static_cast<uint32_t>(kk * 32);
              const uint64_t dbh = smem_desc_k_sw64(bh + off), dbl = smem_desc_k_sw64(bl + off);
              const uint32_t acc = (c | kk) != 0 ? 1u : 0u;
              const uint64_t da1h = smem_desc_k_sw64(a1h + off), da1l = smem_desc_k_sw64(a1l + off);
              const uint64_t da2h = smem_desc_k_sw64(a2h + off), da2l = smem_desc_k_sw64(a2l + off);
              if (!s.split3) {
                // issue order matters for power: alternating kinds per accumulator ran at a 1490 MHz
                // median clock in the power-capped benchmark, both TF32 MMAs first at 1035 MHz
                mma_tf32_w(d0, da1h, dbh, idesc, acc);
                mma_bf16_w(d0, da1l, dbl, idesc16, 1u);
                mma_tf32_w(d1, da2h, dbh, idesc, acc);
                mma_bf16_w(d1, da2l, dbl, idesc16, 1u);
              } else {
                mma_tf32_w(d0, da1h, dbh, idesc, acc);
                mma_tf32_w(d0, da1h, dbl, idesc, 1u);
                mma_tf32_w(d0, da1l, dbh, idesc, 1u);
                mma_tf32_w(d1, da2h, dbh, idesc, acc);
                mma_tf32_w(d1, da2h, dbl, idesc, 1u);
                mma_tf32_w(d1, da2l, dbh, idesc, 1u);
              }
            }
            mma_commit_w(&empty[stage]);
            if (++stage == kStagesA2) {
              stage = 0;
              phase ^= 1u;
            }
          }
          mma_commit_w(&tfull[0]);
          tph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- epilogue
    // 8 warps: warps 2-5 drain accumulator 0 (rows of A block 1), warps 6-9 accumulator 1
    const int q = warp & 3;
    const int a2 = (warp - 2) >> 2;
    const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
    const int e = (warp - 2) * 32 + lane;  // 0..255: one column norm each
    uint32_t tph = 0;
    int tb = 0;  // nbuf parity
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int pb = u / s.nsplit, sp = u % s.nsplit;
      const int t0 = sp * s.tps;
      const int t1 = min(s.nt, t0 + s.tps);
      float rm = __int_as_float(0x7f800000);
      const int64_t myrow = static_cast<int64_t>(pb) * 256 + a2 * 128 + q * 32 + lane;
      // kBidir: this row's ||a||^2, or +inf for rows past nA (excluded from column minima)
      const float narow = kBidir ? (myrow < s.nA ? __ldg(na + myrow) : __int_as_float(0x7f800000)) : 0.0f;
      for (int t = t0; t < t1; ++t) {
        {
          const float n1 = __ldg(nb + static_cast<int64_t>(t) * kBN + e);
          mbar_wait(&tfull[0], tph);
          nbuf[tb][e] = n1;
          asm volatile("bar.sync 1, 256;" ::: "memory");
        }
        tc_fence_after();
        const float4* nbp = reinterpret_cast<const float4*>(nbuf[tb]);
        const uint32_t taddr = tmem_base + lane_addr + static_cast<uint32_t>(a2 * kBN);
        auto chunk = [&](float (&v)[32], int cc) {
          float m[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 n4 = nbp[cc * 8 + i];
            v[4 * i + 0] = fmaf(-2.0f, v[4 * i + 0], n4.x);
            v[4 * i + 1] = fmaf(-2.0f, v[4 * i + 1], n4.y);
            v[4 * i + 2] = fmaf(-2.0f, v[4 * i + 2], n4.z);
            v[4 * i + 3] = fmaf(-2.0f, v[4 * i + 3], n4.w);
            m[i] = fminf(fminf(v[4 * i + 0], v[4 * i + 1]), fminf(v[4 * i + 2], v[4 * i + 3]));
          }
          rm = fminf(rm, fminf(fminf(fminf(m[0], m[1]), fminf(m[2], m[3])),
                               fminf(fminf(m[4], m[5]), fminf(m[6], m[7]))));
          if (kBidir) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i] + narow, 0.0f);
            warp_colmin32(v, lane);
            atomicMin(&colbuf[tb][cc * 32 + lane], __float_as_uint(v[0]));
          }
        };
#pragma unroll 1
        for (int cc = 0; cc < kBN / 32; cc += 2) {
          float v0[32], v1[32];
          tmem_ld32(taddr + cc * 32, v0);
          tmem_ld32(taddr + (cc + 1) * 32, v1);
          tmem_wait_ld();
          chunk(v0, cc);
          chunk(v1, cc + 1);
        }
        tc_fence_before();
        __syncwarp();
        if (kBidir) {
          __threadfence_block();
          unsigned old = 0;
          if (lane == 0) old = atomicAdd(&tilecnt[tb], 1u);
          old = __shfl_sync(0xffffffffu, old, 0);
          if (old == 7u) {  // last of the 8 epilogue warps: flush the tile's column minima
            __threadfence_block();
            for (int j = lane; j < kBN; j += 32) {
              const unsigned val = atomicExch(&colbuf[tb][j], 0x7F800000u);
              const int64_t col = static_cast<int64_t>(t) * kBN + j;
              if (col < s.nB) atomicMin(reinterpret_cast<unsigned*>(colmin) + col, val);
            }
            if (lane == 0) tilecnt[tb] = 0u;
            __threadfence_block();
          }
          __syncwarp();
        }
        if (lane == 0) mbar_arrive(&tempty[0]);
        tph ^= 1u;
        tb ^= 1;
      }
      const int64_t row = static_cast<int64_t>(pb) * 256 + a2 * 128 + q * 32 + lane;
      if (row < s.nA) {
        const float d2 = fmaxf(rm + __ldg(na + row), 0.0f);
        if (s.atomic_out)
          atomicMin(reinterpret_cast<int*>(rowmin + row), __float_as_int(d2));
        else
          rowmin[row] = d2;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

}  // namespace

// Variants (one B200, tools/time_exact.py). The 2-SM pair (cta_group::2) was faster per clock
// with three TF32 MMAs but lost in the sustained, power-capped benchmark; with the TF32 + bf16
// MMAs it measures the same as the single-CTA kernel (547 vs 549 Gpair/s) and stays opt-in.
// Directed sweeps use the two-A-block kernel for D >= 128 (65536 x 262144, D = 256: 549 -> 627
// Gpair/s; D = 128: 1048 -> 1126) and the single-block kernel below (faster at small D, where the
// epilogue is not hidden behind fewer MMAs: D = 64 2118 vs 1896). The fused bidirectional sweep
// keeps the single-block kernel: its column-minimum epilogue is heavier and, not overlapped in the
// two-A kernel, made it slower (D = 256: 34.5 vs 31.5 ms for 65536 x 262144; the two-A kBidir
// instantiation is kept for A/B). option k6_variant = 1 | 3 (two-A) | 2 (2-SM pair, directed) forces a variant.
static int dist_variant(int D) {
  const long long v = opt(OPT_K6_VARIANT);  // 2: CTA pair, 3: two A blocks per CTA, 1: single
  if (v >= 1 && v <= 3) return static_cast<int>(v);
  return D >= 128 ? 3 : 1;
}

int dist_b_box_rows(int D, bool bidir) { return (!bidir && dist_variant(D) == 2) ? 128 : kBN; }
bool k6_split3() {
  return opt(OPT_K6_SPLIT3) == 1;
}

static bool bidir_2a() {
  return opt(OPT_K6_BIDIR_2A) == 1;  // dev A/B: fused bidirectional sweep on the two-A kernel
}
int dist_box_inner(int D, bool bidir) { return ((!bidir || bidir_2a()) && dist_variant(D) == 3) ? kBK2 : kBK; }

cudaError_t launch_dist_rowmin(const DistArgs& a, cudaStream_t st) {
  const bool pair = dist_variant(a.D) == 2 && a.num_sms >= 2 && a.colmin == nullptr;
  const bool twoa = dist_variant(a.D) == 3 && (a.colmin == nullptr || bidir_2a());
  const int rows_per_unit = (pair || twoa) ? 256 : kBM;
  const int ctas_per_unit = pair ? 2 : 1;
  Sched s{};
  s.split3 = k6_split3() ? 1 : 0;
  s.nA = a.nA;
  s.nB = a.nB;
  s.nrb = static_cast<int>((a.nA + rows_per_unit - 1) / rows_per_unit);
  s.nt = static_cast<int>((a.nB + kBN - 1) / kBN);
  s.nk = (a.D + kBK - 1) / kBK;
  s.ks_last = ((a.D - (s.nk - 1) * kBK) + 7) / 8;
  s.nk1 = (a.D + kBK2 - 1) / kBK2;
  s.ks_last1 = ((a.D - (s.nk1 - 1) * kBK2) + 7) / 8;
  const int slots = a.num_sms / ctas_per_unit;  // concurrent units
  // Column splits: units (row block, column range) are dealt round-robin to the persistent
  // CTAs, so the sweep takes ceil(units / slots) rounds of (tps + ~0.5) tile times (the half
  // tile: a unit's pipeline fill / drain and row-minimum merge). Small A (subset HD: 100-250
  // row blocks) needs splits to fill 148 SMs, and the split count decides the last round's
  // occupancy: pick the cheapest of 1..64 splits (ties to fewer: fewer atomic merges).
  int nsplit = 1;
  {
    if (opt(OPT_K6_SPLITS_2X) == 1) {  // dev A/B: the old fill-twice rule
      nsplit = (2 * slots + s.nrb - 1) / s.nrb;
    } else {
      double best = 0.0;
      for (int ns = 1; ns <= 64 && ns <= s.nt; ++ns) {
        const int tps = (s.nt + ns - 1) / ns;
        const int nsa = (s.nt + tps - 1) / tps;
        const int64_t u = static_cast<int64_t>(s.nrb) * nsa;
        const double cost = static_cast<double>((u + slots - 1) / slots) * (tps + 0.5);
        if (ns == 1 || cost < best * 0.995) {
          best = cost;
          nsplit = nsa;
        }
      }
    }
  }
  if (nsplit < 1) nsplit = 1;
  if (nsplit > s.nt) nsplit = s.nt;
  s.tps = (s.nt + nsplit - 1) / nsplit;
  s.nsplit = (s.nt + s.tps - 1) / s.tps;
  s.atomic_out = s.nsplit > 1 ? 1 : 0;
  if (s.atomic_out) {
    cudaError_t e = cudaMemsetAsync(a.rowmin, 0x7F, sizeof(float) * a.nA, st);  // 3.39e38 (finite, > any d2)
    if (e != cudaSuccess) return e;
  }
  const int units = s.nrb * s.nsplit;
  const int nunits = units < slots ? units : slots;
  if (twoa) {
    if (a.colmin != nullptr) {
      cudaError_t e = cudaMemsetAsync(a.colmin, 0x7F, sizeof(float) * a.nB, st);
      if (e != cudaSuccess) return e;
    }
    auto kern = a.colmin != nullptr ? dist_rowmin_2a_kernel<true> : dist_rowmin_2a_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemA2));
    if (e != cudaSuccess) return e;
    count_launch();
    kern<<<nunits, kThreadsA2, kSmemA2, st>>>(a.maps[0], a.maps[1], a.maps[2], a.maps[3], s, a.na, a.nb, a.rowmin,
                                             a.colmin);
    return cudaGetLastError();
  }
  if (pair) {
    cudaError_t e = cudaFuncSetAttribute(dist_rowmin_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kSmem2));
    if (e != cudaSuccess) return e;
    count_launch();
    dist_rowmin_2sm_kernel<<<2 * nunits, kThreads, kSmem2, st>>>(a.maps[0], a.maps[1], a.maps[2], a.maps[3], s,
                                                                   a.na, a.nb, a.rowmin);
    return cudaGetLastError();
  }
  if (a.colmin != nullptr) {
    cudaError_t e = cudaMemsetAsync(a.colmin, 0x7F, sizeof(float) * a.nB, st);
    if (e != cudaSuccess) return e;
    // lane-0 MMA issue below D = 192 (D = 128 undirected cfg3: 255 -> 243 ms), elected above
    auto kern = a.D < 192 ? dist_rowmin_kernel<true, false> : dist_rowmin_kernel<true, true>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes));
    if (e != cudaSuccess) return e;
    count_launch();
    kern<<<nunits, kThreads1, kSmemBytes, st>>>(a.maps[0], a.maps[1], a.maps[2], a.maps[3], s, a.na, a.nb, a.rowmin,
                                                a.colmin);
    return cudaGetLastError();
  }
  {
    cudaError_t e = cudaFuncSetAttribute(dist_rowmin_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kSmemBytes));
    if (e != cudaSuccess) return e;
  }
  count_launch();
  dist_rowmin_kernel<false, true><<<nunits, kThreads1, kSmemBytes, st>>>(a.maps[0], a.maps[1], a.maps[2], a.maps[3], s,
                                                                   a.na, a.nb, a.rowmin, nullptr);
  return cudaGetLastError();
}

}  // namespace prohd
