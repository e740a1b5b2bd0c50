// k_dist.cu — K6: fused split-precision tcgen05 distance + row-minimum kernel.
//
// Computes, for every row a_i of the row operand A and all columns b_j of B,
//     v_ij = ||b_j||^2 - 2 a_i . b_j        (a_i . b_j on tcgen05)
//     rowmin_i = max(0, ||a_i||^2 + min_j v_ij)
// which is min_j ||a_i - b_j||^2 (Eq. (1), inner min). The
// n_A x n_B distance matrix never leaves TMEM/registers.
//
// Split products (SURVEY.md §8(a) "shared fused distance kernel"): K0 writes each coordinate y
// (centred) as hi + lo on two arrays H and L, and each 32-byte K-step issues THREE MMAs into
// one fp32 TMEM accumulator, hi_a.hi_b + hi_a.lo_b + lo_a.hi_b (lo.lo dropped):
//   F16 (default):  kind::f16 on fp16 hi/lo of the power-of-two-scaled coordinates s*y, 16
//                   features per K-step. hi has 11 significant bits and lo the next 11, the same
//                   split as 3xTF32, at twice the TF32 tensor rate and half its operand bytes.
//                   Error per product <= 3 2^-22 |a_i||b_i| (lo's fp16 rounding on both sides,
//                   the dropped lo.lo), plus the fp16 subnormal floor 2^-25/s per coordinate that
//                   K0's scale mode keeps below 3e-6 of ||a||^2+||b||^2 (internal.cuh).
//   TF32 (option k6_split3, the literal north-star 3xTF32): kind::tf32 on fp32 hi (RN to TF32)
//                   and lo, 8 features per K-step.
// The accumulator is scaled by s_i s_j (row and column scales, powers of two, exact): the
// epilogue forms v_ij = fma(-2 / (s_i s_j), acc_ij, ||b_j||^2) — with one scale per set that is
// a per-row constant (the same two instructions per element as unscaled); with per-row scales
// (K0's wide-dynamic-range mode) one extra multiply by 1/s_j per element.
// fp32 accumulation (the tensor core truncates each MMA's sum to the accumulator's precision)
// adds up to ~2^-23 |acc| per MMA; measured on constant-mantissa rows (tools/split_probe.py)
// this is the dominant term at D = 256.
//
// Structure (persistent, 1 CTA per SM, warp-specialised, 320 threads):
//   warp 0      TMA producer: 64-byte box rows (32 fp16 or 16 fp32 features), SWIZZLE_64B,
//               H and L tiles of A and B per stage.
//   warp 1      TMEM allocator (512 columns) and MMA issuer: all 32 lanes run the issue loop
//               and an elect.sync predicate inside the tcgen05.mma / commit asm picks the issuing
//               lane (kElect; the fused bidirectional sweep below D = 192 keeps a lane-0 issuer).
//   warps 2-9   epilogue (8 warps): tcgen05.ld 32x32b.x32 (one TMEM lane = one row per thread),
//               v = fma(k_i, acc, ||b||^2), running min in a register across all B tiles of the
//               unit.
// Three kernels: the single-block kernel (one 128-row block of A per CTA, M=128 N=256, the
// accumulator double-buffered so the epilogue of tile t overlaps the MMAs of t+1; 4 stages of
// 48 KB; directed sweeps at D < 128 and the fused bidirectional sweep), the two-A kernel (two
// 128-row blocks against each B tile, both accumulators = all 512 TMEM columns, 3 stages of
// 64 KB: 2/3 of the operand bytes per pair; literal 3xTF32 and option k6_variant 3), and the
// CTA-pair kernel (2-CTA cluster, M=256 N=256 cta_group::2, B split across the pair, 256-column
// accumulators double-buffered; see its header below) — the default for fp16 sweeps at
// D >= 128 (directed: the bench's dominant kernel; fused bidirectional: kBidir).
// Work unit = (row block, contiguous range of B tiles). With one range the row minimum is
// stored; with several (small n_A) it is combined with an integer atomicMin on the float bits
// (valid since d2 >= 0).
#include "internal.cuh"
#include "sm100.cuh"

#include <cstdio>
#include <cstdlib>

namespace prohd {
namespace {

constexpr uint32_t kRowBytes = 64;                      // one SWIZZLE_64B box row
constexpr uint32_t kATile = kBM * kRowBytes;           // 8 KB: 128 rows
constexpr uint32_t kBTile = kBN * kRowBytes;           // 16 KB: 256 rows
constexpr uint32_t kTmemCols = 512;
constexpr int kThreads1 = 320;  // TMA, MMA, 8 epilogue warps
constexpr int kStages1 = 4;
constexpr uint32_t kStage1Bytes = 2 * kATile + 2 * kBTile;  // 48 KB: A_H, A_L, B_H, B_L
constexpr size_t kSmem1 = static_cast<size_t>(kStages1) * kStage1Bytes + 1024 + 256;
constexpr int kThreadsA2 = 320;
constexpr int kStagesA2 = 3;
constexpr uint32_t kStageA2Bytes = 4 * kATile + 2 * kBTile;  // 64 KB: A1_H, A1_L, A2_H, A2_L, B_H, B_L
constexpr size_t kSmemA2 = static_cast<size_t>(kStagesA2) * kStageA2Bytes + 1024 + 256;

struct Sched {
  int64_t nA, nB;
  int nrb, nt, nsplit, tps;
  int nk, ks_last;  // 64-byte stages over the features, 32-byte K-steps in the last stage
  int atomic_out;
  int D;
};

// the three split MMAs of one 32-byte K-step into accumulator d
template <bool kF16, bool kElect>
__device__ __forceinline__ void mma3(uint32_t d, uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl, uint32_t acc) {
  using namespace sm100;
  constexpr uint32_t id = kF16 ? idesc_f16(kBM, kBN) : idesc_tf32(kBM, kBN);
  if constexpr (kF16) {
    if constexpr (kElect) {
      mma_bf16_w(d, ah, bh, id, acc);  // kind::f16; the idesc selects fp16 operands
      mma_bf16_w(d, ah, bl, id, 1u);
      mma_bf16_w(d, al, bh, id, 1u);
    } else {
      mma_bf16(d, ah, bh, id, acc);
      mma_bf16(d, ah, bl, id, 1u);
      mma_bf16(d, al, bh, id, 1u);
    }
  } else {
    if constexpr (kElect) {
      mma_tf32_w(d, ah, bh, id, acc);
      mma_tf32_w(d, ah, bl, id, 1u);
      mma_tf32_w(d, al, bh, id, 1u);
    } else {
      mma_tf32(d, ah, bh, id, acc);
      mma_tf32(d, ah, bl, id, 1u);
      mma_tf32(d, al, bh, id, 1u);
    }
  }
}

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

// Epilogue helpers. Scale factors: global mode k = -2 / (s_i s_B) per row; per-row mode
// k = -2 / s_i and u_j = 1 / s_j per column (staged with the column norms).
struct EpiScale {
  bool perrow;
  float k;  // this thread's row factor
};
__device__ __forceinline__ EpiScale epi_scale(bool f16, const PrepStats* sta, const PrepStats* stb, const float* sa,
                                              const float* sb, int64_t row, int64_t nA, int D) {
  EpiScale e{false, -2.0f};
  if (!f16) return e;
  e.perrow = prep_mode_perrow(sta, stb, D);
  const float si = row < nA ? __ldg(sa + row) : 1.0f;
  e.k = e.perrow ? -2.0f / si : (-2.0f / si) / __ldg(sb);
  return e;
}

// v[0..31] <- fma(k, acc (* u_j), ||b_j||^2) for one 32-column chunk; returns the chunk minimum
template <bool kPerRow>
__device__ __forceinline__ float epi_chunk(float (&v)[32], float k, const float4* nbp, const float4* ubp) {
  float m[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float4 n4 = nbp[i];
    if constexpr (kPerRow) {
      const float4 u4 = ubp[i];
      v[4 * i + 0] = fmaf(k, v[4 * i + 0] * u4.x, n4.x);
      v[4 * i + 1] = fmaf(k, v[4 * i + 1] * u4.y, n4.y);
      v[4 * i + 2] = fmaf(k, v[4 * i + 2] * u4.z, n4.z);
      v[4 * i + 3] = fmaf(k, v[4 * i + 3] * u4.w, n4.w);
    } else {
      v[4 * i + 0] = fmaf(k, v[4 * i + 0], n4.x);
      v[4 * i + 1] = fmaf(k, v[4 * i + 1], n4.y);
      v[4 * i + 2] = fmaf(k, v[4 * i + 2], n4.z);
      v[4 * i + 3] = fmaf(k, v[4 * i + 3], n4.w);
    }
    m[i] = fminf(fminf(v[4 * i + 0], v[4 * i + 1]), fminf(v[4 * i + 2], v[4 * i + 3]));
  }
  return fminf(fminf(fminf(m[0], m[1]), fminf(m[2], m[3])), fminf(fminf(m[4], m[5]), fminf(m[6], m[7])));
}

// kBidir: the same sweep also produces column minima
// colmin[j] = min_i ||a_i - b_j||^2 (the B->A direction). Per 32-column chunk each warp
// reduces its 32 rows with a butterfly reduce-scatter, the warps combine in shared
// memory, and the last warp of the tile flushes the 256 minima with global atomicMin.
template <bool kBidir, bool kElect, bool kF16>
__global__ void __launch_bounds__(kThreads1, 1)
    dist_rowmin_kernel(const __grid_constant__ CUtensorMap tAh, const __grid_constant__ CUtensorMap tAl,
                       const __grid_constant__ CUtensorMap tBh, const __grid_constant__ CUtensorMap tBl, Sched s,
                       const float* __restrict__ na, const float* __restrict__ nb, const float* __restrict__ sa,
                       const float* __restrict__ sb, const PrepStats* sta, const PrepStats* stb,
                       float* __restrict__ rowmin, float* __restrict__ colmin) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages1 * kStage1Bytes);
  uint64_t* empty = full + kStages1;
  uint64_t* tfull = empty + kStages1;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ unsigned colbuf[2][kBN];  // kBidir: per-accumulator column minima (float bits)
  __shared__ __align__(16) float nbuf[2][kBN];  // column norms of the tile in each accumulator
  __shared__ __align__(16) float ubuf[2][kBN];  // per-row scale mode: 1 / s_j of the tile's columns
  __shared__ unsigned tilecnt[2];
  __shared__ float rbuf[kBM];  // row minima of the second column half, combined at the unit's end

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (kBidir) {
    for (int i = threadIdx.x; i < 2 * kBN; i += blockDim.x) (&colbuf[0][0])[i] = 0x7F800000u;
    if (threadIdx.x < 2) tilecnt[threadIdx.x] = 0u;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages1; ++i) {
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
            uint8_t* st = smem + stage * kStage1Bytes;
            mbar_arrive_expect_tx(&full[stage], kStage1Bytes);
            tma_load_2d(st, &tAh, c * 16, rb * kBM, &full[stage]);
            tma_load_2d(st + kATile, &tAl, c * 16, rb * kBM, &full[stage]);
            tma_load_2d(st + 2 * kATile, &tBh, c * 16, t * kBN, &full[stage]);
            tma_load_2d(st + 2 * kATile + kBTile, &tBl, c * 16, t * kBN, &full[stage]);
            if (++stage == kStages1) {
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
    auto mcommit = [](uint64_t* bar) {
      if constexpr (kElect) mma_commit_w(bar); else mma_commit(bar);
    };
    if (kElect || lane == 0) {
      // ------------------------------------------------------------ MMA issuer
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
            const uint32_t ah = smem_u32(smem + stage * kStage1Bytes);
            const uint32_t al = ah + kATile;
            const uint32_t bh = ah + 2 * kATile;
            const uint32_t bl = bh + kBTile;
            const int ks = (c == s.nk - 1) ? s.ks_last : 2;
            for (int kk = 0; kk < ks; ++kk) {
              const uint32_t off = static_cast<uint32_t>(kk * 32);  // 16 fp16 / 8 tf32 along K
              mma3<kF16, kElect>(d, smem_desc_k_sw64(ah + off), smem_desc_k_sw64(al + off),
                                 smem_desc_k_sw64(bh + off), smem_desc_k_sw64(bl + off), (c | kk) != 0 ? 1u : 0u);
            }
            mcommit(&empty[stage]);
            if (++stage == kStages1) {
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
    const bool perrow = kF16 && prep_mode_perrow(sta, stb, s.D);
    int acc = 0;
    uint32_t aphase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int rb = u / s.nsplit, sp = u % s.nsplit;
      const int t0 = sp * s.tps;
      const int t1 = min(s.nt, t0 + s.tps);
      float rmin = __int_as_float(0x7f800000);
      const int64_t row = static_cast<int64_t>(rb) * kBM + row_local;
      const EpiScale es = epi_scale(kF16, sta, stb, sa, sb, row, s.nA, s.D);
      // kBidir: this row's ||a||^2, or +inf for rows past nA (excluded from column minima)
      const float narow = kBidir ? (row < s.nA ? __ldg(na + row) : __int_as_float(0x7f800000)) : 0.0f;
      for (int t = t0; t < t1; ++t) {
        // the tile's column norms (and per-row-mode column factors): loaded before the
        // accumulator wait, staged in shared memory, read back as broadcasts
        {
          const int64_t col = static_cast<int64_t>(t) * kBN + e;
          const float n1 = __ldg(nb + col);
          const float u1 = perrow ? 1.0f / __ldg(sb + col) : 1.0f;
          mbar_wait(&tfull[acc], aphase);
          nbuf[acc][e] = n1;
          ubuf[acc][e] = u1;
          asm volatile("bar.sync 1, 256;" ::: "memory");  // the 8 epilogue warps
        }
        tc_fence_after();
        const uint32_t taddr = tmem_base + lane_addr + static_cast<uint32_t>(acc * kBN);
        const float4* nbp = reinterpret_cast<const float4*>(nbuf[acc]);
        const float4* ubp = reinterpret_cast<const float4*>(ubuf[acc]);
        auto chunk = [&](float (&v)[32], int cc) {
          const float m = perrow ? epi_chunk<true>(v, es.k, nbp + cc * 8, ubp + cc * 8)
                                 : epi_chunk<false>(v, es.k, nbp + cc * 8, ubp + cc * 8);
          rmin = fminf(rmin, m);
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
// Two-A-block variant: one CTA computes TWO 128-row blocks of A against each 256-column tile
// of B, one fp32 accumulator each (all 512 TMEM columns, so the epilogue of a tile is not
// overlapped with the next tile's MMAs). Stages of 64-byte rows: A1 and A2 H/L 4 x 8 KB + B H/L
// 2 x 16 KB = 64 KB, three in flight: 2/3 of the single-block kernel's operand bytes per pair.
// ============================================================================
template <bool kBidir, bool kF16>
__global__ void __launch_bounds__(kThreadsA2, 1)
    dist_rowmin_2a_kernel(const __grid_constant__ CUtensorMap tAh, const __grid_constant__ CUtensorMap tAl,
                          const __grid_constant__ CUtensorMap tBh, const __grid_constant__ CUtensorMap tBl, Sched s,
                          const float* __restrict__ na, const float* __restrict__ nb, const float* __restrict__ sa,
                          const float* __restrict__ sb, const PrepStats* sta, const PrepStats* stb,
                          float* __restrict__ rowmin, float* __restrict__ colmin) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStagesA2 * kStageA2Bytes);
  uint64_t* empty = full + kStagesA2;
  uint64_t* tfull = empty + kStagesA2;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  __shared__ __align__(16) float nbuf[2][kBN];  // column norms, double-buffered by tile parity
  __shared__ __align__(16) float ubuf[2][kBN];  // per-row scale mode: 1 / s_j
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
          for (int c = 0; c < s.nk; ++c) {
            mbar_wait(&empty[stage], phase ^ 1u);
            uint8_t* st = smem + stage * kStageA2Bytes;
            mbar_arrive_expect_tx(&full[stage], kStageA2Bytes);
            tma_load_2d(st, &tAh, c * 16, pb * 256, &full[stage]);
            tma_load_2d(st + kATile, &tAl, c * 16, pb * 256, &full[stage]);
            tma_load_2d(st + 2 * kATile, &tAh, c * 16, pb * 256 + 128, &full[stage]);
            tma_load_2d(st + 3 * kATile, &tAl, c * 16, pb * 256 + 128, &full[stage]);
            tma_load_2d(st + 4 * kATile, &tBh, c * 16, t * kBN, &full[stage]);
            tma_load_2d(st + 4 * kATile + kBTile, &tBl, c * 16, t * kBN, &full[stage]);
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
          for (int c = 0; c < s.nk; ++c) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t a1h = smem_u32(smem + stage * kStageA2Bytes);
            const uint32_t a1l = a1h + kATile, a2h = a1h + 2 * kATile, a2l = a1h + 3 * kATile;
            const uint32_t bh = a1h + 4 * kATile, bl = bh + kBTile;
            const int ks = (c == s.nk - 1) ? s.ks_last : 2;
            for (int kk = 0; kk < ks; ++kk) {
              const uint32_t off = static_cast<uint32_t>(kk * 32);
              const uint64_t dbh = smem_desc_k_sw64(bh + off), dbl = smem_desc_k_sw64(bl + off);
              const uint32_t acc = (c | kk) != 0 ? 1u : 0u;
              mma3<kF16, true>(d0, smem_desc_k_sw64(a1h + off), smem_desc_k_sw64(a1l + off), dbh, dbl, acc);
              mma3<kF16, true>(d1, smem_desc_k_sw64(a2h + off), smem_desc_k_sw64(a2l + off), dbh, dbl, acc);
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
    const bool perrow = kF16 && prep_mode_perrow(sta, stb, s.D);
    uint32_t tph = 0;
    int tb = 0;  // nbuf parity
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int pb = u / s.nsplit, sp = u % s.nsplit;
      const int t0 = sp * s.tps;
      const int t1 = min(s.nt, t0 + s.tps);
      float rm = __int_as_float(0x7f800000);
      const int64_t myrow = static_cast<int64_t>(pb) * 256 + a2 * 128 + q * 32 + lane;
      const EpiScale es = epi_scale(kF16, sta, stb, sa, sb, myrow, s.nA, s.D);
      // kBidir: this row's ||a||^2, or +inf for rows past nA (excluded from column minima)
      const float narow = kBidir ? (myrow < s.nA ? __ldg(na + myrow) : __int_as_float(0x7f800000)) : 0.0f;
      for (int t = t0; t < t1; ++t) {
        {
          const int64_t col = static_cast<int64_t>(t) * kBN + e;
          const float n1 = __ldg(nb + col);
          const float u1 = perrow ? 1.0f / __ldg(sb + col) : 1.0f;
          mbar_wait(&tfull[0], tph);
          nbuf[tb][e] = n1;
          ubuf[tb][e] = u1;
          asm volatile("bar.sync 1, 256;" ::: "memory");
        }
        tc_fence_after();
        const float4* nbp = reinterpret_cast<const float4*>(nbuf[tb]);
        const float4* ubp = reinterpret_cast<const float4*>(ubuf[tb]);
        const uint32_t taddr = tmem_base + lane_addr + static_cast<uint32_t>(a2 * kBN);
        auto chunk = [&](float (&v)[32], int cc) {
          const float m = perrow ? epi_chunk<true>(v, es.k, nbp + cc * 8, ubp + cc * 8)
                                 : epi_chunk<false>(v, es.k, nbp + cc * 8, ubp + cc * 8);
          rm = fminf(rm, m);
          if (kBidir) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i] + narow, 0.0f);
            warp_colmin32(v, lane);
            atomicMin(&colbuf[tb][cc * 32 + lane], __float_as_uint(v[0]));
          }
        };
        if constexpr (!kBidir) {
          // software-pipelined drain: the next 64 columns load from TMEM while this 64 reduce
          // (two register sets; the accumulators go back to the issuer one load latency sooner)
          float v0[32], v1[32], w0[32], w1[32];
          tmem_ld32(taddr, v0);
          tmem_ld32(taddr + 32, v1);
          tmem_wait_ld();
#pragma unroll
          for (int cc = 0; cc < kBN / 32; cc += 4) {
            tmem_ld32(taddr + (cc + 2) * 32, w0);
            tmem_ld32(taddr + (cc + 3) * 32, w1);
            chunk(v0, cc);
            chunk(v1, cc + 1);
            tmem_wait_ld();
            if (cc + 4 < kBN / 32) {
              tmem_ld32(taddr + (cc + 4) * 32, v0);
              tmem_ld32(taddr + (cc + 5) * 32, v1);
            }
            chunk(w0, cc + 2);
            chunk(w1, cc + 3);
            if (cc + 4 < kBN / 32) tmem_wait_ld();
          }
        } else {
#pragma unroll 1
          for (int cc = 0; cc < kBN / 32; cc += 2) {
            float v0[32], v1[32];
            tmem_ld32(taddr + cc * 32, v0);
            tmem_ld32(taddr + (cc + 1) * 32, v1);
            tmem_wait_ld();
            chunk(v0, cc);
            chunk(v1, cc + 1);
          }
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
      if (myrow < s.nA) {
        const float d2 = fmaxf(rm + __ldg(na + myrow), 0.0f);
        if (s.atomic_out)
          atomicMin(reinterpret_cast<int*>(rowmin + myrow), __float_as_int(d2));
        else
          rowmin[myrow] = d2;
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
// CTA-pair kernel (fp16 split; directed, or with kBidir the fused bidirectional sweep whose
// epilogue also reduces this CTA's 128 rows to column minima): a 2-CTA cluster computes a 256-row block of A against
// 256-column tiles of B with M=256, N=256 `tcgen05.mma.cta_group::2` (three per 16 features).
// Each CTA stages its own 128 rows of A and its 128-row half of the B tile (32 KB per stage with
// hi + lo, 6 stages), so per SM the operand bytes per pair equal the two-A kernel's while each
// CTA's accumulator is only 256 TMEM columns: two of them, double-buffered, and the drain of tile
// t runs under the MMAs of tile t+1 (the two-A kernel's 512-column pair is drained with the
// tensor pipe idle). Per SM the tensor core reads 8 KB of shared memory per 128-clock MMA
// (A 4 KB + B half 4 KB; two-A: 12 KB).
// Barriers: full[] in the leader counts both CTAs' TMA bytes (2-SM TMA, one plain arrive from the
// peer); empty[] and tfull[] in both CTAs take the leader's multicast commit; tempty[] in the
// leader counts the 16 epilogue warps of the pair. Epilogue: 8 warps per CTA, warp w drains TMEM
// lane quarter w % 4 over column half (w - 2) / 4; the two halves of a row meet in shared memory.
// ============================================================================
constexpr int kStagesP = 6;
constexpr uint32_t kHalfP = 128 * kRowBytes;        // 8 KB: 128 rows x 64 B
constexpr uint32_t kStagePBytes = 4 * kHalfP;       // A_H, A_L, B_H half, B_L half
constexpr size_t kSmemP = static_cast<size_t>(kStagesP) * kStagePBytes + 1024 + 256;
constexpr int kThreadsP = 320;

template <bool kBidir>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsP, 1)
    dist_rowmin_pair_kernel(const __grid_constant__ CUtensorMap tAh, const __grid_constant__ CUtensorMap tAl,
                            const __grid_constant__ CUtensorMap tBh, const __grid_constant__ CUtensorMap tBl, Sched s,
                            const float* __restrict__ na, const float* __restrict__ nb, const float* __restrict__ sa,
                            const float* __restrict__ sb, const PrepStats* sta, const PrepStats* stb,
                            float* __restrict__ rowmin, float* __restrict__ colmin) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStagesP * kStagePBytes);
  uint64_t* empty = full + kStagesP;
  uint64_t* tfull = empty + kStagesP;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ __align__(16) float nbuf[2][kBN];  // column norms per accumulator buffer
  __shared__ __align__(16) float ubuf[2][kBN];  // per-row scale mode: 1 / s_j
  __shared__ float rhalf[128];                  // row minima of column half 1, merged by half 0
  __shared__ unsigned colbuf[2][kBN];           // kBidir: this CTA's column minima per accumulator (float bits)
  __shared__ unsigned tilecnt[2];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = static_cast<int>(cluster_id_x());
  const int ncl = static_cast<int>(nclusters_x());
  if (kBidir) {
    for (int i = threadIdx.x; i < 2 * kBN; i += blockDim.x) (&colbuf[0][0])[i] = 0x7F800000u;
    if (threadIdx.x < 2) tilecnt[threadIdx.x] = 0u;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStagesP; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 16);
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
      // ------------------------------------------------------------ TMA producer (both CTAs)
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
            // only the leader arrives (expecting both CTAs' bytes); the peer's TMA completes its
            // bytes on the leader's barrier without an arrive (the tx-count may go transiently
            // negative within the phase: the peer loads a slot only after the MMAs consumed the
            // previous phase of it, so its bytes always land in the phase they belong to)
            const uint32_t fl = mapa(smem_u32(&full[stage]), 0);
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * kStagePBytes);
            uint8_t* st = smem + stage * kStagePBytes;
            tma_load_2d_2sm(st, &tAh, c * 16, arow, fl);
            tma_load_2d_2sm(st + kHalfP, &tAl, c * 16, arow, fl);
            tma_load_2d_2sm(st + 2 * kHalfP, &tBh, c * 16, brow, fl);
            tma_load_2d_2sm(st + 3 * kHalfP, &tBl, c * 16, brow, fl);
            if (++stage == kStagesP) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------------------ MMA issuer (leader, warp-wide)
      constexpr uint32_t id = idesc_f16(256, kBN);
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
            const uint32_t ah = smem_u32(smem + stage * kStagePBytes);
            const uint32_t al = ah + kHalfP, bh = ah + 2 * kHalfP, bl = ah + 3 * kHalfP;
            const int ks = (c == s.nk - 1) ? s.ks_last : 2;
            for (int kk = 0; kk < ks; ++kk) {
              const uint32_t off = static_cast<uint32_t>(kk * 32);
              const uint64_t dah = smem_desc_k_sw64(ah + off), dbh = smem_desc_k_sw64(bh + off);
              mma_f16_2sm_w(d, dah, dbh, id, (c | kk) != 0 ? 1u : 0u);
              mma_f16_2sm_w(d, dah, smem_desc_k_sw64(bl + off), id, 1u);
              mma_f16_2sm_w(d, smem_desc_k_sw64(al + off), dbh, id, 1u);
            }
            mma_commit_2sm_mc_w(&empty[stage], 0x3);
            if (++stage == kStagesP) {
              stage = 0;
              phase ^= 1u;
            }
          }
          mma_commit_2sm_mc_w(&tfull[acc], 0x3);
          acc ^= 1;
          if (acc == 0) aphase ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- epilogue (both CTAs)
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;  // column half
    const int row_local = q * 32 + lane;
    const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
    const int e = (warp - 2) * 32 + lane;  // 0..255: one column norm each
    const bool perrow = prep_mode_perrow(sta, stb, s.D);
    const uint32_t te[2] = {mapa(smem_u32(&tempty[0]), 0), mapa(smem_u32(&tempty[1]), 0)};
    int acc = 0;
    uint32_t aphase = 0;
    for (int u = cid; u < units; u += ncl) {
      const int pb = u / s.nsplit, sp = u % s.nsplit;
      const int t0 = sp * s.tps;
      const int t1 = min(s.nt, t0 + s.tps);
      float rm = __int_as_float(0x7f800000);
      const int64_t myrow = static_cast<int64_t>(pb) * 256 + static_cast<int64_t>(rank) * 128 + row_local;
      const EpiScale es = epi_scale(true, sta, stb, sa, sb, myrow, s.nA, s.D);
      // kBidir: this row's ||a||^2, or +inf for rows past nA (excluded from column minima)
      const float narow = kBidir ? (myrow < s.nA ? __ldg(na + myrow) : __int_as_float(0x7f800000)) : 0.0f;
      for (int t = t0; t < t1; ++t) {
        {
          const int64_t col = static_cast<int64_t>(t) * kBN + e;
          const float n1 = __ldg(nb + col);
          const float u1 = perrow ? 1.0f / __ldg(sb + col) : 1.0f;
          mbar_wait(&tfull[acc], aphase);
          nbuf[acc][e] = n1;
          ubuf[acc][e] = u1;
          asm volatile("bar.sync 1, 256;" ::: "memory");
        }
        tc_fence_after();
        const float4* nbp = reinterpret_cast<const float4*>(nbuf[acc]) + h * 32;
        const float4* ubp = reinterpret_cast<const float4*>(ubuf[acc]) + h * 32;
        const uint32_t taddr = tmem_base + lane_addr + static_cast<uint32_t>(acc * kBN + h * 128);
        auto chunk = [&](float (&v)[32], int cc) {
          const float m = perrow ? epi_chunk<true>(v, es.k, nbp + cc * 8, ubp + cc * 8)
                                 : epi_chunk<false>(v, es.k, nbp + cc * 8, ubp + cc * 8);
          rm = fminf(rm, m);
          if (kBidir) {  // column minima over this warp's 32 rows, merged across the CTA's warps in shared memory
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i] + narow, 0.0f);
            warp_colmin32(v, lane);
            atomicMin(&colbuf[acc][h * 128 + cc * 32 + lane], __float_as_uint(v[0]));
          }
        };
        {
          float v0[32], v1[32], w0[32], w1[32];
          tmem_ld32(taddr, v0);
          tmem_ld32(taddr + 32, v1);
          tmem_wait_ld();
          tmem_ld32(taddr + 64, w0);
          tmem_ld32(taddr + 96, w1);
          chunk(v0, 0);
          chunk(v1, 1);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0)  // accumulator free: the rest is in registers (release.cta arrive on the leader's barrier)
            asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(te[acc]) : "memory");
          chunk(w0, 2);
          chunk(w1, 3);
        }
        if (kBidir) {
          // the last of this CTA's 8 epilogue warps flushes the tile's 256 column minima (the next
          // use of colbuf[acc] is two tiles on, behind two bar.sync of all 8 warps)
          __syncwarp();
          __threadfence_block();
          unsigned old = 0;
          if (lane == 0) old = atomicAdd(&tilecnt[acc], 1u);
          old = __shfl_sync(0xffffffffu, old, 0);
          if (old == 7u) {
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
        acc ^= 1;
        if (acc == 0) aphase ^= 1u;
      }
      // the two column halves of each row meet in shared memory (the per-tile bar.sync above
      // orders this unit's rhalf writes after the previous unit's reads)
      if (h == 1) rhalf[row_local] = rm;
      asm volatile("bar.sync 2, 256;" ::: "memory");
      if (h == 0 && myrow < s.nA) {
        const float d2 = fmaxf(fminf(rm, rhalf[row_local]) + __ldg(na + myrow), 0.0f);
        if (s.atomic_out)
          atomicMin(reinterpret_cast<int*>(rowmin + myrow), __float_as_int(d2));
        else
          rowmin[myrow] = d2;
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

template <typename K>
cudaError_t launch_k(K kern, int grid, int threads, size_t smem, cudaStream_t st, const DistArgs& a, const Sched& s) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  count_launch();
  kern<<<grid, threads, smem, st>>>(a.maps[0], a.maps[1], a.maps[2], a.maps[3], s, a.na, a.nb, a.sa, a.sb, a.sta,
                                    a.stb, a.rowmin, a.colmin);
  return cudaGetLastError();
}

}  // namespace

// Variants (one B200). fp16 sweeps at D >= 128, directed and fused bidirectional (the latter up
// to kBidirPairMaxWork, below), use the CTA-pair kernel (the literal 3xTF32 split at D >= 128:
// the two-A kernel directed, the single-block kernel bidirectional) and the single-block kernel below (faster at small D,
// where the epilogue is not hidden behind fewer MMAs). option k6_variant = 1 | 2 | 3 forces the
// single-block / pair / two-A kernel; k6_bidir_2a = 0 | 1 | 2 runs the bidirectional sweep on
// the single-block / two-A / pair kernel.
static int dist_variant(int D) {
  const long long v = opt(OPT_K6_VARIANT);
  if (v == 1 || v == 2 || v == 3) return static_cast<int>(v);
  return D >= 128 ? 2 : 1;  // 2: the CTA pair where it applies (fp16 directed), else the two-A kernel
}

// Fused bidirectional sweeps (option k6_bidir_2a unset): the pair kernel up to kBidirPairMaxWork
// = nA nB D, the single-block kernel above. Measured on a B200: short sweeps
// (subset HD, cfg3) run 4-17 % faster on the pair; a multi-second D = 256 sweep is power-capped
// and the pair kernel, tensor pipe and butterfly epilogue both busy, settles at a lower clock
// (cfg5 undirected 5.03 s single-block, 5.71 s pair).
constexpr double kBidirPairMaxWork = 1.0e14;
bool k6_uses_pair(int D, bool f16, bool bidir, int64_t nA, int64_t nB) {
  if (!f16 || dist_variant(D) != 2) return false;
  if (!bidir) return true;
  const long long b = opt(OPT_K6_BIDIR_2A);  // 0 single-block, 1 two-A, 2 pair
  if (b >= 0) return b == 2;
  return static_cast<double>(nA) * static_cast<double>(nB) * D <= kBidirPairMaxWork;
}

bool k6_split3() { return opt(OPT_K6_SPLIT3) == 1; }

cudaError_t launch_dist_rowmin(const DistArgs& a, cudaStream_t st) {
  const bool pair =
      k6_uses_pair(a.D, a.f16, a.colmin != nullptr, a.nA, a.nB) && a.maps_bhalf != nullptr && a.num_sms >= 2;
  const bool twoa = !pair && dist_variant(a.D) >= 2 && (a.colmin == nullptr || opt(OPT_K6_BIDIR_2A) == 1);
  const int rows_per_unit = (twoa || pair) ? 256 : kBM;
  Sched s{};
  s.nA = a.nA;
  s.nB = a.nB;
  s.D = a.D;
  s.nrb = static_cast<int>((a.nA + rows_per_unit - 1) / rows_per_unit);
  s.nt = static_cast<int>((a.nB + kBN - 1) / kBN);
  const int fps = a.f16 ? 32 : 16;  // features per 64-byte stage row
  const int fpk = fps / 2;          // features per 32-byte K-step
  s.nk = (a.D + fps - 1) / fps;
  s.ks_last = (a.D - (s.nk - 1) * fps + fpk - 1) / fpk;
  const int slots = pair ? a.num_sms / 2 : a.num_sms;  // concurrent units
  // Column splits: units (row block, column range) are dealt round-robin to the persistent
  // CTAs, so the sweep takes ceil(units / slots) rounds of (tps + ~0.5) tile times (the half
  // tile: a unit's pipeline fill / drain and row-minimum merge). Small A (subset HD: 100-250
  // row blocks) needs splits to fill 148 SMs, and the split count decides the last round's
  // occupancy: pick the cheapest of 1..64 splits (ties to fewer: fewer atomic merges).
  int nsplit = 1;
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
  if (nsplit < 1) nsplit = 1;
  if (nsplit > s.nt) nsplit = s.nt;
  s.tps = (s.nt + nsplit - 1) / nsplit;
  s.nsplit = (s.nt + s.tps - 1) / s.tps;
  s.atomic_out = s.nsplit > 1 ? 1 : 0;
  if (s.atomic_out) {
    cudaError_t e = cudaMemsetAsync(a.rowmin, 0x7F, sizeof(float) * a.nA, st);  // 3.39e38 (finite, > any d2)
    if (e != cudaSuccess) return e;
  }
  if (a.colmin != nullptr) {
    cudaError_t e = cudaMemsetAsync(a.colmin, 0x7F, sizeof(float) * a.nB, st);
    if (e != cudaSuccess) return e;
  }
  const int units = s.nrb * s.nsplit;
  const int grid = units < slots ? units : slots;
  const bool bidir = a.colmin != nullptr;
  if (pair) {
    auto kern = bidir ? dist_rowmin_pair_kernel<true> : dist_rowmin_pair_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemP));
    if (e != cudaSuccess) return e;
    count_launch();
    kern<<<2 * grid, kThreadsP, kSmemP, st>>>(a.maps[0], a.maps[1], a.maps_bhalf[0], a.maps_bhalf[1], s, a.na, a.nb,
                                              a.sa, a.sb, a.sta, a.stb, a.rowmin, a.colmin);
    return cudaGetLastError();
  }
  if (twoa) {
    if (bidir)
      return a.f16 ? launch_k(dist_rowmin_2a_kernel<true, true>, grid, kThreadsA2, kSmemA2, st, a, s)
                   : launch_k(dist_rowmin_2a_kernel<true, false>, grid, kThreadsA2, kSmemA2, st, a, s);
    return a.f16 ? launch_k(dist_rowmin_2a_kernel<false, true>, grid, kThreadsA2, kSmemA2, st, a, s)
                 : launch_k(dist_rowmin_2a_kernel<false, false>, grid, kThreadsA2, kSmemA2, st, a, s);
  }
  if (bidir) {
    // lane-0 MMA issue below D = 192 (D = 128 undirected cfg3: 255 -> 243 ms), elected above
    if (a.D < 192)
      return a.f16 ? launch_k(dist_rowmin_kernel<true, false, true>, grid, kThreads1, kSmem1, st, a, s)
                   : launch_k(dist_rowmin_kernel<true, false, false>, grid, kThreads1, kSmem1, st, a, s);
    return a.f16 ? launch_k(dist_rowmin_kernel<true, true, true>, grid, kThreads1, kSmem1, st, a, s)
                 : launch_k(dist_rowmin_kernel<true, true, false>, grid, kThreads1, kSmem1, st, a, s);
  }
  return a.f16 ? launch_k(dist_rowmin_kernel<false, true, true>, grid, kThreads1, kSmem1, st, a, s)
               : launch_k(dist_rowmin_kernel<false, true, false>, grid, kThreads1, kSmem1, st, a, s);
}

}  // namespace prohd
