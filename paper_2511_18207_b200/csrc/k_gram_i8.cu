// k_gram_i8.cu — K1 on the int8 tensor cores: the shifted Gram G = sum_p (p - s)(p - s)^T of
// A u B and the column sums S_X = sum_{x in X} (x - s), for D <= 256 (D % 4 == 0): gram_i8_kernel
// (CTA pairs) for 128 < D <= 256, gram_i8s_kernel (single CTAs, below) for D <= 128.
//
// PAPER.md Alg. 1 line 1 and Alg. 2 lines 1-2: the principal
// components are eigenvectors of C = G / N - (mu - s)(mu - s)^T (moments_finalize, k_moments.cu).
//
// Arithmetic (an exact-integer Ozaki scheme). Per feature j a power of two 2^k_j and an integer
// shift S_j (s_j = the shift kernel's sample mean, or 0 when the data sit near the origin;
// M_j = max over ALL rows of |x - s_j| from one HBM-bound pass, mapped to <= 2^30) turn every
// value into the 32-bit fixed-point integer F = rint(x 2^k_j - S_j) (exact when S_j = 0; with a
// shift the fused multiply-add rounds x 2^k - S to 24 bits first). F is written as four balanced 8-bit
// digits, F - c0 = sum_t d_t 2^(8 (3 - t)), t = 0 the most significant: the bytes of F with the
// three low bytes XOR 0x80 (c0 = 128 (2^16 + 2^8 + 1), a constant shift per column). Then
//     (F_i - c0)(F_j - c0) = sum_{t,u} d_t(i) d_u(j) 2^(8 (6 - t - u))
// and sum_p d_t(x_pi) d_u(x_pj) is an exact int8 x int8 -> int32 tensor-core product. Levels
// L = t + u <= 5 are kept: only d_3 d_3 (weight 1, |.| <= 2^14) is dropped, zero-mean, against
// products of |F| up to 2^30 (levels <= 3 alone would drop terms up to 2^32, too much for
// small values of heavy-tailed columns, whose leading digits are zero). The Gram is symmetric,
// so G_L = sum_{t+u=L} D_t^T D_u needs only the symmetric part of Z_L = 2 D_0^T D_L + sum_{t,u>0}
// D_t^T D_u (L > 0), Z_0 = 4 D_0^T D_0: M_j 2^k_j <= 2^30 - 256 keeps d_0 in [-64, 63], so the
// DOUBLED top digit 2 d_0 is an int8 plane and each pair (0, u), (u, 0) costs one product
// instead of two -- 12 products per point instead of 15; the reduce takes (Z + Z^T) / 2. The
// products of one level share an int32 TMEM accumulator, which grows by at most 3 * 128^2 per
// point, so it is drained to fp64 every <= 43648 points (exact).
// The result is the Gram about s'_j = (S_j + c0) 2^-k_j (exact fixed-point shift), written with
// s' into the moments buffers: G_ij = 2^(-k_i - k_j) sum_L 2^(8 (6 - L)) G_L, S_X = 2^-k sum F'.
// A non-finite value sets an overflow flag; the caller then reruns the moments on the fp64
// DMMA path (k_gram.cu), which reports PROHD_E_DATA.
//
// Kernel (cta_group::2, CTA pairs). One MMA M = 256 (all features, 128 per CTA) x N = 256 (all
// features, 128 per CTA) x K = 32 points covers the full Gram; each SM holds 128 rows x 256
// columns of int32 per level, so a pair holds two levels (all 512 TMEM columns): pair type 0
// accumulates levels {0, 3} (1 + 3 products), type 1 levels {1, 4} (1 + 3), type 2 levels {2, 5}
// (2 + 2). A group = one pair of each type over the same rows of A and of B (L2 serves the
// repeated reads); 24 groups = 144 SMs.
// Per CTA (320 threads):
//   warp 0     TMA: raw fp32 chunks [64 points x 128 features] (this CTA's feature half),
//              3 stages of 32 KB.
//   warp 1     (leader CTA) MMA issuer: per 64-point chunk 2 K-steps x 4 tcgen05.mma.cta_group::2
//              .kind::i8 over the two CTAs' digit planes; commit -> slice stage free (both CTAs).
//   warps 2-5  slicers: warp = every 4th point of the chunk, lane = 4 features: one 16-byte load,
//              F for the 4 values, a 4 x 4 byte transpose (PRMT) and one 32-bit store per digit
//              plane: 4 MN-major SWIZZLE_128B planes [64 points x 128 feature bytes] (2 stages of
//              32 KB; conflict-free: a warp writes one 128-byte row); type-0 pairs also add F' up per
//              set (int64 column sums). Arrive (cluster scope) on the leader's slices-full barrier.
//   warps 6-9  drain: TMEM lane quarter warp % 4 = feature rows; int32 -> fp64, both levels
//              weighted, added into this CTA's fp64 slab [128][256] in global memory.
// gram_i8_reduce_kernel sums the slabs in a fixed order (deterministic) and applies 2^(-k_i-k_j);
// gram_i8_sym_kernel takes the symmetric part.
#include "api_common.cuh"  // TMA descriptor encoder
#include "internal.cuh"
#include "prohd_kernels.cuh"
#include "sm100.cuh"

namespace prohd {
namespace {

constexpr int kPts = 64;          // points per chunk = bytes per digit-plane row (SWIZZLE_64B)
constexpr int kFeat = 128;        // features per CTA
constexpr int kRawStages = 3;
constexpr int kSlStages = 4;
constexpr uint32_t kRawBytes = kPts * kFeat * 4;   // 32 KB
constexpr uint32_t kPlane = kFeat * kPts;          // 8 KB
constexpr uint32_t kSlBytes = 4 * kPlane;          // 32 KB
constexpr int kSlicers = 8;      // slicer / drain warps (2-9), two per SM sub-partition
constexpr int kThreads = 64 + 32 * kSlicers;
constexpr int kDrainWarps = 8;   // slicer warps 0-7 also drain: 4 TMEM lane quarters x 2 column halves
constexpr int kDrainChunks = 682;  // 43648 points x 3 products x 2^14 < 2^31: int32 headroom
constexpr int kColmaxBlocks = 148 * 8;
constexpr size_t kSmem = static_cast<size_t>(kRawStages) * kRawBytes + kSlStages * kSlBytes + 1024 + 512;  // + barriers

struct I8Args {
  int64_t nA, nB;
  int D, ngroups;
  const float* scale;    // [256] 2^k_j
  const float* shiftf;   // [256] S_j (integer-valued float)
  double* slab;          // [ngroups * 6 CTAs][128][256]
  const double* cpart;   // [ncs blocks][2][D] fp64 column sums of A, B (i8_colmax_kernel)
  int ncs;
  unsigned* overflow;
  int ablate;            // dev timing only (option k1_ablate): 1 skip the slicing work, 2 skip the MMAs
  int small;             // D <= 128: gram_i8s_kernel (one CTA per level set), nt0 + nt1 CTAs;
                         // 2: D <= 64, gram_i8d_kernel (paired digit planes), nt0 CTAs
  int nt0, nt1;          //   CTAs of level set 0 ({0,1,2,3}) and of level set 1 ({4,5})
};

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  const long long t0 = clock64();
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(sm100::smem_u32(bar)), "r"(parity)
        : "memory");
    if (!ok && clock64() - t0 > 40000000000ll) __trap();
  } while (!ok);
}

// mbarrier wait with a suspend-time hint: a waiting thread sleeps in hardware instead of spinning
// on the issue slots its scheduler shares with the slicer warps
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  const long long t0 = clock64();
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 200000;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(sm100::smem_u32(bar)), "r"(parity)
        : "memory");
    if (!ok && clock64() - t0 > 40000000000ll) __trap();
  } while (!ok);
}
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ void mma_i8_2sm(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// kind::i8: D s32 (2), A and B s8 (1), both MN-major (bits 15, 16)
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t M, uint32_t N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
// MN-major operand with SWIZZLE_128B: one 128-byte row (the CTA's 128 features) per K index
// (point), 8-row (1 KB) swizzle atoms stacked along K (SBO = 1 KB); a single atom along MN, so
// LBO is unused. Canonical layout Sw<3,4,3> o ((T,8,m),(8,k)) : ((1,T,LBO),(8T,SBO)).
__device__ __forceinline__ uint64_t smem_desc_mn_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;            // LBO (unused: one MN atom)
  d |= static_cast<uint64_t>(1024u >> 4) << 32;    // SBO: next 8 K-rows
  d |= static_cast<uint64_t>(1u) << 46;            // version (sm_100)
  d |= static_cast<uint64_t>(2u) << 61;            // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void tmem_ld32i(uint32_t taddr, int (&v)[32]) {
  sm100::tmem_ld32(taddr, reinterpret_cast<float(&)[32]>(v));
}

// chunk schedule of one group: A rows [a0, a1) then B rows [b0, b1), 64 rows per chunk
struct Range {
  int64_t a0, a1, b0, b1;
  int na, nb;  // chunks
};
__device__ __forceinline__ Range group_range(const I8Args& a, int g, int ngroups) {
  Range r;
  r.a0 = a.nA * g / ngroups;
  r.a1 = a.nA * (g + 1) / ngroups;
  r.b0 = a.nB * g / ngroups;
  r.b1 = a.nB * (g + 1) / ngroups;
  r.na = static_cast<int>((r.a1 - r.a0 + kPts - 1) / kPts);
  r.nb = static_cast<int>((r.b1 - r.b0 + kPts - 1) / kPts);
  return r;
}

// Slice one raw chunk into the four digit planes (slicer warp ws, lane = features 4 lane .. +3 of the
// CTA's 128): xr = the raw stage (four SWIZZLE_128B boxes of 32 features x 64 points; box lane / 8
// holds features 32 (lane / 8) .., row p, 16-byte chunk (lane % 8) ^ (p % 8)), pl = the slice stage.
__device__ __forceinline__ void slice_chunk(uint32_t xr, uint32_t pl, int ws, int lane, int valid, const float (&sc)[4],
                                            const float (&sh)[4]) {
  // all of this warp's points of the chunk are loaded first (8 independent 16-byte loads in
  // flight), then converted: the shared-memory latency is not on each point's dependency chain
  constexpr int kPer = kPts / kSlicers;
  float4 xs[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int p = ws + kSlicers * u;
    xs[u] = lds128(xr + p * 128 + ((((lane & 7) ^ (p & 7)) & 7) << 4));
  }
  // one 4-point group: y = x 2^k - S (rows past the range: F = c0, i.e. F - c0 = 0), F, the four
  // digit bytes per feature, 4 x 4 byte transpose, one 32-bit store per digit plane
  auto slice_point = [&](int u, bool ok) {
    const int p = ws + kSlicers * u;
    const float4 x4 = xs[u];
    const float y0 = ok ? fmaf(x4.x, sc[0], -sh[0]) : 8421504.0f, y1 = ok ? fmaf(x4.y, sc[1], -sh[1]) : 8421504.0f;
    const float y2 = ok ? fmaf(x4.z, sc[2], -sh[2]) : 8421504.0f, y3 = ok ? fmaf(x4.w, sc[3], -sh[3]) : 8421504.0f;
    const uint32_t w0i = static_cast<uint32_t>(__float2int_rn(y0)), w1i = static_cast<uint32_t>(__float2int_rn(y1));
    const uint32_t w2i = static_cast<uint32_t>(__float2int_rn(y2)), w3i = static_cast<uint32_t>(__float2int_rn(y3));
    // plane t (t = 0 the top byte) gets byte 3 - t of the 4 features; the three low planes XOR
    // 0x80 per byte (balanced digits of F - c0)
    const uint32_t x01l = __byte_perm(w0i, w1i, 0x5140), x01h = __byte_perm(w0i, w1i, 0x7362);
    const uint32_t x23l = __byte_perm(w2i, w3i, 0x5140), x23h = __byte_perm(w2i, w3i, 0x7362);
    const uint32_t b0 = __byte_perm(x01l, x23l, 0x5410) ^ 0x80808080u;
    const uint32_t b1 = __byte_perm(x01l, x23l, 0x7632) ^ 0x80808080u;
    const uint32_t b2 = __byte_perm(x01h, x23h, 0x5410) ^ 0x80808080u;
    // plane 0 holds the DOUBLED top digit 2 d_0 (|d_0| <= 64, d_0 <= 63): per-byte shift
    const uint32_t b3 = (__byte_perm(x01h, x23h, 0x7632) << 1) & 0xFEFEFEFEu;
    // SWIZZLE_128B MN-major: row p (128 B), 16-byte chunk (lane / 4) XOR (p % 8)
    const uint32_t off = static_cast<uint32_t>((p >> 3) * 1024 + (p & 7) * 128 +
                                               ((((lane >> 2) ^ (p & 7)) & 7) << 4) + (lane & 3) * 4);
    sts32(pl + 0 * kPlane + off, b3);
    sts32(pl + 1 * kPlane + off, b2);
    sts32(pl + 2 * kPlane + off, b1);
    sts32(pl + 3 * kPlane + off, b0);
  };
  if (valid == kPts) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) slice_point(u, true);
  } else {  // the last, ragged chunk of a set
#pragma unroll
    for (int u = 0; u < kPer; ++u) slice_point(u, ws + kSlicers * u < valid);
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gram_i8_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, I8Args a) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* raw = smem;
  uint8_t* sl = smem + kRawStages * kRawBytes;
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(sl + kSlStages * kSlBytes);
  uint64_t* raw_empty = raw_full + kRawStages;
  uint64_t* sl_full = raw_empty + kRawStages;  // leader: 8 slicer warps of the pair
  uint64_t* sl_empty = sl_full + kSlStages;    // both: MMA commit (multicast)
  uint64_t* tfull = sl_empty + kSlStages;      // both: MMA commit (multicast)
  uint64_t* tempty = tfull + 1;                // leader: 8 drain warps of the pair
  uint64_t* sl_fwd = tempty + 1;               // peer: its slicer warps, forwarded by one thread
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sl_fwd + kSlStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int type = pair % 3, g = pair / 3;
  const Range R = group_range(a, g, a.ngroups);
  const int nchunks = R.na + R.nb;
  const int cta = blockIdx.x;  // slab index

  if (threadIdx.x == 0) {
    for (int i = 0; i < kRawStages; ++i) {
      mbar_init(&raw_full[i], 1);
      mbar_init(&raw_empty[i], kSlicers);
    }
    for (int i = 0; i < kSlStages; ++i) {
      mbar_init(&sl_full[i], kSlicers + 1);  // the leader's slicer warps + one forwarded arrival
      mbar_init(&sl_empty[i], 1);
      mbar_init(&sl_fwd[i], kSlicers);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tempty[0], 2 * kDrainWarps);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tA);
    tma_prefetch(&tB);
  }
  if (warp == 1) tmem_alloc_2sm<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int c = 0; c < nchunks; ++c) {
        mbar_wait(&raw_empty[st], ph ^ 1u);
        mbar_arrive_expect_tx(&raw_full[st], kRawBytes);
        const bool inA = c < R.na;
        const int64_t row = inA ? R.a0 + static_cast<int64_t>(c) * kPts : R.b0 + static_cast<int64_t>(c - R.na) * kPts;
        // four [32 features x 64 rows] SWIZZLE_128B boxes (128-byte rows): the whole 128-feature half
        for (int bx = 0; bx < 4; ++bx)
          tma_load_2d(raw + st * kRawBytes + bx * (kRawBytes / 4), inA ? &tA : &tB,
                      static_cast<int>(rank) * kFeat + bx * 32, static_cast<int>(row), &raw_full[st]);
        if (++st == kRawStages) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (leader CTA)
    if (rank == 0 && lane == 0 && a.ablate < 4) {
      constexpr uint32_t idesc = idesc_i8(256, 256);
      // (t, u, accumulator slot), plane 0 = 2 d_0: type 0 = levels {0 -> slot 0, 3 -> slot 1},
      // type 1 = {1, 4}, type 2 = {2, 5}; the pairs (0, u) and (u, 0) are one product 2 d_0 d_u
      // (the reduce symmetrises), (0, 0) is 4 d_0 d_0 (drain weight / 4)
      int tt[4], uu[4], ss[4];
      if (type == 0) {
        const int t0[4] = {0, 0, 1, 2}, u0[4] = {0, 3, 2, 1}, s0[4] = {0, 1, 1, 1};
        for (int i = 0; i < 4; ++i) tt[i] = t0[i], uu[i] = u0[i], ss[i] = s0[i];
      } else if (type == 1) {
        const int t1[4] = {0, 1, 3, 2}, u1[4] = {1, 3, 1, 2}, s1[4] = {0, 1, 1, 1};
        for (int i = 0; i < 4; ++i) tt[i] = t1[i], uu[i] = u1[i], ss[i] = s1[i];
      } else {
        const int t2[4] = {0, 1, 2, 3}, u2[4] = {2, 1, 3, 2}, s2[4] = {0, 0, 1, 1};
        for (int i = 0; i < 4; ++i) tt[i] = t2[i], uu[i] = u2[i], ss[i] = s2[i];
      }
      int st = 0;
      uint32_t ph = 0, tph = 0;
      int since = 0;  // chunks accumulated since the last drain
      for (int c = 0; c < nchunks; ++c) {
        if (since == 0 && c > 0) {
          mbar_wait_cluster(&tempty[0], tph ^ 1u);  // the drain warps of both CTAs have read TMEM
          tc_fence_after();
        }
        mbar_wait_cluster(&sl_full[st], ph);
        tc_fence_after();
        const uint32_t base = smem_u32(sl + st * kSlBytes);
        for (int kk = 0; kk < (a.ablate >= 2 ? 0 : 2); ++kk) {
          for (int i = 0; i < 4; ++i) {  // K = 32 points = 4 swizzle atoms of 8 rows: +4 KB per K-step
            const uint64_t da = smem_desc_mn_sw128(base + tt[i] * kPlane + kk * 4096);
            const uint64_t db = smem_desc_mn_sw128(base + uu[i] * kPlane + kk * 4096);
            const bool first = since == 0 && kk == 0 && (i == 0 || ss[i] != ss[i - 1]);
            mma_i8_2sm(tmem_base + static_cast<uint32_t>(ss[i] * 256), da, db, idesc, first ? 0u : 1u);
          }
        }
        mma_commit_2sm_mc(&sl_empty[st], 0x3);
        if (++st == kSlStages) {
          st = 0;
          ph ^= 1u;
        }
        if (++since == kDrainChunks || c == nchunks - 1) {
          mma_commit_2sm_mc(&tfull[0], 0x3);
          since = 0;
          tph ^= 1u;
        }
      }
    }
    if (rank == 1 && lane == 0 && a.ablate < 4) {
      // forwarder: the peer's slicer warps arrive on a local barrier; one cluster-scope release
      // arrival per chunk on the leader's slices-full barrier (instead of one per warp)
      const uint32_t leader_full = mapa(smem_u32(&sl_full[0]), 0);
      int st = 0;
      uint32_t ph = 0;
      for (int c = 0; c < nchunks; ++c) {
        mbar_wait(&sl_fwd[st], ph);
        mbar_arrive_cluster(leader_full + static_cast<uint32_t>(st * 8));
        if (++st == kSlStages) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ slicers (+ drains)
    // warp ws = warp - 2 takes points ws, ws + 8, ... of each 64-point chunk; lane l takes features
    // 4l..4l+3 of the CTA's 128: one 16-byte shared load per point, F for the four values, a 4 x 4
    // byte transpose and one 32-bit store per digit plane (MN-major: row = point, 128 feature
    // bytes; a warp writes one 128-byte row, conflict-free under the XOR swizzle)
    const int ws = warp - 2;
    const int fg0 = static_cast<int>(rank) * kFeat + 4 * lane;
    float sc[4], sh[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool live = fg0 + i < a.D;
      sc[i] = live ? __ldg(a.scale + fg0 + i) : 0.0f;  // features >= D: y = -(-c0) = c0, F - c0 = 0
      sh[i] = live ? __ldg(a.shiftf + fg0 + i) : -8421504.0f;
    }
    const uint32_t leader_te = mapa(smem_u32(&tempty[0]), 0);
    const uint32_t raw_u32 = smem_u32(raw), sl_u32 = smem_u32(sl);
    // drain role: TMEM lane quarter ws % 4, column half ws / 4 of both level slots
    const int q = warp & 3, half = ws >> 2;
    const int rowl = q * 32 + lane;
    const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
    // level weights 2^(8 (6 - L)) / 2^48 = 2^(-8 L): slots of type 0 = levels {0, 3} (level 0
    // holds 4 d_0 d_0: weight / 4), type 1 = {1, 4}, type 2 = {2, 5}
    const double w0 = type == 0 ? 0.25 : (type == 1 ? 0x1p-8 : 0x1p-16);
    const double w1 = type == 0 ? 0x1p-24 : (type == 1 ? 0x1p-32 : 0x1p-40);
    // slab layout [column 256][row 128]: a warp's 32 lanes (rows) store 256 contiguous bytes
    double* out = a.slab + static_cast<int64_t>(cta) * kFeat * 256 + half * 128 * kFeat + rowl;
    int rst = 0, sst = 0, since = 0, ndr = 0;
    uint32_t rph = 0, sph = 0, tph = 0;
    for (int c = 0; c < nchunks; ++c) {
      const bool inA = c < R.na;
      const int64_t row0 = inA ? R.a0 + static_cast<int64_t>(c) * kPts : R.b0 + static_cast<int64_t>(c - R.na) * kPts;
      const int64_t rend = inA ? R.a1 : R.b1;
      const int valid = static_cast<int>(min(static_cast<int64_t>(kPts), rend - row0));
      mbar_wait(&raw_full[rst], rph);
      if (a.ablate < 4) mbar_wait(&sl_empty[sst], sph ^ 1u);
      // raw box (lane / 8) holds features 32 (lane / 8) ..; row p, 16-byte chunk (lane % 8) ^ (p % 8)
      const uint32_t xr = raw_u32 + rst * kRawBytes + (lane >> 3) * (kRawBytes / 4);
      const uint32_t pl = sl_u32 + sst * kSlBytes;
      if (!(a.ablate & 1)) slice_chunk(xr, pl, ws, lane, valid, sc, sh);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&raw_empty[rst]);
        if (a.ablate < 4) mbar_arrive(rank == 0 ? &sl_full[sst] : &sl_fwd[sst]);  // CTA scope; the peer's are forwarded
      }
      if (++rst == kRawStages) {
        rst = 0;
        rph ^= 1u;
      }
      if (++sst == kSlStages) {
        sst = 0;
        sph ^= 1u;
      }
      if (a.ablate >= 4) continue;
      if ((++since == kDrainChunks || c == nchunks - 1) && ws >= kDrainWarps) {
        since = 0;
      } else if (since == kDrainChunks || c == nchunks - 1) {
        // drain window ends with this chunk: TMEM -> fp64 slab (this warp: its lane quarter, its
        // 128-column half of both level slots), then release the accumulators to the MMA issuer
        since = 0;
        mbar_wait_sleep(&tfull[0], tph);
        tph ^= 1u;
        tc_fence_after();
#pragma unroll 1
        for (int cc = 0; cc < 128; cc += 32) {
          int v0[32], v1[32];
          tmem_ld32i(tmem_base + lane_addr + static_cast<uint32_t>(half * 128 + cc), v0);
          tmem_ld32i(tmem_base + lane_addr + static_cast<uint32_t>(256 + half * 128 + cc), v1);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const double v = static_cast<double>(v0[i]) * w0 + static_cast<double>(v1[i]) * w1;
            out[(cc + i) * kFeat] = ndr == 0 ? v : out[(cc + i) * kFeat] + v;
          }
        }
        ++ndr;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_te);
      }
    }
    if (nchunks == 0 && ws < kDrainWarps)
      for (int j2 = 0; j2 < 128; ++j2) out[j2 * kFeat] = 0.0;  // an empty group contributes zeros
    // |y| <= 2^30 by the exact column max; non-finite input is flagged by the pre-pass
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm<512>(tmem_base);
  }
}

__device__ __forceinline__ void mma_i8_1sm(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// D <= 128 (gram_i8s_kernel): the whole Gram is one M = 128 x N = 128 block (features past D have
// zero digits), so one CTA (cta_group::1) holds four 128-column int32 level accumulators in its
// 512 TMEM columns. Level set 0 = levels {0, 1, 2, 3}: 1 + 1 + 2 + 3 = 7 products per K-step;
// level set 1 = levels {4, 5}: 3 + 2 = 5 products. The CTAs of a set split the rows of A u B
// (the two sets read every row once each), and the sets get CTAs in the ratio 7 : 5.
// Same roles and stages as gram_i8_kernel: warp 0 TMA (raw chunks, 64 points x 128 features),
// warp 1 TMEM allocation and the MMA issuer, warps 2-9 slicers and, at the end of a drain window,
// drains (lane quarter warp % 4, column half (warp - 2) / 4 of every slot) into the CTA's fp64
// slab [128 columns][128 rows].
constexpr int kSmallSlab = 128 * 128;  // doubles per CTA slab
constexpr int kSet0Share = 7, kSetShares = 12;

__global__ void __launch_bounds__(kThreads, 1)
    gram_i8s_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, I8Args a) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* raw = smem;
  uint8_t* sl = smem + kRawStages * kRawBytes;
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(sl + kSlStages * kSlBytes);
  uint64_t* raw_empty = raw_full + kRawStages;
  uint64_t* sl_full = raw_empty + kRawStages;  // the 8 slicer warps
  uint64_t* sl_empty = sl_full + kSlStages;    // MMA commit
  uint64_t* tfull = sl_empty + kSlStages;      // MMA commit at the end of a drain window
  uint64_t* tempty = tfull + 1;                // the 8 drain warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int set = static_cast<int>(blockIdx.x) < a.nt0 ? 0 : 1;
  const int g = set == 0 ? static_cast<int>(blockIdx.x) : static_cast<int>(blockIdx.x) - a.nt0;
  const Range R = group_range(a, g, set == 0 ? a.nt0 : a.nt1);
  const int nchunks = R.na + R.nb;
  const int nslot = set == 0 ? 4 : 2;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kRawStages; ++i) {
      mbar_init(&raw_full[i], 1);
      mbar_init(&raw_empty[i], kSlicers);
    }
    for (int i = 0; i < kSlStages; ++i) {
      mbar_init(&sl_full[i], kSlicers);
      mbar_init(&sl_empty[i], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tempty[0], kDrainWarps);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tA);
    tma_prefetch(&tB);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int c = 0; c < nchunks; ++c) {
        mbar_wait(&raw_empty[st], ph ^ 1u);
        mbar_arrive_expect_tx(&raw_full[st], kRawBytes);
        const bool inA = c < R.na;
        const int64_t row = inA ? R.a0 + static_cast<int64_t>(c) * kPts : R.b0 + static_cast<int64_t>(c - R.na) * kPts;
        for (int bx = 0; bx < 4; ++bx)  // boxes past D are zero-filled by the TMA unit
          tma_load_2d(raw + st * kRawBytes + bx * (kRawBytes / 4), inA ? &tA : &tB, bx * 32, static_cast<int>(row),
                      &raw_full[st]);
        if (++st == kRawStages) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_i8(128, 128);
      // (t, u, slot); plane 0 = 2 d_0, so (0, u) stands for (0, u) + (u, 0) after the final
      // symmetrisation and (0, 0) is 4 d_0 d_0
      int tt[7], uu[7], ss[7];
      int np;
      if (set == 0) {
        const int t0[7] = {0, 0, 0, 1, 0, 1, 2}, u0[7] = {0, 1, 2, 1, 3, 2, 1}, s0[7] = {0, 1, 2, 2, 3, 3, 3};
        for (int i = 0; i < 7; ++i) tt[i] = t0[i], uu[i] = u0[i], ss[i] = s0[i];
        np = 7;
      } else {
        const int t1[5] = {1, 2, 3, 2, 3}, u1[5] = {3, 2, 1, 3, 2}, s1[5] = {0, 0, 0, 1, 1};
        for (int i = 0; i < 5; ++i) tt[i] = t1[i], uu[i] = u1[i], ss[i] = s1[i];
        for (int i = 5; i < 7; ++i) tt[i] = uu[i] = ss[i] = 0;
        np = 5;
      }
      int st = 0;
      uint32_t ph = 0, tph = 0;
      int since = 0;
      for (int c = 0; c < nchunks; ++c) {
        if (since == 0 && c > 0) {
          mbar_wait(&tempty[0], tph ^ 1u);  // the drain warps have read TMEM
          tc_fence_after();
        }
        mbar_wait(&sl_full[st], ph);
        tc_fence_after();
        const uint32_t base = smem_u32(sl + st * kSlBytes);
        for (int kk = 0; kk < (a.ablate >= 2 ? 0 : 2); ++kk) {
          for (int i = 0; i < np; ++i) {
            const uint64_t da = smem_desc_mn_sw128(base + tt[i] * kPlane + kk * 4096);
            const uint64_t db = smem_desc_mn_sw128(base + uu[i] * kPlane + kk * 4096);
            const bool first = since == 0 && kk == 0 && (i == 0 || ss[i] != ss[i - 1]);
            mma_i8_1sm(tmem_base + static_cast<uint32_t>(ss[i] * 128), da, db, idesc, first ? 0u : 1u);
          }
        }
        mma_commit(&sl_empty[st]);
        if (++st == kSlStages) {
          st = 0;
          ph ^= 1u;
        }
        if (++since == kDrainChunks || c == nchunks - 1) {
          mma_commit(&tfull[0]);
          since = 0;
          tph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ slicers (+ drains)
    const int ws = warp - 2;
    const int fg0 = 4 * lane;
    float sc[4], sh[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool live = fg0 + i < a.D;
      sc[i] = live ? __ldg(a.scale + fg0 + i) : 0.0f;  // features >= D: F - c0 = 0
      sh[i] = live ? __ldg(a.shiftf + fg0 + i) : -8421504.0f;
    }
    const uint32_t raw_u32 = smem_u32(raw), sl_u32 = smem_u32(sl);
    const int q = warp & 3, half = ws >> 2;
    const int rowl = q * 32 + lane;
    const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
    // level weights 2^(-8 L) (level 0 holds 4 d_0 d_0: weight / 4)
    double wt[4];
    if (set == 0) {
      wt[0] = 0.25;
      wt[1] = 0x1p-8;
      wt[2] = 0x1p-16;
      wt[3] = 0x1p-24;
    } else {
      wt[0] = 0x1p-32;
      wt[1] = 0x1p-40;
      wt[2] = wt[3] = 0.0;
    }
    double* out = a.slab + static_cast<int64_t>(blockIdx.x) * kSmallSlab + half * 64 * 128 + rowl;
    int rst = 0, sst = 0, since = 0, ndr = 0;
    uint32_t rph = 0, sph = 0, tph = 0;
    for (int c = 0; c < nchunks; ++c) {
      const bool inA = c < R.na;
      const int64_t row0 = inA ? R.a0 + static_cast<int64_t>(c) * kPts : R.b0 + static_cast<int64_t>(c - R.na) * kPts;
      const int64_t rend = inA ? R.a1 : R.b1;
      const int valid = static_cast<int>(min(static_cast<int64_t>(kPts), rend - row0));
      mbar_wait(&raw_full[rst], rph);
      mbar_wait(&sl_empty[sst], sph ^ 1u);
      const uint32_t xr = raw_u32 + rst * kRawBytes + (lane >> 3) * (kRawBytes / 4);
      const uint32_t pl = sl_u32 + sst * kSlBytes;
      if (!(a.ablate & 1)) slice_chunk(xr, pl, ws, lane, valid, sc, sh);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&raw_empty[rst]);
        mbar_arrive(&sl_full[sst]);
      }
      if (++rst == kRawStages) {
        rst = 0;
        rph ^= 1u;
      }
      if (++sst == kSlStages) {
        sst = 0;
        sph ^= 1u;
      }
      if (++since == kDrainChunks || c == nchunks - 1) {
        // drain window ends: TMEM -> fp64 slab (this warp: its lane quarter, its 64-column half of
        // every slot, the slots weighted and added in a fixed order), then release the accumulators
        since = 0;
        mbar_wait_sleep(&tfull[0], tph);
        tph ^= 1u;
        tc_fence_after();
#pragma unroll 1
        for (int cc = 0; cc < 64; cc += 32) {
          double acc[32];
#pragma unroll 1
          for (int sl2 = 0; sl2 < nslot; ++sl2) {
            int v[32];
            tmem_ld32i(tmem_base + lane_addr + static_cast<uint32_t>(sl2 * 128 + half * 64 + cc), v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[i] = sl2 == 0 ? static_cast<double>(v[i]) * wt[0]
                                                           : fma(static_cast<double>(v[i]), wt[sl2], acc[i]);
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) out[(cc + i) * 128] = ndr == 0 ? acc[i] : out[(cc + i) * 128] + acc[i];
        }
        ++ndr;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[0]);
      }
    }
    if (nchunks == 0)
      for (int j2 = 0; j2 < 64; ++j2) out[j2 * 128] = 0.0;  // an empty range contributes zeros
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

// D <= 64 (gram_i8d_kernel): two digit planes share one 128-byte row (features 0-63 of plane t in
// bytes 0-63, of plane t' in bytes 64-127): P0 = [2 d_0 | d_1], P1 = [d_2 | d_3]. One M = N = 128
// MMA of two paired planes computes four useful 64 x 64 products (its quadrants), so three MMAs
// per K-step cover every ordered digit pair: R0 = P0 x P0, R1 = P0 x P1 (standing for P1 x P0 too:
// the final symmetrisation makes D_u^T D_t count as D_t^T D_u, so R1 is weighted x 2), R2 = P1 x P1
// (including d_3 d_3: exact). Three 128-column regions of TMEM, ONE CTA type: every row is read and
// sliced once. Each quadrant of a region gains one product (|.| <= 2^14) per point: drained every
// kDrainChunksD chunks. The drain weights each (region, quadrant) by its level 2^(-8 L), the digit
// doubling and the x2 of R1, into a per-CTA slab [quadrant][64 j][64 i] of fp64.
constexpr int kDrainChunksD = 256;
__device__ __forceinline__ void slice_chunk_pair(uint32_t xr, uint32_t pl, int ws, int lane, int valid,
                                                 const float (&sc)[4], const float (&sh)[4]) {
  if (lane >= 16) return;  // features 64-127 do not exist for D <= 64
  constexpr int kPer = kPts / kSlicers;
  float4 xs[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int p = ws + kSlicers * u;
    xs[u] = lds128(xr + p * 128 + ((((lane & 7) ^ (p & 7)) & 7) << 4));
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int p = ws + kSlicers * u;
    const bool ok = p < valid;
    const float4 x4 = xs[u];
    const float y0 = ok ? fmaf(x4.x, sc[0], -sh[0]) : 8421504.0f, y1 = ok ? fmaf(x4.y, sc[1], -sh[1]) : 8421504.0f;
    const float y2 = ok ? fmaf(x4.z, sc[2], -sh[2]) : 8421504.0f, y3 = ok ? fmaf(x4.w, sc[3], -sh[3]) : 8421504.0f;
    const uint32_t w0i = static_cast<uint32_t>(__float2int_rn(y0)), w1i = static_cast<uint32_t>(__float2int_rn(y1));
    const uint32_t w2i = static_cast<uint32_t>(__float2int_rn(y2)), w3i = static_cast<uint32_t>(__float2int_rn(y3));
    const uint32_t x01l = __byte_perm(w0i, w1i, 0x5140), x01h = __byte_perm(w0i, w1i, 0x7362);
    const uint32_t x23l = __byte_perm(w2i, w3i, 0x5140), x23h = __byte_perm(w2i, w3i, 0x7362);
    const uint32_t b0 = __byte_perm(x01l, x23l, 0x5410) ^ 0x80808080u;             // d_3
    const uint32_t b1 = __byte_perm(x01l, x23l, 0x7632) ^ 0x80808080u;             // d_2
    const uint32_t b2 = __byte_perm(x01h, x23h, 0x5410) ^ 0x80808080u;             // d_1
    const uint32_t b3 = (__byte_perm(x01h, x23h, 0x7632) << 1) & 0xFEFEFEFEu;      // 2 d_0
    // SWIZZLE_128B MN-major rows of 128 bytes: bytes 4 lane .. (chunk lane / 4) and 64 + 4 lane ..
    // (chunk 4 + lane / 4), each XOR (p % 8)
    const uint32_t rowb = static_cast<uint32_t>((p >> 3) * 1024 + (p & 7) * 128 + (lane & 3) * 4);
    const uint32_t lo = rowb + ((((lane >> 2) ^ (p & 7)) & 7) << 4);
    const uint32_t hi = rowb + ((((4 + (lane >> 2)) ^ (p & 7)) & 7) << 4);
    sts32(pl + lo, b3);
    sts32(pl + hi, b2);
    sts32(pl + kPlane + lo, b1);
    sts32(pl + kPlane + hi, b0);
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    gram_i8d_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, I8Args a) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* raw = smem;
  uint8_t* sl = smem + kRawStages * kRawBytes;
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(sl + kSlStages * kSlBytes);
  uint64_t* raw_empty = raw_full + kRawStages;
  uint64_t* sl_full = raw_empty + kRawStages;
  uint64_t* sl_empty = sl_full + kSlStages;
  uint64_t* tfull = sl_empty + kSlStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  constexpr uint32_t kRawD = kRawBytes / 2;  // two [32 features x 64 points] boxes

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Range R = group_range(a, static_cast<int>(blockIdx.x), a.nt0);
  const int nchunks = R.na + R.nb;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kRawStages; ++i) {
      mbar_init(&raw_full[i], 1);
      mbar_init(&raw_empty[i], kSlicers);
    }
    for (int i = 0; i < kSlStages; ++i) {
      mbar_init(&sl_full[i], kSlicers);
      mbar_init(&sl_empty[i], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tempty[0], kDrainWarps);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tA);
    tma_prefetch(&tB);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int c = 0; c < nchunks; ++c) {
        mbar_wait(&raw_empty[st], ph ^ 1u);
        mbar_arrive_expect_tx(&raw_full[st], kRawD);
        const bool inA = c < R.na;
        const int64_t row = inA ? R.a0 + static_cast<int64_t>(c) * kPts : R.b0 + static_cast<int64_t>(c - R.na) * kPts;
        for (int bx = 0; bx < 2; ++bx)
          tma_load_2d(raw + st * kRawBytes + bx * (kRawBytes / 4), inA ? &tA : &tB, bx * 32, static_cast<int>(row),
                      &raw_full[st]);
        if (++st == kRawStages) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_i8(128, 128);
      int st = 0;
      uint32_t ph = 0, tph = 0;
      int since = 0;
      for (int c = 0; c < nchunks; ++c) {
        if (since == 0 && c > 0) {
          mbar_wait(&tempty[0], tph ^ 1u);
          tc_fence_after();
        }
        mbar_wait(&sl_full[st], ph);
        tc_fence_after();
        const uint32_t base = smem_u32(sl + st * kSlBytes);
        for (int kk = 0; kk < (a.ablate >= 2 ? 0 : 2); ++kk) {
          const uint32_t acc = (since == 0 && kk == 0) ? 0u : 1u;
          const uint64_t p0 = smem_desc_mn_sw128(base + kk * 4096), p1 = smem_desc_mn_sw128(base + kPlane + kk * 4096);
          mma_i8_1sm(tmem_base + 0, p0, p0, idesc, acc);
          mma_i8_1sm(tmem_base + 128, p0, p1, idesc, acc);
          mma_i8_1sm(tmem_base + 256, p1, p1, idesc, acc);
        }
        mma_commit(&sl_empty[st]);
        if (++st == kSlStages) {
          st = 0;
          ph ^= 1u;
        }
        if (++since == kDrainChunksD || c == nchunks - 1) {
          mma_commit(&tfull[0]);
          since = 0;
          tph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    const int ws = warp - 2;
    const int fg0 = 4 * lane;
    float sc[4], sh[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool live = fg0 + i < a.D;
      sc[i] = live ? __ldg(a.scale + fg0 + i) : 0.0f;
      sh[i] = live ? __ldg(a.shiftf + fg0 + i) : -8421504.0f;
    }
    const uint32_t raw_u32 = smem_u32(raw), sl_u32 = smem_u32(sl);
    const int q = warp & 3, half = ws >> 2;
    const int row = q * 32 + lane;            // TMEM lane: A-operand byte row = (row / 64 plane, feature row % 64)
    const int ar = row >> 6, fi = row & 63;
    const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
    const int quad = 2 * ar + half;
    // weights of region R at this quadrant (see the kernel comment): level 2^(-8 L), / 2 per doubled
    // d_0 factor, x 2 for R1
    const double w00[3] = {0.25, 0x1p-16, 0x1p-32}, w01[3] = {0x1p-9, 0x1p-24, 0x1p-40};
    const double w10[3] = {0x1p-9, 0x1p-23, 0x1p-40}, w11[3] = {0x1p-16, 0x1p-31, 0x1p-48};
    double wt[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) wt[r] = quad == 0 ? w00[r] : (quad == 1 ? w01[r] : (quad == 2 ? w10[r] : w11[r]));
    double* out = a.slab + static_cast<int64_t>(blockIdx.x) * kSmallSlab + quad * 4096 + fi;
    int rst = 0, sst = 0, since = 0, ndr = 0;
    uint32_t rph = 0, sph = 0, tph = 0;
    for (int c = 0; c < nchunks; ++c) {
      const bool inA = c < R.na;
      const int64_t row0 = inA ? R.a0 + static_cast<int64_t>(c) * kPts : R.b0 + static_cast<int64_t>(c - R.na) * kPts;
      const int64_t rend = inA ? R.a1 : R.b1;
      const int valid = static_cast<int>(min(static_cast<int64_t>(kPts), rend - row0));
      mbar_wait(&raw_full[rst], rph);
      mbar_wait(&sl_empty[sst], sph ^ 1u);
      const uint32_t xr = raw_u32 + rst * kRawBytes + (lane >> 3) * (kRawBytes / 4);
      const uint32_t pl = sl_u32 + sst * kSlBytes;
      if (!(a.ablate & 1)) slice_chunk_pair(xr, pl, ws, lane, valid, sc, sh);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&raw_empty[rst]);
        mbar_arrive(&sl_full[sst]);
      }
      if (++rst == kRawStages) {
        rst = 0;
        rph ^= 1u;
      }
      if (++sst == kSlStages) {
        sst = 0;
        sph ^= 1u;
      }
      if (++since == kDrainChunksD || c == nchunks - 1) {
        since = 0;
        mbar_wait_sleep(&tfull[0], tph);
        tph ^= 1u;
        tc_fence_after();
#pragma unroll 1
        for (int cc = 0; cc < 64; cc += 32) {
          double acc[32];
#pragma unroll 1
          for (int r = 0; r < 3; ++r) {
            int v[32];
            tmem_ld32i(tmem_base + lane_addr + static_cast<uint32_t>(r * 128 + half * 64 + cc), v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i)
              acc[i] = r == 0 ? static_cast<double>(v[i]) * wt[0] : fma(static_cast<double>(v[i]), wt[r], acc[i]);
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) out[(cc + i) * 64] = ndr == 0 ? acc[i] : out[(cc + i) * 64] + acc[i];
        }
        ++ndr;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[0]);
      }
    }
    if (nchunks == 0)
      for (int j2 = 0; j2 < 64; ++j2) out[j2 * 64] = 0.0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

// exact per-feature max |x - s_j| over all rows of A and B (one HBM-bound read) and fp64 column
// sums of A and of B: thread = a 16-byte column piece (D % 4 == 0), rows strided over the grid;
// block max -> atomicMax on the non-negative float bits (non-finite values force +inf); block
// sums (fixed order) -> csum_part[block][set][D] for gram_i8_reduce_kernel (fixed order again).
// Non-finite input propagates into the sums and is flagged there.
__global__ void __launch_bounds__(256) i8_colmax_kernel(const float* __restrict__ A, int64_t nA,
                                                        const float* __restrict__ B, int64_t nB, int D,
                                                        const double* __restrict__ s, unsigned* colmax,
                                                        double* csum_part) {
  const int P = D / 4;  // pieces per row
  const int rows_per_block = blockDim.x / P;
  const int piece = threadIdx.x % P, rsub = threadIdx.x / P;
  __shared__ unsigned red[256 * 4];
  __shared__ double sred[256 * 8];
  float m[4] = {0.f, 0.f, 0.f, 0.f};
  double sum[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
  float sf[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) sf[i] = static_cast<float>(s[4 * piece + i]);
  if (rsub < rows_per_block) {
    const int64_t N = nA + nB;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * rows_per_block;
    int64_t r = static_cast<int64_t>(blockIdx.x) * rows_per_block + rsub;
    // four rows in flight per iteration (memory-level parallelism: the register budget limits the
    // resident threads), then the remainder one at a time
    for (; r + 3 * stride < N; r += 4 * stride) {
      float4 vv[4];
      bool ia[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t ru = r + u * stride;
        ia[u] = ru < nA;
        vv[u] = __ldg(reinterpret_cast<const float4*>(ia[u] ? A + ru * D : B + (ru - nA) * D) + piece);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float4 v = vv[u];
        m[0] = fmaxf(m[0], fabsf(v.x - sf[0]));
        m[1] = fmaxf(m[1], fabsf(v.y - sf[1]));
        m[2] = fmaxf(m[2], fabsf(v.z - sf[2]));
        m[3] = fmaxf(m[3], fabsf(v.w - sf[3]));
        if (ia[u]) {  // warp-uniform: a warp's lanes read pieces of the same row
          sum[0][0] += static_cast<double>(v.x);
          sum[0][1] += static_cast<double>(v.y);
          sum[0][2] += static_cast<double>(v.z);
          sum[0][3] += static_cast<double>(v.w);
        } else {
          sum[1][0] += static_cast<double>(v.x);
          sum[1][1] += static_cast<double>(v.y);
          sum[1][2] += static_cast<double>(v.z);
          sum[1][3] += static_cast<double>(v.w);
        }
      }
    }
    for (; r < N; r += stride) {
      const bool inA = r < nA;
      const float* row = inA ? A + r * D : B + (r - nA) * D;
      const float4 v = __ldg(reinterpret_cast<const float4*>(row) + piece);
      m[0] = fmaxf(m[0], fabsf(v.x - sf[0]));
      m[1] = fmaxf(m[1], fabsf(v.y - sf[1]));
      m[2] = fmaxf(m[2], fabsf(v.z - sf[2]));
      m[3] = fmaxf(m[3], fabsf(v.w - sf[3]));
      if (inA) {  // warp-uniform: a warp's lanes read pieces of the same row
        sum[0][0] += static_cast<double>(v.x);
        sum[0][1] += static_cast<double>(v.y);
        sum[0][2] += static_cast<double>(v.z);
        sum[0][3] += static_cast<double>(v.w);
      } else {
        sum[1][0] += static_cast<double>(v.x);
        sum[1][1] += static_cast<double>(v.y);
        sum[1][2] += static_cast<double>(v.z);
        sum[1][3] += static_cast<double>(v.w);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    red[threadIdx.x * 4 + i] = __float_as_uint(m[i]);
    sred[threadIdx.x * 8 + i] = sum[0][i];
    sred[threadIdx.x * 8 + 4 + i] = sum[1][i];
  }
  __syncthreads();
  if (rsub == 0) {
    unsigned mm[4] = {0u, 0u, 0u, 0u};
    double sa[4] = {0.0, 0.0, 0.0, 0.0}, sb[4] = {0.0, 0.0, 0.0, 0.0};
    for (int q = 0; q < rows_per_block; ++q) {
      const int t = q * P + piece;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        mm[i] = max(mm[i], red[t * 4 + i]);
        sa[i] += sred[t * 8 + i];
        sb[i] += sred[t * 8 + 4 + i];
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      atomicMax(&colmax[4 * piece + i], mm[i]);
      csum_part[(static_cast<int64_t>(blockIdx.x) * 2 + 0) * D + 4 * piece + i] = sa[i];
      csum_part[(static_cast<int64_t>(blockIdx.x) * 2 + 1) * D + 4 * piece + i] = sb[i];
    }
  }
}

// per-feature 2^k (the largest power of two with M_j 2^k <= 2^30, M_j = max |x - s_j| over all
// rows: F stays within +-2^30, half the int32 range) and the integer shift S_j = rint(s_j 2^k),
// rounded so that it is exact in fp32 (the slicer subtracts it in an FMA)
__global__ void i8_scale_kernel(int D, const double* __restrict__ s, const unsigned* __restrict__ colmax,
                                float* scale, float* shiftf, unsigned* overflow) {
  for (int f = threadIdx.x; f < D; f += blockDim.x) {
    const float M = __uint_as_float(colmax[f]);
    int k = 0;
    if (!(M < 3.0e38f)) {
      atomicOr(overflow, 1u);  // non-finite input (or out of range): the DMMA path reports it
    } else if (M > 0.0f) {
      int e;
      frexp(static_cast<double>(M), &e);  // M < 2^e
      k = 30 - e;
      // |F| <= M 2^k + 1/2 (+ the fp32 rounding of the FMA, ulp 64 below 2^30): keep F <= 2^30 - 64
      // so the top digit lies in [-64, 63] and the doubled top plane fits int8 (colmax itself is
      // rounded to fp32: a 2^-24 relative margin)
      if (ldexp(static_cast<double>(M), k) > 0x1p30 - 256.0) --k;
    }
    k = k > 100 ? 100 : (k < -100 ? -100 : k);
    const double sck = ldexp(1.0, k);
    scale[f] = static_cast<float>(sck);
    shiftf[f] = static_cast<float>(rint(static_cast<double>(static_cast<float>(s[f] * sck))));
  }
}

// G <- (G + G^T) / 2: the slabs hold Z = sum_L 2^(-8L) Z_L with Z_L + Z_L^T = 2 G_L (the pairs
// (0, u), u > 0, are accumulated once as 2 d_0 d_u); thread (i, j > i) owns both entries
__global__ void __launch_bounds__(256) gram_i8_sym_kernel(int D, double* G) {
  const int i = blockIdx.x, j = threadIdx.x;
  if (i < D && j < D && j > i) {
    const double v = 0.5 * (G[static_cast<int64_t>(i) * D + j] + G[static_cast<int64_t>(j) * D + i]);
    G[static_cast<int64_t>(i) * D + j] = v;
    G[static_cast<int64_t>(j) * D + i] = v;
  }
}

// G^T = 2^(-k_i - k_j) sum over groups and pair types of the slabs (fixed order), S_X, s'.
// Block = slab column i, thread = feature row j: every slab column is read coalesced (1 KB per
// CTA half), and the 3 x ngroups loads of a thread are independent (memory-level parallelism).
// The transpose is immaterial: gram_i8_sym_kernel takes the symmetric part.
__global__ void __launch_bounds__(256) gram_i8_reduce_kernel(I8Args a, double* G, double* SA, double* SB, double* s) {
  const int D = a.D;
  const int i = blockIdx.x, j = threadIdx.x;
  if (i < D && j < D) {
    const int r = j / kFeat, row = j % kFeat;
    const int64_t cstride = static_cast<int64_t>(kFeat) * 256;  // one CTA slab
    const double* base = a.slab + static_cast<int64_t>(r) * cstride + static_cast<int64_t>(i) * kFeat + row;
    double part[4] = {0.0, 0.0, 0.0, 0.0};  // fixed interleave over groups: deterministic
#pragma unroll 4
    for (int g = 0; g < a.ngroups; ++g) {
      const double* gb = base + static_cast<int64_t>(g * 3) * 2 * cstride;
      part[g & 3] += __ldg(gb) + __ldg(gb + 2 * cstride) + __ldg(gb + 4 * cstride);  // types 0, 1, 2
    }
    const double acc = (part[0] + part[1]) + (part[2] + part[3]);
    // slabs carry sum_L 2^(-8L) G_L = 2^-48 sum_L 2^(8 (6 - L)) G_L
    G[static_cast<int64_t>(i) * D + j] =
        ldexp(acc, 48) / (static_cast<double>(a.scale[i]) * static_cast<double>(a.scale[j]));
  }
  // column sums of feature i (this block's row index): thread t adds partials t, t + 256, ... of
  // A and of B, then a fixed tree over the block -- deterministic, and the 1184 partials are read
  // by 256 threads instead of one sequential chain
  __shared__ double red[2][256];
  double sa = 0.0, sb = 0.0;
  if (i < D)
    for (int b = j; b < a.ncs; b += blockDim.x) {
      sa += a.cpart[(static_cast<int64_t>(b) * 2 + 0) * D + i];
      sb += a.cpart[(static_cast<int64_t>(b) * 2 + 1) * D + i];
    }
  red[0][j] = sa;
  red[1][j] = sb;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (j < o) {
      red[0][j] += red[0][j + o];
      red[1][j] += red[1][j + o];
    }
    __syncthreads();
  }
  if (j == 0 && i < D) {
    sa = red[0][0];
    sb = red[1][0];
    if (!isfinite(sa) || !isfinite(sb)) atomicOr(a.overflow, 1u);  // non-finite input: the DMMA path reports it
    const double sp = (static_cast<double>(a.shiftf[i]) + 128.0 * 65793.0) / static_cast<double>(a.scale[i]);
    SA[i] = sa - static_cast<double>(a.nA) * sp;  // sums about s' = (S + c0) 2^-k
    SB[i] = sb - static_cast<double>(a.nB) * sp;
    s[i] = sp;
  }
}

// Sharded phase (prohd_local_moments_i8): the moments about the fixed-point shift s' re-expressed
// about the caller's shift s, d = s' - s: sum (x - s)(x - s)^T = G' + d S'^T + S' d^T + N d d^T with
// S' = S'_A + S'_B, and S_X = S'_X + n_X d (d is below the grid step 2^-k_j; fp64 throughout).
__global__ void __launch_bounds__(256) i8_reshift_gram_kernel(int D, int64_t N, const double* __restrict__ s_to,
                                                              const double* __restrict__ s_from,
                                                              const double* __restrict__ SA,
                                                              const double* __restrict__ SB, double* G) {
  const int i = blockIdx.x;
  const double di = s_from[i] - s_to[i], Si = SA[i] + SB[i];
  for (int j = threadIdx.x; j < D; j += blockDim.x) {
    const double dj = s_from[j] - s_to[j], Sj = SA[j] + SB[j];
    // every term symmetric in (i, j) bit for bit: G stays exactly symmetric
    G[static_cast<int64_t>(i) * D + j] += (di * Sj + Si * dj) + static_cast<double>(N) * (di * dj);
  }
}
__global__ void i8_reshift_sums_kernel(int D, int64_t nA, int64_t nB, const double* __restrict__ s_to, double* s_from,
                                       double* SA, double* SB) {
  for (int j = threadIdx.x; j < D; j += blockDim.x) {
    const double d = s_from[j] - s_to[j];
    SA[j] += static_cast<double>(nA) * d;
    SB[j] += static_cast<double>(nB) * d;
    s_from[j] = s_to[j];
  }
}

// D <= 128: G = 2^(-k_i - k_j) sym(sum over CTA slabs), the symmetric part taken in the same pass
// (block i reads column i and row i of every slab: 0.5 (sum_c Z_c[i][j] + sum_c Z_c[j][i]) is the
// same value for blocks i and j). Thread (grp, j) sums the slabs grp, grp + ngrp, ... in order,
// then thread j adds the groups' partials in order (deterministic); the column sums as in
// gram_i8_reduce_kernel.
constexpr int kSRedThreads = 512;
__global__ void __launch_bounds__(kSRedThreads) gram_i8s_reduce_kernel(I8Args a, double* G, double* SA, double* SB,
                                                                      double* s) {
  const int D = a.D;
  const int i = blockIdx.x, t = threadIdx.x;
  const int ngrp = kSRedThreads / D;  // D <= 128: >= 4 groups
  const int grp = t / D, j = t % D;
  __shared__ double part[2][kSRedThreads];
  const int nct = a.nt0 + a.nt1;
  if (grp < ngrp) {
    // coalesced: the slabs' column i (contiguous over j); the transpose is summed by
    // gram_i8_sym_kernel afterwards (a strided second read here cost as much as the Gram at cfg2)
    double p0 = 0.0, p1 = 0.0;
    if (a.small == 2) {  // gram_i8d_kernel slabs [quadrant][64 column][64 row]: the quadrants add up
      const double* col = a.slab + static_cast<int64_t>(i) * 64 + j;
      for (int c = grp; c < nct; c += ngrp) {
        const int64_t o = static_cast<int64_t>(c) * kSmallSlab;
        p0 += (__ldg(col + o) + __ldg(col + o + 4096)) + (__ldg(col + o + 8192) + __ldg(col + o + 12288));
      }
    } else {  // gram_i8s_kernel slabs [column 128][row 128]
      const double* col = a.slab + static_cast<int64_t>(i) * 128 + j;
      int c = grp;
      for (; c + ngrp < nct; c += 2 * ngrp) {
        p0 += __ldg(col + static_cast<int64_t>(c) * kSmallSlab);
        p1 += __ldg(col + static_cast<int64_t>(c + ngrp) * kSmallSlab);
      }
      if (c < nct) p0 += __ldg(col + static_cast<int64_t>(c) * kSmallSlab);
    }
    part[0][t] = p0 + p1;
  }
  __syncthreads();
  if (t < D) {
    double p = 0.0;
    for (int g2 = 0; g2 < ngrp; ++g2) p += part[0][g2 * D + t];
    // slabs carry 2^-48 sum_L 2^(8 (6 - L)) G_L (gram_i8_sym_kernel then takes the symmetric part)
    G[static_cast<int64_t>(i) * D + t] =
        ldexp(p, 48) / (static_cast<double>(a.scale[i]) * static_cast<double>(a.scale[t]));
  }
  __syncthreads();
  double sa = 0.0, sb = 0.0;
  for (int b = t; b < a.ncs; b += kSRedThreads) {
    sa += a.cpart[(static_cast<int64_t>(b) * 2 + 0) * D + i];
    sb += a.cpart[(static_cast<int64_t>(b) * 2 + 1) * D + i];
  }
  part[0][t] = sa;
  part[1][t] = sb;
  __syncthreads();
  for (int o = kSRedThreads / 2; o > 0; o >>= 1) {
    if (t < o) {
      part[0][t] += part[0][t + o];
      part[1][t] += part[1][t + o];
    }
    __syncthreads();
  }
  if (t == 0) {
    sa = part[0][0];
    sb = part[1][0];
    if (!isfinite(sa) || !isfinite(sb)) atomicOr(a.overflow, 1u);
    const double sp = (static_cast<double>(a.shiftf[i]) + 128.0 * 65793.0) / static_cast<double>(a.scale[i]);
    SA[i] = sa - static_cast<double>(a.nA) * sp;
    SB[i] = sb - static_cast<double>(a.nB) * sp;
    s[i] = sp;
  }
}

}  // namespace

bool plan_gram_i8(int64_t nA, int64_t nB, int D, int num_sms, GramI8Plan& p) {
  if (D > 256 || D % 4 != 0 || nA < 0 || nB < 0 || nA + nB < 1) return false;  // a shard may hold one set only
  const int sms = num_sms > 0 ? num_sms : 148;
  p.D = D;
  p.csum_count = static_cast<int64_t>(kColmaxBlocks) * 2 * D;
  if (D <= 128) {
    // one CTA per SM; at least 4 chunks per CTA (option k1_i8_ctas caps the count: tests force
    // mid-sweep drains with it)
    int64_t T = (nA + nB) / (4 * kPts);
    if (T > sms) T = sms;
    if (opt(OPT_K1_I8_CTAS) > 0 && T > opt(OPT_K1_I8_CTAS)) T = opt(OPT_K1_I8_CTAS);
    if (T < 2) T = 2;
    if (D <= 64) {  // paired digit planes: one CTA type (gram_i8d_kernel)
      p.small = 2;
      p.nt0 = static_cast<int>(T);
      p.nt1 = 0;
      p.ngroups = 0;
      p.nctas = p.nt0;
      p.slab_doubles = static_cast<int64_t>(p.nctas) * kSmallSlab;
      return true;
    }
    p.small = 1;
    p.nt0 = static_cast<int>((T * kSet0Share + kSetShares / 2) / kSetShares);
    if (p.nt0 < 1) p.nt0 = 1;
    p.nt1 = static_cast<int>(T) - p.nt0;
    if (p.nt1 < 1) p.nt1 = 1;
    p.ngroups = 0;
    p.nctas = p.nt0 + p.nt1;
    p.slab_doubles = static_cast<int64_t>(p.nctas) * kSmallSlab;
    return true;
  }
  const int pairs = sms / 2;
  int groups = pairs / 3;  // a group = one pair of each type
  const int64_t per = (nA + nB) / (groups > 0 ? groups : 1);
  if (per < 4 * kPts) groups = static_cast<int>((nA + nB) / (4 * kPts));  // small problems: fewer groups
  if (opt(OPT_K1_I8_CTAS) > 0 && groups * 6 > opt(OPT_K1_I8_CTAS)) groups = static_cast<int>(opt(OPT_K1_I8_CTAS) / 6);
  if (groups < 1) return false;
  p.small = 0;
  p.ngroups = groups;
  p.nctas = groups * 6;
  p.slab_doubles = static_cast<int64_t>(p.nctas) * kFeat * 256;
  return true;
}

size_t gram_i8_ws_bytes(const GramI8Plan& p) {
  return static_cast<size_t>(round_up(p.slab_doubles * 8, 256) + round_up(p.csum_count * 8, 256) + 256 * 4 * 3 +
                             256);
}

cudaError_t launch_gram_i8(const GramI8Plan& p, const float* A, int64_t nA, const float* B, int64_t nB,
                           uint8_t* ws, double* s, double* G, double* SA, double* SB, unsigned* overflow,
                           cudaStream_t st, const float* colmax_in, const double* s_to) {
  const int D = p.D;
  double* slab = reinterpret_cast<double*>(ws);
  double* cpart = reinterpret_cast<double*>(ws + round_up(p.slab_doubles * 8, 256));
  float* scale = reinterpret_cast<float*>(ws + round_up(p.slab_doubles * 8, 256) + round_up(p.csum_count * 8, 256));
  float* shiftf = scale + 256;
  CUtensorMap maps[2];
  char err[256];
  // raw fp32 boxes [32 features x 64 rows], SWIZZLE_128B (four per chunk and CTA)
  PFN_encodeTiled enc = get_encode();
  if (enc == nullptr) return cudaErrorNotSupported;
  // a set without rows (a shard of the sharded phase) gets the other set's map: it is never read
  const float* src[2] = {nA > 0 ? A : B, nB > 0 ? B : A};
  const int64_t rows[2] = {nA > 0 ? nA : nB, nB > 0 ? nB : nA};
  for (int i = 0; i < 2; ++i) {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(rows[i])};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(D) * 4};
    cuuint32_t box[2] = {32u, static_cast<cuuint32_t>(kPts)};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(src[i]), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  (void)err;
  unsigned* colmax = reinterpret_cast<unsigned*>(shiftf + 256);
  cudaError_t e0 = cudaMemsetAsync(colmax, 0, sizeof(unsigned) * 256, st);
  if (e0 != cudaSuccess) return e0;
  count_launch();
  i8_colmax_kernel<<<kColmaxBlocks, 256, 0, st>>>(A, nA, B, nB, D, s, colmax, cpart);
  count_launch();
  // the grid: this call's own column maxima, or (sharded phase) the MAX over ranks
  i8_scale_kernel<<<1, 256, 0, st>>>(D, s, colmax_in != nullptr ? reinterpret_cast<const unsigned*>(colmax_in) : colmax,
                                     scale, shiftf, overflow);
  I8Args a{nA, nB, D, p.ngroups, scale, shiftf, slab, cpart, kColmaxBlocks, overflow,
           opt(OPT_K1_ABLATE) > 0 ? static_cast<int>(opt(OPT_K1_ABLATE)) : 0, p.small, p.nt0, p.nt1};
  auto kern = p.small == 2 ? gram_i8d_kernel : (p.small == 1 ? gram_i8s_kernel : gram_i8_kernel);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem));
  if (e != cudaSuccess) return e;
  count_launch();
  kern<<<p.nctas, kThreads, kSmem, st>>>(maps[0], maps[1], a);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (p.small) {
    count_launch();
    gram_i8s_reduce_kernel<<<D, kSRedThreads, 0, st>>>(a, G, SA, SB, s);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    count_launch();
    gram_i8_sym_kernel<<<D, 256, 0, st>>>(D, G);
  } else {
    count_launch();
    gram_i8_reduce_kernel<<<D, 256, 0, st>>>(a, G, SA, SB, s);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    count_launch();
    gram_i8_sym_kernel<<<D, 256, 0, st>>>(D, G);
  }
  if (s_to != nullptr) {
    count_launch(2);
    i8_reshift_gram_kernel<<<D, 256, 0, st>>>(D, nA + nB, s_to, s, SA, SB, G);
    i8_reshift_sums_kernel<<<1, 256, 0, st>>>(D, nA, nB, s_to, s, SA, SB);
  }
  return cudaGetLastError();
}

cudaError_t launch_colmax_i8(const GramI8Plan& p, const float* A, int64_t nA, const float* B, int64_t nB,
                             uint8_t* ws, const double* s, float* colmax_out, cudaStream_t st) {
  const int D = p.D;
  double* cpart = reinterpret_cast<double*>(ws + round_up(p.slab_doubles * 8, 256));
  float* scale = reinterpret_cast<float*>(ws + round_up(p.slab_doubles * 8, 256) + round_up(p.csum_count * 8, 256));
  unsigned* colmax = reinterpret_cast<unsigned*>(scale + 512);
  cudaError_t e = cudaMemsetAsync(colmax, 0, sizeof(unsigned) * 256, st);
  if (e != cudaSuccess) return e;
  count_launch();
  i8_colmax_kernel<<<kColmaxBlocks, 256, 0, st>>>(A, nA, B, nB, D, s, colmax, cpart);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return cudaMemcpyAsync(colmax_out, colmax, sizeof(float) * D, cudaMemcpyDeviceToDevice, st);
}

}  // namespace prohd
