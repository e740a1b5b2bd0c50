// k_project_tc.cu — K3 on the tensor cores: pi = X u_l for the k+1 directions of one set
// (Alg. 1 lines 3-4 and Alg. 2 lines 4-5; pi = x^T u),
// as a skinny tcgen05 GEMM P[128 points x 32 directions] per tile, 3xTF32, plus max ||x||^2
// for K4's guard band.
//
// With x = xh + xl (xh = x with the low 13 mantissa bits cleared, xl = x - xh exact) and
// u = uh + ul likewise (u = the fp32 direction U32),
//     x . u ~= xh . [uh ; ul]  (one N = 64 MMA: columns 0-31 xh.uh, 32-63 xh.ul)
//            + xl . uh          (one N = 32 MMA on the first 32 rows: columns 64-95)
// and the epilogue adds the three columns of each direction. Each operand tile is read
// by the tensor core once per K-step (2 MMAs instead of 3), which keeps shared memory
// below its bandwidth at the HBM rate of streaming the points.
//
// Error bound (used by K4's collect_kernel through eps_coef, prohd_kernels.cuh):
//   |pi_tc - pi_64| <= [ 2^-24 (u64 -> u32) + 3 * 2^-20 (dropped xl.ul, TF32 truncation of
//   xl and ul) + (D / 8 + 1) * 2^-19 (fp32 accumulation inside the tensor core, modelled
//   pessimistically as 2^-19 (|acc| + sum |products|) per K = 8 MMA, |acc| <= ||x||; the
//   xh.ul and xl.uh chains are 2^-10 smaller) + 3 * 2^-24 (epilogue adds) ] * ||x||, since
//   sum_i |x_i| |u_i| <= ||x|| ||u|| = ||x||.
// tests/test_gpu_select.py measures the actual |pi_tc - pi_64| / ||x|| on every BASELINE
// config against this bound.
//
// The tensor core reads an fp32 operand as TF32 by ignoring its low 13 mantissa bits
// (truncation), so the TMA-staged box itself is the xh operand and only xl is written.
// Measured: bit-identical projections with an explicitly truncated xh on all five BASELINE
// generators; were the hardware to round instead, xh + xl would miss x by up to 2^-11 |x| and
// tests/test_gpu_select.py (error <= eps, measured ~1e-7 ||x||) would fail.
//
// Structure (persistent, 1 CTA per SM, 448 threads, warp-specialised like K6):
//   warp 0     TMA producer: per K-chunk (32 features) a [128 x 32] fp32 box, SWIZZLE_128B,
//              into a kStagesP-deep ring (128 KB in flight per SM: the HBM latency-bandwidth
//              product at the per-SM share of the bandwidth).
//   warp 1     TMEM allocation (2 accumulators x 128 columns) and the single-thread MMA
//              issuer: per K-step of 8, MMA(xh, [uh;ul], N=64) and MMA(xl, uh, N=32); commits
//              free the box slot and the xl slot.
//   warps 2-9  converters (2 per SM sub-partition): a warp owns 16 point rows of the box, a
//              lane one half row (lanes 2i, 2i + 1 share row i, so a quarter-warp touches 8
//              distinct 16-B bank groups); it writes xl = x - trunc(x) into one of kLoSlots xl
//              tiles and accumulates ||x||^2 (fp32, halves combined by one shuffle per tile);
//              fence.proxy.async, then one arrive per warp.
//   warps 10-13 epilogue: tcgen05.ld of the 96 columns (row = point), pi_l = c_l + c_{32+l}
//              + c_{64+l}, stored direction-major P32[l * n + p] (coalesced per l); or, with the
//              sampled K4 (k_select.cu launch_select_sampled), (index, pi_l) appended to the
//              list of every (direction, tail) whose sample threshold the point passes.
// The directions are written once per CTA into shared memory in the UMMA K-major SWIZZLE_128B
// layout: per K-chunk a 64-row tile, rows 0-31 uh and rows 32-63 ul (zero past L and D).
#include "api_common.cuh"
#include "prohd_kernels.cuh"
#include "sm100.cuh"

namespace prohd {
namespace {

constexpr int kStagesP = 8;                   // TMA boxes in flight
constexpr int kLoSlots = 2;                   // xl tiles
constexpr int kPThreads = 448;
constexpr uint32_t kPBox = 128 * 128;         // 16 KB: 128 points x 32 fp32
constexpr uint32_t kPStage = kPBox;           // xh = the TMA-staged fp32 box
constexpr uint32_t kUChunk = 64 * 128;        // 8 KB: [uh ; ul] 64 rows x 32 fp32
constexpr int kPMaxChunks = 8;                // D <= 256
constexpr uint32_t kPTmemCols = 256;          // 2 accumulators x 128 columns (96 used)
constexpr size_t kPSmem =
    static_cast<size_t>(kStagesP) * kPStage + kLoSlots * kPBox + kPMaxChunks * kUChunk + 1024 + 256;

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// UMMA instruction descriptor, kind::tf32 (see sm100.cuh)
__host__ __device__ constexpr uint32_t idesc_p(uint32_t M, uint32_t N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ float tf32_trunc(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }
// explicit shared-space accesses (the 1024-aligned carve-out is a generic pointer to the compiler)
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

__global__ void __launch_bounds__(kPThreads, 1)
    project_tc_kernel(const __grid_constant__ CUtensorMap tX, int64_t n, int D, const float* __restrict__ U32, int L,
                      float* __restrict__ P32, unsigned* maxnorm2, ProjectFuse fz) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* lobase = smem + kStagesP * kPStage;     // [kLoSlots] xl tiles
  uint8_t* ubase = lobase + kLoSlots * kPBox;       // [chunk][uh rows 0-31 ; ul rows 32-63]
  const int nk = (D + 31) / 32;
  uint64_t* full = reinterpret_cast<uint64_t*>(ubase + kPMaxChunks * kUChunk);
  uint64_t* conv = full + kStagesP;
  uint64_t* empty = conv + kStagesP;
  uint64_t* loempty = empty + kStagesP;
  uint64_t* tfull = loempty + kLoSlots;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ unsigned bmax;
  __shared__ float sthr[64];  // fused selection: per (direction, tail) sample threshold
  __shared__ unsigned wcnt[4][64];  // fused selection: fill counts of the epilogue warps' slabs

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t ntiles = (n + 127) / 128;

  // directions: rows r and 32 + r of chunk c hold uh and ul of features 32c .. 32c+31 of
  // direction r (0 past L / D), 16-B piece j of each 128-B row at position j ^ (row & 7)
  for (int e = threadIdx.x; e < nk * 32 * 32; e += blockDim.x) {
    const int c = e / 1024, r = (e / 32) % 32, k = e % 32;
    const int f = c * 32 + k;
    const float u = (r < L && f < D) ? U32[static_cast<int64_t>(r) * D + f] : 0.0f;
    const float uh = tf32_trunc(u);
    const uint32_t piece = (((k >> 2) ^ (r & 7)) << 4) + (k & 3) * 4;  // (r + 32) & 7 == r & 7
    *reinterpret_cast<float*>(ubase + c * kUChunk + r * 128 + piece) = uh;
    *reinterpret_cast<float*>(ubase + c * kUChunk + (32 + r) * 128 + piece) = u - uh;
  }
  if (fz.state != nullptr) {
    for (int i = threadIdx.x; i < 2 * L; i += blockDim.x) sthr[i] = __uint_as_float(fz.state[i * 4 + 0]);
    for (int i = threadIdx.x; i < 4 * 64; i += blockDim.x) (&wcnt[0][0])[i] = 0u;
  }
  if (threadIdx.x == 0) {
    bmax = 0u;
    for (int i = 0; i < kStagesP; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&conv[i], 8);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < kLoSlots; ++i) mbar_init(&loempty[i], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) tma_prefetch(&tX);
  if (warp == 1) tmem_alloc<kPTmemCols>(tmem_slot);
  fence_proxy_async();  // the direction tiles are read by the tensor core (async proxy)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int c = 0; c < nk; ++c) {
          mbar_wait(&empty[stage], phase ^ 1u);
          mbar_arrive_expect_tx(&full[stage], kPBox);
          tma_load_2d(smem + stage * kPStage, &tX, c * 32, static_cast<int32_t>(t * 128), &full[stage]);
          if (++stage == kStagesP) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    {
      // ------------------------------------------------------------ MMA issuer (warp-wide, elected lane issues)
      constexpr uint32_t id64 = idesc_p(128, 64), id32 = idesc_p(128, 32);
      const uint32_t u0 = smem_u32(ubase);
      int stage = 0;
      uint32_t phase = 0;
      int lslot = 0;
      int acc = 0;
      uint32_t aphase = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(&tempty[acc], aphase ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(acc * 128);
        for (int c = 0; c < nk; ++c) {
          mbar_wait(&conv[stage], phase);
          tc_fence_after();
          const uint32_t xh = smem_u32(smem + stage * kPStage), xl = smem_u32(lobase + lslot * kPBox);
          const uint32_t ub = u0 + c * kUChunk;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t off = static_cast<uint32_t>(kk * 32);  // 8 tf32 along K
            const uint32_t accum = (c | kk) != 0 ? 1u : 0u;
            mma_tf32_w(d, smem_desc_k_sw128(xh + off), smem_desc_k_sw128(ub + off), id64, accum);       // xh.[uh;ul]
            mma_tf32_w(d + 64, smem_desc_k_sw128(xl + off), smem_desc_k_sw128(ub + off), id32, accum);  // xl.uh
          }
          mma_commit_w(&empty[stage]);
          mma_commit_w(&loempty[lslot]);
          lslot = lslot + 1 == kLoSlots ? 0 : lslot + 1;
          if (++stage == kStagesP) {
            stage = 0;
            phase ^= 1u;
          }
        }
        mma_commit_w(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) aphase ^= 1u;
      }
    }
    __syncwarp();
  } else if (warp < 10) {
    // -------------------------------------------------------------- converters
    const int r = (warp - 2) * 16 + (lane >> 1);  // point row of the box
    const int half = lane & 1;                     // 16-B pieces 4 half .. 4 half + 3 of the row
    int stage = 0;
    uint32_t phase = 0;
    int lslot = 0;
    uint32_t lphase = 0;
    float wmax = 0.0f;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      float nrm = 0.0f;
      for (int c = 0; c < nk; ++c) {
        mbar_wait(&full[stage], phase);
        mbar_wait(&loempty[lslot], lphase ^ 1u);
        const uint32_t xh = smem_u32(smem + stage * kPStage + r * 128);
        const uint32_t xl = smem_u32(lobase + lslot * kPBox + r * 128);
#pragma unroll
        for (int q0 = 0; q0 < 4; ++q0) {
          const int q = half * 4 + ((q0 + r) & 3);  // quarter-warp: 4 rows x 2 halves = 8 bank groups
          const float4 v = lds128(xh + q * 16);
          nrm = fmaf(v.x, v.x, nrm);
          nrm = fmaf(v.y, v.y, nrm);
          nrm = fmaf(v.z, v.z, nrm);
          nrm = fmaf(v.w, v.w, nrm);
          const float4 h = make_float4(tf32_trunc(v.x), tf32_trunc(v.y), tf32_trunc(v.z), tf32_trunc(v.w));
          sts128(xl + q * 16, make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w));
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[stage]);
        if (++lslot == kLoSlots) {
          lslot = 0;
          lphase ^= 1u;
        }
        if (++stage == kStagesP) {
          stage = 0;
          phase ^= 1u;
        }
      }
      nrm += __shfl_xor_sync(0xffffffffu, nrm, 1);  // the two halves of the row
      if (t * 128 + r < n)  // non-finite input must poison the max (fmaxf would drop a NaN)
        wmax = (isfinite(nrm) && isfinite(wmax)) ? fmaxf(wmax, nrm) : __int_as_float(0x7fffffff);
    }
    atomicMax(&bmax, __float_as_uint(wmax));  // non-negative floats (and the NaN pattern) order as uints
  } else {
    // -------------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quarter
    const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
    int acc = 0;
    uint32_t aphase = 0;
    const int slab = blockIdx.x * 4 + (warp - 10);  // fused selection: this warp's slab
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const uint32_t ta = tmem_base + lane_addr + static_cast<uint32_t>(acc * 128);
      float a0[32], a1[32], a2[32];
      tmem_ld32(ta, a0);
      tmem_ld32(ta + 32, a1);
      tmem_ld32(ta + 64, a2);
      tmem_wait_ld();
      const int64_t p = t * 128 + q * 32 + lane;
      if (fz.state == nullptr) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (p < n) {
#pragma unroll
          for (int l = 0; l < 32; ++l)
            if (l < L) P32[static_cast<int64_t>(l) * n + p] = (a0[l] + a1[l]) + a2[l];
        }
      } else {
        // fused K4 pre-selection: (index, pi32) of every point beyond its list's sample
        // threshold, appended to this warp's private slab of the list (P32 is not written).
        // Pass 1 (unrolled, a few instructions per direction): the lists this lane's point
        // enters, as bits of (lo, hi) = lists 0-31, 32-63. Pass 2 only if the warp has any: a
        // rolled loop over the warp's lists that reloads the direction's three accumulator
        // columns from TMEM (the accumulator is released after it), a ballot, the fill count
        // (lane 0, shared memory) and the stores. Small executed code: the converters' loop
        // keeps the instruction cache.
        const bool ok = p < n;
        unsigned bits_lo = 0, bits_hi = 0;
        if (fz.ablate != 1) {
#pragma unroll
          for (int l = 0; l < 32; ++l)
            if (l < L) {
              const float v = (a0[l] + a1[l]) + a2[l];
              const unsigned b2 = (ok && v >= sthr[2 * l] ? 1u : 0u) | (ok && v <= sthr[2 * l + 1] ? 2u : 0u);
              if (2 * l < 32)
                bits_lo |= b2 << (2 * l);
              else
                bits_hi |= b2 << (2 * l - 32);
            }
        }
        const unsigned wlo = __reduce_or_sync(0xffffffffu, bits_lo), whi = __reduce_or_sync(0xffffffffu, bits_hi);
        if ((wlo | whi) != 0u && fz.ablate != 2) {
          unsigned* wc = wcnt[warp - 10];
          const unsigned below = (1u << lane) - 1u;
          const int64_t sbase = static_cast<int64_t>(slab) * 2 * L;
#pragma unroll 1
          for (int half = 0; half < 2; ++half) {
            unsigned wb = half == 0 ? wlo : whi;
            const unsigned mine = half == 0 ? bits_lo : bits_hi;
#pragma unroll 1
            while (wb != 0u) {
              const int bit = __ffs(wb) - 1;
              wb &= wb - 1u;
              const int lt = 32 * half + bit, l = lt >> 1;
              const bool pr = (mine >> bit) & 1u;
              const unsigned bal = __ballot_sync(0xffffffffu, pr);
              float c0, c1, c2;
              asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=f"(c0) : "r"(ta + l));
              asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=f"(c1) : "r"(ta + 32 + l));
              asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=f"(c2) : "r"(ta + 64 + l));
              tmem_wait_ld();
              const float v = (c0 + c1) + c2;  // pass 1's value (same operations, same order)
              unsigned base = 0;
              if (lane == 0) {
                base = wc[lt];
                wc[lt] = base + __popc(bal);
              }
              base = __shfl_sync(0xffffffffu, base, 0);
              const unsigned pos = base + __popc(bal & below);
              if (pr && pos < static_cast<unsigned>(fz.capw)) {
                const int64_t e = (sbase + lt) * fz.capw + pos;
                fz.sidx[e] = static_cast<int>(p);
                fz.sval[e] = v;
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
      acc ^= 1;
      if (acc == 0) aphase ^= 1u;
    }
    if (fz.state != nullptr) {  // slab fill counts (may exceed capw: the filter then fails the list)
      __syncwarp();
      for (int i = lane; i < 2 * L; i += 32) fz.wcount[slab * 2 * L + i] = wcnt[warp - 10][i];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(maxnorm2, bmax);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kPTmemCols>(tmem_base);
  }
}

}  // namespace

double project_tc_eps_coef(int D) {
  const double nk8 = static_cast<double>((D + 31) / 32 * 4);  // K = 8 MMAs per accumulator chain
  return 0x1p-24 + 3 * 0x1p-20 + (nk8 + 1) * 0x1p-19 + 3 * 0x1p-24;
}

bool project_tc_supported(int64_t n, int D, int L) {
  if (opt(OPT_K3_SIMT) == 1) return false;  // dev A/B: the SIMT tile kernel
  return n >= 1 && D % 4 == 0 && D <= 32 * kPMaxChunks && L >= 1 && L <= 32 && n <= 0x7FFFFFFFll;
}

cudaError_t launch_project_tc(const float* X, int64_t n, int D, const float* U32, int L, float* P32,
                              unsigned* maxnorm2, int num_sms, cudaStream_t st, const ProjectFuse* fuse,
                              int64_t row_stride) {
  CUtensorMap map;
  char err[256];
  if (!make_tmap_2d(&map, X, n, D, 128, err, sizeof(err), kBK, row_stride)) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(project_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kPSmem));
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (n + 127) / 128;
  const int grid = static_cast<int>(ntiles < num_sms ? ntiles : num_sms);
  count_launch();
  project_tc_kernel<<<grid, kPThreads, kPSmem, st>>>(map, n, D, U32, L, P32, maxnorm2,
                                                     fuse != nullptr ? *fuse : ProjectFuse{});
  return cudaGetLastError();
}

}  // namespace prohd
