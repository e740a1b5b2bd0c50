// k_gram.cu — K1 main pass: the fp64 Gram G = sum_{p in A u B} (p - s)(p - s)^T and the
// column sums S_A, S_B on the fp64 tensor pipe (DMMA), warp-specialised.
//
// PAPER.md Alg. 2 lines 1-2: the principal directions are eigenvectors of the
// covariance of the stacked set [X; Y]; K1 (k_moments.cu) turns (S_A, S_B, G) into the
// centroids (Alg. 1 line 1) and C = G/N - (mu - s)(mu - s)^T.
//
// Work decomposition. The upper triangle of G is cut into 32x32 warp tiles (I <= J over
// 32-feature blocks) and the tiles into GROUPS of <= 12 that together need <= 8 feature
// blocks (<= 256 features, staged in "slots"): for D <= 256 every group stages all of D and
// the tiles are split evenly (D = 256: 36 tiles in 3 groups of 12); for larger D each 4x4
// square of blocks on or above the diagonal gives one or two groups. A group with fewer
// than 12 tiles runs each tile on kRep = 2 or 4 warps that take alternate k-steps (partial
// accumulators summed by the reduce kernel), so small D still fills the MMA warps.
// A diagonal tile issues only its 10 8x8 blocks on or above the diagonal (A = B fragments).
// The diagonal tiles go four to a group, on warps 0-3 (one per SM sub-partition, whose DMMA
// pipe its 3 warps share), and each group gets CTAs in proportion to its busiest
// sub-partition's DMMA count: D = 256 has groups of 4+8, 4+8 and 0+12 tiles (42, 42 and 48
// DMMAs per k-step) over 47, 47 and 54 point ranges, against 48 x 49 when every tile was full.
// CTA = (group g, point range r), blockIdx = grp[g].cta0 + r, ONE CTA per SM, one wave.
//
// CTA = 16 warps:
//   warps 12-15 (loaders): thread ct owns 16-B pieces (4 features) of fixed column 4 (ct % P)
//            (P = 16-B pieces per staged row) in rows ct / P + (128 / P) it of every 16-point
//            chunk; it cp.asyncs them into a 4-stage fp32 ring, waits for its own copies only
//            (no loader barrier), converts each value ONCE to fp64 on the integer pipe (the
//            fp64 pipe is the DMMA pipe's shared resource; exact for normals and signed zeros,
//            a warp-uniform F2F fallback for subnormal / inf / nan; an fp64 subtraction only
//            when the shift kernel kept a shift s) into a 4-buffer fp64 tile ring.
//   warps 0-11 (MMA): warp w runs tile w % ntiles on k-steps (w / ntiles) + kRep u; per
//            k-step it loads 4 A and 4 B fragments (8 LDS.64, issued one k-step ahead) and
//            issues 16 DMMA.8x8x4 into a 32x32 fp64 register accumulator (64 regs).
// The column sums are NOT taken by the Gram warps: any fp64 add in a Gram CTA runs on the adder
// the DMMAs share and was measured to cost far more than its count suggests (fp64 adds in the
// loaders: 9.6 -> 12.6-13.1 ms; one extra DMMA per k-step against an indicator operand: 9.6 ->
// 11.1 ms). At D >= 224 the launch's last CTAs (colsum_role, one per SM of their own) stream the
// rows with 1-D bulk copies and add them up while the Gram CTAs run; below that colsum_kernel
// takes them in a separate HBM-bound pass (~0.65 ms at cfg5). The reduce kernel forms
// S_X = sum x - n_X s.
// Three MMA warps per SM sub-partition keep the DMMA pipe fed through the fragment-load and
// barrier gaps that left it 26% idle with two (the 8-warp, 2-CTA/SM version).
// Buffer hand-off with mbarriers: full[b] (loader warps arrive, MMA warps wait) and
// empty[b] (MMA warps arrive, loaders wait). Every warp writes its own partial slot;
// gram_reduce_kernel sums the slots in a fixed order (deterministic, bit-identical runs).
#include "internal.cuh"
#include "prohd_kernels.cuh"
#include "sm100.cuh"


namespace prohd {
namespace {

constexpr int kGT = 512;       // threads per CTA
constexpr int kMW = 12;        // MMA warps
constexpr int kGMC = 16;       // points per chunk (= 4 DMMA k-steps)
constexpr int kGNS = 4;        // fp32 staging stages
constexpr int kGNB = 4;        // fp64 tile buffers
constexpr int kSlotsMax = 8;   // staged feature blocks (<= 256 features)
constexpr int kRowF = 32 * kSlotsMax;                  // staged floats per row (max)
constexpr int kGLd = kRowF + 4;                        // fp64 row stride (conflict-free fragment loads)
constexpr int kGStageF = kGMC * kRowF;                 // floats per staging stage
constexpr size_t kGSmem = sizeof(float) * kGNS * kGStageF + sizeof(double) * kGNB * kGMC * kGLd;

struct GramArgs {
  const float* A;
  const float* B;
  int64_t nA, nB;
  int D;
  const double* s;
  int ngroups;
  double* Gpart;    // [cta][kMW warps][32][32]
  int ngram;        // Gram CTAs; CTAs ngram .. ngram + cs_ctas - 1 take the column sums
  int cs_ctas;
  int64_t cs_per;   // rows per column-sum CTA
  double* Cpart;        // column-sum partials [cs_blocks][2 sets][D]
  int cs_blocks;
  GramGroup grp[kGramMaxGroups];
};

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Column sums inside the Gram launch (D % 4 == 0): the last cs_ctas CTAs (one per SM, like
// the Gram CTAs) each stream a contiguous row range of A u B through shared memory with 1-D
// bulk copies (kCsBuf x 64 KB in flight; a chunk never straddles the A/B boundary) and add
// it up in fp64 on their own SMs' fp64 pipes, concurrently with the DMMA-bound Gram CTAs.
// Thread t sums column t % D over rows t / D, t / D + H, ... (H = 512 / D row phases);
// partial slot (q H + h) of Cpart, combined in a fixed order by gram_reduce_kernel.
constexpr int kCsBuf = 3;
constexpr uint32_t kCsBytes = 65536;
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   sm100::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(sm100::smem_u32(bar))
               : "memory");
}
__device__ __noinline__ void colsum_role(const GramArgs& a, uint8_t* gsm) {
  __shared__ uint64_t cbar[kCsBuf];
  const int tid = threadIdx.x;
  const int D = a.D;
  const int q = blockIdx.x - a.ngram;
  const int64_t N = a.nA + a.nB;
  const int64_t r0 = static_cast<int64_t>(q) * a.cs_per;
  const int64_t r1 = r0 + a.cs_per < N ? r0 + a.cs_per : N;
  const int64_t rpc = kCsBytes / (4 * D);  // rows per chunk
  // chunk k of this range: rows [c0, c1), cut at nA
  auto chunk = [&](int64_t& c0, int64_t& c1, int64_t at) {
    c0 = at;
    c1 = c0 + rpc < r1 ? c0 + rpc : r1;
    if (c0 < a.nA && c1 > a.nA) c1 = a.nA;
  };
  if (tid == 0) {
    for (int i = 0; i < kCsBuf; ++i) sm100::mbar_init(&cbar[i], 1);
    sm100::fence_mbar_init();
  }
  __syncthreads();
  const int H = kGT / D > 0 ? kGT / D : 1;
  const int c = tid % D, h = tid / D;
  const bool act = D <= kGT ? h < H : true;
  double sa = 0.0, sb = 0.0;
  // thread 0 keeps the ring full: chunk starts are sequential, so it walks them itself
  int64_t next = r0;
  auto issue = [&](int buf) {
    if (next >= r1) return;
    int64_t c0, c1;
    chunk(c0, c1, next);
    const float* src = c0 < a.nA ? a.A + c0 * D : a.B + (c0 - a.nA) * D;
    const uint32_t bytes = static_cast<uint32_t>((c1 - c0) * D * 4);
    sm100::mbar_arrive_expect_tx(&cbar[buf], bytes);
    bulk_g2s(gsm + static_cast<size_t>(buf) * kCsBytes, src, bytes, &cbar[buf]);
    next = c1;
  };
  if (tid == 0)
    for (int i = 0; i < kCsBuf; ++i) issue(i);
  int64_t at = r0;
  for (int k = 0; at < r1; ++k) {
    int64_t c0, c1;
    chunk(c0, c1, at);
    const int buf = k % kCsBuf;
    sm100::mbar_wait(&cbar[buf], (k / kCsBuf) & 1);
    const float* x = reinterpret_cast<const float*>(gsm + static_cast<size_t>(buf) * kCsBytes);
    const int rows = static_cast<int>(c1 - c0);
    double s = 0.0;
    if (act && c < D) {
      // 4 independent chains (fp64 add latency), combined in a fixed order
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
      int rr = h;
      for (; rr + 3 * H < rows; rr += 4 * H) {
#pragma unroll
        for (int u = 0; u < 4; ++u) s4[u] += static_cast<double>(x[(rr + u * H) * D + c]);
      }
      for (; rr < rows; rr += H) s4[0] += static_cast<double>(x[rr * D + c]);
      s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    }
    if (c0 < a.nA)
      sa += s;
    else
      sb += s;
    __syncthreads();  // everyone is done with buf
    if (tid == 0) issue(buf);
    at = c1;
  }
  if (act && c < D) {
    double* cp = a.Cpart + static_cast<int64_t>(q * H + h) * 2 * D;
    cp[c] = sa;
    cp[D + c] = sb;
  }
}

template <bool kVec, int kRep>
__global__ void __launch_bounds__(kGT, 1) gram_kernel(const __grid_constant__ GramArgs a) {
  extern __shared__ __align__(16) uint8_t gsm[];
  if (static_cast<int>(blockIdx.x) >= a.ngram) {
    colsum_role(a, gsm);
    return;
  }
  float* stage = reinterpret_cast<float*>(gsm);                                  // [kGNS][kGMC][32 nslot]
  double* tile = reinterpret_cast<double*>(gsm + sizeof(float) * kGNS * kGStageF);  // [kGNB][kGMC][kGLd]
  int g = 0;
  while (g + 1 < a.ngroups && static_cast<int>(blockIdx.x) >= a.grp[g + 1].cta0) ++g;
  const GramGroup& G = a.grp[g];
  const int r = blockIdx.x - G.cta0;
  const int64_t N = a.nA + a.nB;
  const int64_t p0 = static_cast<int64_t>(r) * G.per;
  const int64_t p1 = p0 + G.per < N ? p0 + G.per : N;
  const int nch = p1 > p0 ? static_cast<int>((p1 - p0 + kGMC - 1) / kGMC) : 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rowf = 32 * G.nslot;  // staged floats per row
  // full[b]: the 4 loader warps wrote buffer b; empty[b]: the 12 MMA warps have its fragments
  // in registers. mbarriers rather than bar.sync: an MMA warp ahead of the others runs on
  // into the next buffers instead of meeting them at every chunk.
  __shared__ uint64_t full[kGNB], empty[kGNB];
  if (tid == 0) {
    for (int i = 0; i < kGNB; ++i) {
      sm100::mbar_init(&full[i], kGT / 32 - kMW);
      sm100::mbar_init(&empty[i], kMW);
    }
    sm100::fence_mbar_init();
  }
  __syncthreads();

  if (warp >= kMW) {
    // ------------------------------------------------------------------ loaders
    const int ct = tid - 32 * kMW;
    const int P = rowf / 4;               // 16-B pieces per staged row (8, 16, 32 or 64)
    const int R = 128 / P;                // rows per pass of the 128 loader threads
    const int NP = kGMC / R;              // pieces per thread per chunk (1, 2, 4 or 8)
    const int c4 = ct % P, r0 = ct / P;   // column piece, first row
    const int sl = c4 >> 3;               // slot
    const int col = 4 * c4;               // column in the staged row
    const int ff = G.fb[sl] * 32 + (col & 31);  // first global feature of the piece
    double s4[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) s4[j] = ff + j < a.D ? a.s[ff + j] : 0.0;
    // warp-uniform (the __any_sync below needs every lane)
    const bool shifted = __any_sync(0xffffffffu, s4[0] != 0.0 || s4[1] != 0.0 || s4[2] != 0.0 || s4[3] != 0.0);
    const uint32_t stage_u32 = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
    const uint64_t Aaddr = reinterpret_cast<uint64_t>(a.A), Baddr = reinterpret_cast<uint64_t>(a.B);
    auto issue = [&](int c) {
      if (c < nch) {
        const uint32_t dst0 = stage_u32 + static_cast<uint32_t>(((c % kGNS) * kGStageF + col) * 4);
        const int64_t q0 = p0 + static_cast<int64_t>(c) * kGMC;
#pragma unroll
        for (int it = 0; it < kSlotsMax; ++it) {
          if (it >= NP) break;
          const int pr = r0 + R * it;
          const int64_t p = q0 + pr;
          const uint64_t rowa = p < a.nA ? Aaddr + static_cast<uint64_t>(p * a.D) * 4
                                         : Baddr + static_cast<uint64_t>((p - a.nA) * a.D) * 4;
          const uint32_t dst = dst0 + static_cast<uint32_t>(pr * rowf * 4);
          if (kVec) {
            const bool ok = p < p1 && ff < a.D;  // D % 4 == 0: all 4 features valid or none
            cp_async16(dst, ok ? reinterpret_cast<const void*>(rowa + static_cast<uint64_t>(ff) * 4) : a.A,
                       ok ? 16 : 0);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const bool ok = p < p1 && ff + j < a.D;
              cp_async4(dst + 4 * j, ok ? reinterpret_cast<const void*>(rowa + static_cast<uint64_t>(ff + j) * 4) : a.A,
                        ok ? 4 : 0);
            }
          }
        }
      }
      cp_commit();
    };
#pragma unroll
    for (int c = 0; c < kGNS - 1; ++c) issue(c);
    for (int c = 0; c < nch; ++c) {
      cp_wait<kGNS - 2>();  // this thread's pieces of chunk c have landed (it reads only those)
      float4 x[kSlotsMax];  // NP <= 8 pieces
      const float* src = stage + (c % kGNS) * kGStageF + col;
#pragma unroll
      for (int it = 0; it < kSlotsMax; ++it)
        if (it < NP) x[it] = *reinterpret_cast<const float4*>(src + (r0 + R * it) * rowf);
      issue(c + kGNS - 1);  // overwrites stage (c - 1) % kGNS, whose values this thread has consumed
      bool special = false;
      if (!shifted) {
#pragma unroll
        for (int it = 0; it < kSlotsMax; ++it) {
          if (it < NP) {
            const unsigned u[4] = {__float_as_uint(x[it].x), __float_as_uint(x[it].y), __float_as_uint(x[it].z),
                                   __float_as_uint(x[it].w)};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const unsigned m = u[j] & 0x7FFFFFFFu;
              special |= (m - 1u < 0x007FFFFFu) | (m >= 0x7F800000u);  // subnormal, inf, nan
            }
          }
        }
      }
      special = __any_sync(0xffffffffu, special);
      const int64_t q0 = p0 + static_cast<int64_t>(c) * kGMC;
      const int b = c % kGNB;
      if (c >= kGNB) sm100::mbar_wait(&empty[b], ((c / kGNB) - 1) & 1);  // MMA warps released buffer b
      double* dst = tile + b * kGMC * kGLd + col;
#pragma unroll
      for (int it = 0; it < kSlotsMax; ++it) {
        if (it >= NP) break;
        const int pr = r0 + R * it;
        const float xs[4] = {x[it].x, x[it].y, x[it].z, x[it].w};
        double v[4];
        if (shifted) {
          // large common offset: x - s_f in fp64 (fp64 pipe); rows past the range stay 0
          const bool in = q0 + pr < p1;
#pragma unroll
          for (int j = 0; j < 4; ++j) v[j] = in ? static_cast<double>(xs[j]) - s4[j] : 0.0;
        } else if (special) {
#pragma unroll
          for (int j = 0; j < 4; ++j) v[j] = static_cast<double>(xs[j]);
        } else {
          // normal numbers and signed zeros: sign | (e + 896) << 20 | mant >> 3, mant << 29
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const unsigned u = __float_as_uint(xs[j]);
            const unsigned hi = (static_cast<unsigned>(static_cast<int>(u) >> 3) & 0x8FFFFFFFu) +
                                ((u & 0x7FFFFFFFu) != 0u ? 0x38000000u : 0u);
            v[j] = __hiloint2double(static_cast<int>(hi), static_cast<int>(u << 29));
          }
        }
        double2* d2 = reinterpret_cast<double2*>(dst + pr * kGLd);
        d2[0] = make_double2(v[0], v[1]);
        d2[1] = make_double2(v[2], v[3]);
      }
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&full[b]);
    }
    cp_wait<0>();
  } else {
    // ------------------------------------------------------------------ DMMA warps
    const bool active = warp < G.ntiles * kRep;
    const int t = active ? warp % G.ntiles : 0;
    const int ri = active ? warp / G.ntiles : 0;  // k-steps ri, ri + kRep, ... of each chunk
    const int sI = G.si[t], sJ = G.sj[t];
    const bool dg = sI == sJ;  // diagonal tile: the 10 8x8 blocks on or above its diagonal, A = B fragments
    const int fr = lane >> 2, fk = lane & 3;
    constexpr int kS = 4 / kRep;  // k-steps per chunk for this warp

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double af[2][4], bf[2][4];
    const int oI = sI * 32 + fr, oJ = sJ * 32 + fr;
    auto ldfrag = [&](const double* row, double (&A_)[4], double (&B_)[4]) {
      if (active) {
#pragma unroll
        for (int i = 0; i < 4; ++i) A_[i] = row[oI + i * 8];
        if (!dg)
#pragma unroll
          for (int j = 0; j < 4; ++j) B_[j] = row[oJ + j * 8];
      }
    };
    auto mma16 = [&](const double (&A_)[4], const double (&B_)[4]) {
      if (active) {
        if (dg) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = i; j < 4; ++j) dmma(acc[i][j], A_[i], A_[j]);
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(acc[i][j], A_[i], B_[j]);
        }
      }
    };
    if constexpr (kS >= 2) {
      // fragments double-buffered in registers: the loads of the warp's next k-step (the next
      // chunk's first one after its FULL barrier) are issued before the 16 DMMAs of this one
      if (nch > 0) {
        sm100::mbar_wait(&full[0], 0);
        ldfrag(tile + (ri * 4 + fk) * kGLd, af[0], bf[0]);
      }
      for (int c = 0; c < nch; ++c) {
        const int b = c % kGNB;
        const double* tb = tile + b * kGMC * kGLd;
#pragma unroll
        for (int u = 0; u < kS; ++u) {
          const int cur = u & 1, nxt = cur ^ 1;
          if (u + 1 < kS) {
            ldfrag(tb + ((ri + kRep * (u + 1)) * 4 + fk) * kGLd, af[nxt], bf[nxt]);
          } else if (c + 1 < nch) {
            const int bn = (c + 1) % kGNB;
            sm100::mbar_wait(&full[bn], ((c + 1) / kGNB) & 1);
            ldfrag(tile + bn * kGMC * kGLd + (ri * 4 + fk) * kGLd, af[nxt], bf[nxt]);
          }
          mma16(af[cur], bf[cur]);
        }
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&empty[b]);
      }
    } else {
      for (int c = 0; c < nch; ++c) {
        const int b = c % kGNB;
        sm100::mbar_wait(&full[b], (c / kGNB) & 1);
        ldfrag(tile + b * kGMC * kGLd + (ri * 4 + fk) * kGLd, af[0], bf[0]);
        mma16(af[0], bf[0]);
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&empty[b]);
      }
    }
    double* out = a.Gpart + (static_cast<int64_t>(blockIdx.x) * kMW + warp) * 1024;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        *reinterpret_cast<double2*>(out + (i * 8 + fr) * 32 + j * 8 + 2 * fk) =
            make_double2(acc[i][j][0], acc[i][j][1]);
  }
}

// G (full symmetric D x D) and S_A, S_B from the partials, in a fixed order (bit-identical
// runs): CTA = 32 consecutive elements x of one (group, tile); warp w sums the partials of
// ranges r = w, w + 8, ... (and every k-step replica) for its lane's element, then the 8 warp
// sums combine in warp order. The sums of S_X run on CTA 0..ceil(D / 256) - 1 likewise.
__global__ void __launch_bounds__(256) gram_reduce_kernel(const __grid_constant__ GramArgs a, double* __restrict__ Gout,
                                                          double* __restrict__ SA, double* __restrict__ SB) {
  const int D = a.D;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ double part[2][8][32];
  const int nblk = a.ngroups * kMW * 32;  // element blocks of 32
  if (static_cast<int>(blockIdx.x) < nblk) {
    const int g = blockIdx.x / (kMW * 32), t = (blockIdx.x / 32) % kMW;
    const int x = (blockIdx.x % 32) * 32 + lane;
    const GramGroup& G = a.grp[g];
    if (t >= G.ntiles) return;  // uniform per CTA
    double acc = 0.0;
    for (int r = warp; r < G.rpg; r += 8)
      for (int q = 0; q < G.rep; ++q)
        acc += a.Gpart[(static_cast<int64_t>(G.cta0 + r) * kMW + q * G.ntiles + t) * 1024 + x];
    part[0][warp][lane] = acc;
    __syncthreads();
    if (warp == 0) {
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) v += part[0][w][lane];
      const int I = G.fb[G.si[t]], J = G.fb[G.sj[t]];
      const int ii = x / 32, jj = x % 32;
      const int i = I * 32 + ii, j = J * 32 + jj;
      if (!(I == J && ii > jj) && i < D && j < D) {  // diagonal tiles: upper triangle is authoritative
        Gout[static_cast<int64_t>(i) * D + j] = v;
        Gout[static_cast<int64_t>(j) * D + i] = v;
      }
    }
    return;
  }
  // S_X = sum_{x in X} x - n_X s (colsum_kernel partials about the origin)
  const int f0 = (blockIdx.x - nblk) * 32 + lane;
  const bool fv = f0 < D;
  double sa = 0.0, sb = 0.0;
  if (fv)
    for (int q = warp; q < a.cs_blocks; q += 8) {
      sa += a.Cpart[(static_cast<int64_t>(q) * 2 + 0) * D + f0];
      sb += a.Cpart[(static_cast<int64_t>(q) * 2 + 1) * D + f0];
    }
  part[0][warp][lane] = sa;
  part[1][warp][lane] = sb;
  __syncthreads();
  if (warp == 0 && fv) {
    double va = 0.0, vb = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      va += part[0][w][lane];
      vb += part[1][w][lane];
    }
    SA[f0] = va - static_cast<double>(a.nA) * a.s[f0];
    SB[f0] = vb - static_cast<double>(a.nB) * a.s[f0];
  }
}

// Column sums of A and of B about the origin, fp64: CTA q takes a contiguous range of the
// rows of A u B; thread (row lane, column piece) adds every L-th row of the range; the L row
// lanes combine in shared memory in a fixed order -> Cpart[q][set][f]. HBM-bound.
template <int W>
__global__ void __launch_bounds__(256) colsum_kernel(const float* __restrict__ A, int64_t nA,
                                                     const float* __restrict__ B, int64_t nB, int D, int64_t per,
                                                     double* __restrict__ Cpart) {
  const int P = (D + W - 1) / W;          // W-feature pieces per row
  const int L = P >= 256 ? 1 : 256 / P;   // row lanes (1: the CTA loops over blocks of 256 pieces)
  const int64_t N = nA + nB;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * per;
  const int64_t r1 = r0 + per < N ? r0 + per : N;
  __shared__ double red[2][1024];
  for (int pcb = 0; pcb < (L == 1 ? P : 1); pcb += 256) {
    const int lr = L == 1 ? 0 : static_cast<int>(threadIdx.x) / P;
    const int pc = L == 1 ? pcb + static_cast<int>(threadIdx.x) : static_cast<int>(threadIdx.x) % P;
    const bool act = pc < P && lr < L;
    double sa[W], sb[W];
#pragma unroll
    for (int j = 0; j < W; ++j) sa[j] = sb[j] = 0.0;
    if (act) {
      const int f0 = pc * W;
      // 4 rows per step, loads issued before the adds (HBM latency)
      for (int64_t r = r0 + lr; r < r1; r += 4 * static_cast<int64_t>(L)) {
        float v[4][W];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t rr = r + static_cast<int64_t>(u) * L;
          const bool ok = rr < r1;
          const float* row = rr < nA ? A + rr * D : B + (rr - nA) * D;
          if constexpr (W == 4) {
            const float4 q = ok ? __ldg(reinterpret_cast<const float4*>(row + f0)) : make_float4(0.f, 0.f, 0.f, 0.f);
            v[u][0] = q.x;
            v[u][1] = q.y;
            v[u][2] = q.z;
            v[u][3] = q.w;
          } else {
            v[u][0] = ok ? __ldg(row + f0) : 0.0f;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool inA = r + static_cast<int64_t>(u) * L < nA;
#pragma unroll
          for (int j = 0; j < W; ++j) {
            if (inA)
              sa[j] += static_cast<double>(v[u][j]);
            else
              sb[j] += static_cast<double>(v[u][j]);
          }
        }
      }
    }
    if (L == 1) {
      if (act)
#pragma unroll
        for (int j = 0; j < W; ++j)
          if (pc * W + j < D) {
            Cpart[(static_cast<int64_t>(blockIdx.x) * 2 + 0) * D + pc * W + j] = sa[j];
            Cpart[(static_cast<int64_t>(blockIdx.x) * 2 + 1) * D + pc * W + j] = sb[j];
          }
      continue;
    }
    for (int l = 0; l < L; ++l) {  // fixed order over the row lanes
      if (act && lr == l)
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const int f = pc * W + j;
          if (f < D) {
            red[0][f] = (l == 0 ? 0.0 : red[0][f]) + sa[j];
            red[1][f] = (l == 0 ? 0.0 : red[1][f]) + sb[j];
          }
        }
      __syncthreads();
    }
    for (int f = threadIdx.x; f < D; f += blockDim.x) {
      Cpart[(static_cast<int64_t>(blockIdx.x) * 2 + 0) * D + f] = red[0][f];
      Cpart[(static_cast<int64_t>(blockIdx.x) * 2 + 1) * D + f] = red[1][f];
    }
  }
}

}  // namespace

// Host-side grouping of the upper-triangle 32x32 tiles (see the file header).
bool plan_gram(int64_t nA, int64_t nB, int D, int num_sms, GramPlan& p) {
  const int nb = (D + 31) / 32;
  if (nb > kGramMaxFb) return false;
  p = GramPlan{};
  p.ngroups = 0;
  // one group: the given tiles over the given feature blocks (slot = position in fbs)
  auto add_group = [&](const int* fbs, int nfb, const int (*tiles)[2], int nt) -> bool {
    if (p.ngroups >= kGramMaxGroups || nt < 1 || nt > kMW || nfb > kSlotsMax) return false;
    GramGroup& G = p.grp[p.ngroups++];
    G = GramGroup{};
    G.nslot = 1;
    while (G.nslot < nfb) G.nslot = static_cast<unsigned char>(G.nslot * 2);
    for (int s = 0; s < kSlotsMax; ++s) G.fb[s] = static_cast<unsigned char>(s < nfb ? fbs[s] : kGramMaxFb - 1);
    G.nfb = static_cast<unsigned char>(nfb);
    for (int t = 0; t < nt; ++t) {
      for (int q = 0; q < 2; ++q) {
        int s = 0;
        while (s < nfb && fbs[s] != tiles[t][q]) ++s;
        if (s == nfb) return false;
        (q == 0 ? G.si : G.sj)[t] = static_cast<unsigned char>(s);
      }
    }
    G.ntiles = static_cast<unsigned char>(nt);
    G.rep = static_cast<unsigned char>(nt * 4 <= kMW ? 4 : nt * 2 <= kMW ? 2 : 1);
    return true;
  };
  if (nb <= kSlotsMax) {
    // every group stages all nb blocks; the T = nb (nb + 1) / 2 tiles split evenly over the
    // groups, the nb diagonal tiles (10 of 16 DMMAs per k-step) dealt out four per group first
    // and placed on warps 0-3 (one per SM sub-partition, whose DMMA pipe the warps share)
    int fbs[kSlotsMax], dl[kSlotsMax][2], ol[64][2], nd = 0, no = 0;
    for (int s = 0; s < nb; ++s) fbs[s] = s;
    for (int i = 0; i < nb; ++i)
      for (int j = i; j < nb; ++j) {
        int(*l)[2] = i == j ? dl : ol;
        int& c = i == j ? nd : no;
        l[c][0] = i;
        l[c][1] = j;
        ++c;
      }
    const int T = nd + no;
    const int ng = (T + kMW - 1) / kMW;
    int di = 0, oi = 0;
    for (int g = 0; g < ng; ++g) {
      const int sz = T * (g + 1) / ng - T * g / ng;
      int tl[kMW][2], n = 0;
      while (n < sz && n < 4 && di < nd) {
        tl[n][0] = dl[di][0];
        tl[n][1] = dl[di][1];
        ++n, ++di;
      }
      while (n < sz && oi < no) {
        tl[n][0] = ol[oi][0];
        tl[n][1] = ol[oi][1];
        ++n, ++oi;
      }
      while (n < sz && di < nd) {
        tl[n][0] = dl[di][0];
        tl[n][1] = dl[di][1];
        ++n, ++di;
      }
      if (!add_group(fbs, nb, tl, n)) return false;
    }
  } else {
    // 4x4 squares of blocks on or above the diagonal: <= 8 blocks, <= 16 tiles -> 1 or 2 groups
    for (int a = 0; a < nb; a += 4)
      for (int b = a; b < nb; b += 4) {
        int fbs[kSlotsMax], nfb = 0, tl[16][2], T = 0;
        for (int i = a; i < a + 4 && i < nb; ++i) fbs[nfb++] = i;
        if (b != a)
          for (int j = b; j < b + 4 && j < nb; ++j) fbs[nfb++] = j;
        for (int pass = 0; pass < 2; ++pass)  // diagonal tiles first (warps 0-3)
          for (int i = a; i < a + 4 && i < nb; ++i)
            for (int j = b; j < b + 4 && j < nb; ++j)
              if (i <= j && (i == j) == (pass == 0)) {
                tl[T][0] = i;
                tl[T][1] = j;
                ++T;
              }
        const int ng = (T + kMW - 1) / kMW;
        for (int g = 0; g < ng; ++g) {
          const int t0 = T * g / ng, t1 = T * (g + 1) / ng;
          if (!add_group(fbs, nfb, tl + t0, t1 - t0)) return false;
        }
      }
  }
  // the kernel instantiates kRep per launch: every group must share one
  for (int g = 1; g < p.ngroups; ++g)
    if (p.grp[g].rep != p.grp[0].rep) {
      unsigned char m = p.grp[0].rep;
      for (int q = 0; q < p.ngroups; ++q) m = p.grp[q].rep < m ? p.grp[q].rep : m;
      for (int q = 0; q < p.ngroups; ++q) p.grp[q].rep = m;
      break;
    }
  // Cost model: warp w runs on SM sub-partition w % 4 and issues 16 (10 on a diagonal tile)
  // DMMAs per k-step; a group's CTA time per point is set by its busiest sub-partition. The
  // one-wave CTA budget is split over the groups in proportion to that load (largest
  // remaining time per range first), and every group cuts A u B into its own rpg ranges.
  const int64_t N = nA + nB;
  const int64_t chunks = N > 0 ? (N + kGMC - 1) / kGMC : 1;
  // Column sums in the same launch on cs_ctas SMs of their own when the Gram is slow enough per
  // byte to hide them: a column-sum SM streams ~66 GB/s (measured), so 7 of them match the
  // DMMA-bound Gram on the other 141 at D = 256 (cfg5 moments 9.27 -> 8.91 ms; 8: 9.11, 6: 10.19)
  // but not at D = 128, where the Gram costs half as much per byte (cfg3 0.80 -> 1.36 ms). D >= 224,
  // D % 4 == 0, enough rows; option k1_cs_sms overrides the count (0 = the colsum_kernel pass).
  p.cs_ctas = 0;
  {
    int cs = D >= 224 ? 7 : 0;
    if (opt(OPT_K1_CS_SMS) >= 0) cs = static_cast<int>(opt(OPT_K1_CS_SMS));
    const int sms = num_sms > 0 ? num_sms : 148;
    if (cs > 0 && D % 4 == 0 && D <= kGT && N >= static_cast<int64_t>(64) * sms && cs < sms / 2) p.cs_ctas = cs;
  }
  const int budget = (num_sms > 0 ? num_sms : 148) - p.cs_ctas;
  for (int g = 0; g < p.ngroups; ++g) {
    GramGroup& G = p.grp[g];
    int sp[4] = {0, 0, 0, 0};
    for (int w = 0; w < G.ntiles * G.rep && w < kMW; ++w) {
      const int t = w % G.ntiles;
      sp[w % 4] += G.si[t] == G.sj[t] ? 10 : 16;
    }
    G.load = sp[0];
    for (int q = 1; q < 4; ++q) G.load = sp[q] > G.load ? sp[q] : G.load;
    if (G.load < 1) G.load = 1;
    G.rpg = 1;
  }
  // beta: a per-point cost outside the DMMA pipe, in DMMA units (dev A/B: option k1_beta_milli)
  double beta = 0.0;
  if (opt(OPT_K1_BETA_MILLI) >= 0) beta = 1e-3 * static_cast<double>(opt(OPT_K1_BETA_MILLI));
  for (int used = p.ngroups; used < budget; ++used) {
    int best = -1;
    double bt = 0.0;
    for (int g = 0; g < p.ngroups; ++g) {
      const double t = (p.grp[g].load + beta) / p.grp[g].rpg;
      if (p.grp[g].rpg < chunks && t > bt) {
        bt = t;
        best = g;
      }
    }
    if (best < 0) break;
    ++p.grp[best].rpg;
  }
  p.nctas = 0;
  for (int g = 0; g < p.ngroups; ++g) {
    GramGroup& G = p.grp[g];
    G.per = ((N + G.rpg - 1) / G.rpg + kGMC - 1) / kGMC * kGMC;
    G.cta0 = p.nctas;
    p.nctas += G.rpg;
  }
  p.gpart_doubles = static_cast<int64_t>(p.nctas) * kMW * 1024;
  if (p.cs_ctas > 0) {
    const int H = kGT / D > 0 ? kGT / D : 1;
    p.cs_per = (N + p.cs_ctas - 1) / p.cs_ctas;
    p.cs_blocks = p.cs_ctas * H;
  } else {
    p.cs_blocks = 4 * (num_sms > 0 ? num_sms : 148);
    if (p.cs_blocks > N) p.cs_blocks = static_cast<int>(N > 0 ? N : 1);
    p.cs_per = (N + p.cs_blocks - 1) / p.cs_blocks;
  }
  p.spart_doubles = static_cast<int64_t>(p.cs_blocks) * 2 * D;
  return true;
}

cudaError_t launch_gram(const GramPlan& p, const float* A, int64_t nA, const float* B, int64_t nB, int D,
                        const double* s, double* Gpart, double* Spart, double* Gout, double* SA, double* SB,
                        cudaStream_t st) {
  GramArgs a{};
  a.A = A;
  a.B = B;
  a.nA = nA;
  a.nB = nB;
  a.D = D;
  a.s = s;
  a.ngroups = p.ngroups;
  a.Gpart = Gpart;
  for (int g = 0; g < p.ngroups; ++g) a.grp[g] = p.grp[g];
  a.Cpart = Spart;
  a.cs_blocks = p.cs_blocks;
  a.ngram = p.nctas;
  a.cs_ctas = p.cs_ctas;
  a.cs_per = p.cs_per;
  const bool vec = (D % 4) == 0;
  const int rep = p.grp[0].rep;
  auto kern = vec ? (rep == 4 ? gram_kernel<true, 4> : rep == 2 ? gram_kernel<true, 2> : gram_kernel<true, 1>)
                  : (rep == 4 ? gram_kernel<false, 4> : rep == 2 ? gram_kernel<false, 2> : gram_kernel<false, 1>);
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kGSmem))) !=
      cudaSuccess)
    return e;
  if (p.cs_ctas == 0) {
    count_launch();
    if (vec)
      colsum_kernel<4><<<p.cs_blocks, 256, 0, st>>>(A, nA, B, nB, D, p.cs_per, Spart);
    else
      colsum_kernel<1><<<p.cs_blocks, 256, 0, st>>>(A, nA, B, nB, D, p.cs_per, Spart);
  }
  count_launch();
  kern<<<p.nctas + p.cs_ctas, kGT, kGSmem, st>>>(a);
  count_launch();
  gram_reduce_kernel<<<p.ngroups * kMW * 32 + (D + 31) / 32, 256, 0, st>>>(a, Gout, SA, SB);
  return cudaGetLastError();
}

}  // namespace prohd
