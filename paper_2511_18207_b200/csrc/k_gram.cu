// k_gram.cu — K1 main pass: the fp64 Gram G = sum_{p in A u B} (p - s)(p - s)^T and the
// column sums S_A, S_B on the fp64 tensor pipe (DMMA), warp-specialised.
//
// PAPER.md Alg. 2 lines 1-2: the principal directions are eigenvectors of the
// covariance of the stacked set [X; Y]; K1 (k_moments.cu) turns (S_A, S_B, G) into the
// centroids (Alg. 1 line 1) and C = G/N - (mu - s)(mu - s)^T.
//
// Work decomposition. The upper triangle of G is cut into 32x32 warp tiles (I <= J over
// 32-feature blocks) and the tiles into GROUPS of <= 4 that together need <= 4 feature
// blocks (<= 128 features): every off-diagonal 64x64 block is one group of 4 tiles, and
// the 3 upper tiles of consecutive diagonal 64x64 blocks are packed 4 at a time. At
// D = 256 that is 36 tiles in 9 full groups, so no warp idles. CTA = (point range r,
// group g), blockIdx = r * ngroups + g: the ngroups CTAs reading the same rows are
// adjacent in launch order, run concurrently, and share the rows through L2.
//
// CTA = 8 warps, 2 CTAs per SM:
//   warps 4-7 (loaders): cp.async the 128 needed features of the next kMC points into an
//            fp32 staging ring (NS stages, 16-B pieces, zero fill past the range), then
//            convert each element once to fp64 (x - s_f) into an fp64 tile ring (NB
//            buffers) and accumulate the column sums of the feature blocks this group owns
//            (the group holding the diagonal tile (f, f)). The conversion runs on the
//            integer pipe and the subtraction only where s_f != 0: the shift kernel keeps
//            s = 0 unless the data's mean offset is large against its spread, so in the
//            common case the loaders put no work on the fp64 pipe that the DMMAs share
//            (products of fp32 values are exact in fp64 either way).
//   warps 0-3 (MMA): warp w owns tile w of the group; per 4-point k-step it loads 4 A and
//            4 B fragments (8 LDS.64) and issues 16 DMMA.8x8x4 into a 32x32 fp64 register
//            accumulator (64 regs).
// Buffer hand-off with named barriers: FULL[b] (loaders arrive, MMA warps sync) and
// EMPTY[b] (MMA warps arrive, loaders sync). Every CTA writes its own partial slot;
// gram_reduce_kernel sums the slots in a fixed order (deterministic, bit-identical runs).
#include "internal.cuh"
#include "prohd_kernels.cuh"

namespace prohd {
namespace {

constexpr int kGT = 256;       // threads per CTA
constexpr int kGMC = 16;       // points per chunk (= 4 DMMA k-steps)
constexpr int kGNS = 4;        // fp32 staging stages
constexpr int kGNB = 4;        // fp64 tile buffers
constexpr int kGLd = 132;      // fp64 row stride: 128 features + 4 (conflict-free fragment loads)
constexpr int kGStageF = kGMC * 128;                   // floats per staging stage
constexpr size_t kGSmem = sizeof(float) * kGNS * kGStageF + sizeof(double) * kGNB * kGMC * kGLd;

struct GramArgs {
  const float* A;
  const float* B;
  int64_t nA, nB;
  int D;
  const double* s;
  int ngroups, rpg;
  int64_t per;      // points per range (multiple of kGMC)
  double* Gpart;    // [cta][4 tiles][32][32]
  double* Spart;    // [cta][4 slots][2 sets][32]
  short owner[2 * kGramMaxFb];  // per 32-feature block: (group, slot) holding its column sums
  GramGroup grp[kGramMaxGroups];
};

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
// fp32 -> fp64 on the integer pipe (the fp64 pipe is shared with the DMMAs): exact for
// normal numbers and signed zeros; f32_special() flags the rest (subnormal, inf, nan).
__device__ __forceinline__ bool f32_special(float x) {
  const unsigned u = __float_as_uint(x);
  const unsigned e = (u >> 23) & 0xFFu;
  return e == 0xFFu || (e == 0u && (u & 0x7FFFFFu) != 0u);
}
__device__ __forceinline__ double f32_to_f64_normal(float x) {
  const unsigned u = __float_as_uint(x);
  const unsigned e = (u >> 23) & 0xFFu;
  const unsigned sign = u & 0x80000000u, mant = u & 0x7FFFFFu;
  const unsigned hi = e == 0u ? sign : (sign | ((e + 896u) << 20) | (mant >> 3));
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(mant << 29));
}
__device__ __forceinline__ double f32_to_f64(float x) {
  return f32_special(x) ? static_cast<double>(x) : f32_to_f64_normal(x);
}
// (s, c) += x with Knuth's TwoSum: s + c tracks the running sum, c collects the exact
// rounding error of every addition (fp32 pipe).
__device__ __forceinline__ void two_sum_acc(float& s, float& c, float x) {
  const float t = s + x;
  const float bb = t - s;
  const float e = (s - (t - bb)) + (x - bb);
  s = t;
  c += e;
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
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

// barrier ids: FULL[b] = 1 + b, EMPTY[b] = 1 + kGNB + b, loaders only = 1 + 2 kGNB
template <bool kVec>
__global__ void __launch_bounds__(kGT, 2) gram_kernel(const __grid_constant__ GramArgs a) {
  extern __shared__ __align__(16) uint8_t gsm[];
  float* stage = reinterpret_cast<float*>(gsm);                                  // [kGNS][kGMC][128]
  double* tile = reinterpret_cast<double*>(gsm + sizeof(float) * kGNS * kGStageF);  // [kGNB][kGMC][kGLd]
  const int g = blockIdx.x % a.ngroups;
  const int r = blockIdx.x / a.ngroups;
  const GramGroup& G = a.grp[g];
  const int64_t N = a.nA + a.nB;
  const int64_t p0 = static_cast<int64_t>(r) * a.per;
  const int64_t p1 = p0 + a.per < N ? p0 + a.per : N;
  const int nch = p1 > p0 ? static_cast<int>((p1 - p0 + kGMC - 1) / kGMC) : 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp >= 4 && kVec) {
    // ------------------------------------------------------------------ loaders, D % 4 == 0
    // Thread (lw, lane) owns 16-B piece (row lw + 4 it, features fb[sl] * 32 + 4 sub .. + 3)
    // of every chunk: it issues that piece's cp.async, waits for its own copies only (no
    // loader barrier), converts the 4 values and writes them to the fp64 tile as 2 x 16 B.
    // A warp covers one 512-B row per it: conflict-free LDS.128 / STS.128.
    const int ct = tid - 128, lw = ct >> 5;
    const int sl = lane >> 3, sub = lane & 7;
    const int ff = sl < G.nfb ? G.fb[sl] * 32 + sub * 4 : a.D;
    const bool fv = ff < a.D;  // D % 4 == 0: the 4 features are all valid or all absent
    const int col = sl * 32 + sub * 4;
    const bool own = fv && G.own[sl];
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
    if (fv)
#pragma unroll
      for (int j = 0; j < 4; ++j) s4[j] = a.s[ff + j];
    // warp-uniform (the __any_sync below needs every lane): lanes without features convert zeros
    const bool shifted = __any_sync(0xffffffffu, s4[0] != 0.0 || s4[1] != 0.0 || s4[2] != 0.0 || s4[3] != 0.0);
    double sA[4] = {0.0, 0.0, 0.0, 0.0}, sB[4] = {0.0, 0.0, 0.0, 0.0};
    const uint32_t stage_u32 = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
    const uint64_t Aaddr = reinterpret_cast<uint64_t>(a.A), Baddr = reinterpret_cast<uint64_t>(a.B);
    auto issue = [&](int c) {
      if (c < nch) {
        const uint32_t dst0 = stage_u32 + static_cast<uint32_t>(((c % kGNS) * kGStageF + col) * 4);
        const int64_t q0 = p0 + static_cast<int64_t>(c) * kGMC;
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int pr = lw + 4 * it;
          const int64_t p = q0 + pr;
          const bool ok = fv && p < p1;
          const uint64_t src = p < a.nA ? Aaddr + static_cast<uint64_t>(p * a.D + ff) * 4
                                        : Baddr + static_cast<uint64_t>((p - a.nA) * a.D + ff) * 4;
          cp_async16(dst0 + static_cast<uint32_t>(pr * 128 * 4), ok ? reinterpret_cast<const void*>(src) : a.A,
                     ok ? 16 : 0);
        }
      }
      cp_commit();
    };
#pragma unroll
    for (int c = 0; c < kGNS - 1; ++c) issue(c);
    for (int c = 0; c < nch; ++c) {
      cp_wait<kGNS - 2>();  // this thread's pieces of chunk c have landed (it reads only those)
      float4 x[4];
      const float* src = stage + (c % kGNS) * kGStageF + col;
#pragma unroll
      for (int it = 0; it < 4; ++it) x[it] = *reinterpret_cast<const float4*>(src + (lw + 4 * it) * 128);
      issue(c + kGNS - 1);  // overwrites stage (c - 1) % kGNS, whose values this thread has consumed
      const int64_t q0 = p0 + static_cast<int64_t>(c) * kGMC;
      double v[4][4];
      if (!shifted) {
        // integer-pipe fp32 -> fp64 for normals and signed zeros; a warp-uniform F2F fallback
        // if any of the warp's values is subnormal, inf or nan
        bool special = false;
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const float xs[4] = {x[it].x, x[it].y, x[it].z, x[it].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const unsigned u = __float_as_uint(xs[j]);
            const unsigned m = u & 0x7FFFFFFFu;
            special |= (m - 1u < 0x007FFFFFu) | (m >= 0x7F800000u);
            const unsigned hi = ((static_cast<unsigned>(static_cast<int>(u) >> 3) & 0x8FFFFFFFu)) +
                                (m != 0u ? 0x38000000u : 0u);
            v[it][j] = __hiloint2double(static_cast<int>(hi), static_cast<int>(u << 29));
          }
        }
        if (__any_sync(0xffffffffu, special)) {
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            v[it][0] = static_cast<double>(x[it].x);
            v[it][1] = static_cast<double>(x[it].y);
            v[it][2] = static_cast<double>(x[it].z);
            v[it][3] = static_cast<double>(x[it].w);
          }
        }
      } else {
        // large common offset: x - s_f in fp64 (fp64 pipe); rows past the range stay 0
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const bool in = q0 + lw + 4 * it < p1;
          v[it][0] = in ? static_cast<double>(x[it].x) - s4[0] : 0.0;
          v[it][1] = in ? static_cast<double>(x[it].y) - s4[1] : 0.0;
          v[it][2] = in ? static_cast<double>(x[it].z) - s4[2] : 0.0;
          v[it][3] = in ? static_cast<double>(x[it].w) - s4[3] : 0.0;
        }
      }
      const int b = c % kGNB;
      if (c >= kGNB) named_sync(1 + kGNB + b, kGT);  // MMA warps released buffer b
      double* dst = tile + b * kGMC * kGLd + col;
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        double2* d2 = reinterpret_cast<double2*>(dst + (lw + 4 * it) * kGLd);
        d2[0] = make_double2(v[it][0], v[it][1]);
        d2[1] = make_double2(v[it][2], v[it][3]);
      }
      named_arrive(1 + b, kGT);
      if (own) {
        // column sums of the owned block (rows past the range are 0)
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          if (q0 + lw + 4 * it < a.nA) {
#pragma unroll
            for (int j = 0; j < 4; ++j) sA[j] += v[it][j];
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) sB[j] += v[it][j];
          }
        }
      }
    }
    for (int c = (nch > kGNB ? nch - kGNB : 0); c < nch; ++c) named_sync(1 + kGNB + (c % kGNB), kGT);
    cp_wait<0>();
    // combine the 4 loader warps' column sums in a fixed order through the (now idle) staging ring
    named_sync(1 + 2 * kGNB, 128);
    double* red = reinterpret_cast<double*>(stage);  // [lw][slot][32][2]
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      red[((lw * 4 + sl) * 32 + sub * 4 + j) * 2 + 0] = sA[j];
      red[((lw * 4 + sl) * 32 + sub * 4 + j) * 2 + 1] = sB[j];
    }
    named_sync(1 + 2 * kGNB, 128);
    {
      const int slot = ct >> 5;
      double ra = 0.0, rb = 0.0;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        ra += red[((w * 4 + slot) * 32 + lane) * 2 + 0];
        rb += red[((w * 4 + slot) * 32 + lane) * 2 + 1];
      }
      double* sp = a.Spart + (static_cast<int64_t>(blockIdx.x) * 4 + slot) * 64;
      sp[lane] = ra;
      sp[32 + lane] = rb;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ loaders, D % 4 != 0
    const int ct = tid - 128;
    const int slot = ct >> 5;
    const int f = slot < G.nfb ? G.fb[slot] * 32 + lane : a.D;
    const bool fvalid = f < a.D;
    const double sf = fvalid ? a.s[f] : 0.0;  // 0 unless the shift kernel kept a shift (large offsets)
    const bool shifted = sf != 0.0;
    const bool own = fvalid && G.own[slot];
    double ssA = 0.0, ssB = 0.0;
    const uint32_t stage_u32 = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
    auto issue = [&](int c) {  // chunk c into stage c % kGNS (one commit group per chunk)
      if (c < nch) {
        const uint32_t dst0 = stage_u32 + static_cast<uint32_t>((c % kGNS) * kGStageF * 4);
        const int64_t q0 = p0 + static_cast<int64_t>(c) * kGMC;
        if (kVec) {
          // kGMC rows x 32 pieces of 16 B (4 slots x 8), kGMC * 32 / 128 pieces per thread
#pragma unroll
          for (int it = 0; it < kGMC * 32 / 128; ++it) {
            const int q = ct + 128 * it;
            const int pr = q >> 5, sl = (q >> 3) & 3, sub = q & 7;
            const int64_t p = q0 + pr;
            const int ff = sl < G.nfb ? G.fb[sl] * 32 + sub * 4 : a.D;
            const bool ok = p < p1 && ff < a.D;
            const float* src = p < a.nA ? a.A + p * a.D : a.B + (p - a.nA) * a.D;
            cp_async16(dst0 + static_cast<uint32_t>((pr * 128 + sl * 32 + sub * 4) * 4), ok ? src + ff : a.A,
                       ok ? 16 : 0);
          }
        } else {
          // D % 4 != 0: 4-byte pieces, this thread's own feature column
#pragma unroll 4
          for (int pr = 0; pr < kGMC; ++pr) {
            const int64_t p = q0 + pr;
            const bool ok = p < p1 && fvalid;
            const float* src = p < a.nA ? a.A + p * a.D : a.B + (p - a.nA) * a.D;
            cp_async4(dst0 + static_cast<uint32_t>((pr * 128 + ct) * 4), ok ? src + f : a.A, ok ? 4 : 0);
          }
        }
      }
      cp_commit();
    };
#pragma unroll
    for (int c = 0; c < kGNS - 1; ++c) issue(c);
    for (int c = 0; c < nch; ++c) {
      cp_wait<kGNS - 2>();       // this thread's pieces of chunk c have landed
      named_sync(1 + 2 * kGNB, 128);  // ... and everyone's; stage (c-1) % kGNS is free again
      issue(c + kGNS - 1);
      const int b = c % kGNB;
      if (c >= kGNB) named_sync(1 + kGNB + b, kGT);  // MMA warps released buffer b
      const float* src = stage + (c % kGNS) * kGStageF + ct;
      double* dst = tile + b * kGMC * kGLd + ct;
      const int64_t q0 = p0 + static_cast<int64_t>(c) * kGMC;
      if (!shifted) {
        // common case: raw values (zero-filled past the range and for absent features);
        // all kGMC shared loads are issued first, then converted on the integer pipe
        // (a warp-uniform F2F fallback if any value is subnormal, inf or nan); the owned
        // column sums use an error-free fp32 TwoSum per chunk, then 4 DADDs.
        float x[kGMC];
#pragma unroll
        for (int pr = 0; pr < kGMC; ++pr) x[pr] = src[pr * 128];
        bool special = false;
#pragma unroll
        for (int pr = 0; pr < kGMC; ++pr) special |= f32_special(x[pr]);
        if (__any_sync(0xffffffffu, special)) {
#pragma unroll
          for (int pr = 0; pr < kGMC; ++pr) dst[pr * kGLd] = static_cast<double>(x[pr]);
        } else {
#pragma unroll
          for (int pr = 0; pr < kGMC; ++pr) dst[pr * kGLd] = f32_to_f64_normal(x[pr]);
        }
        if (own) {
          float sA = 0.0f, cA = 0.0f, sB = 0.0f, cB = 0.0f;
          if (q0 + kGMC <= a.nA) {
#pragma unroll
            for (int pr = 0; pr < kGMC; ++pr) two_sum_acc(sA, cA, x[pr]);
          } else if (q0 >= a.nA) {
#pragma unroll
            for (int pr = 0; pr < kGMC; ++pr) two_sum_acc(sB, cB, x[pr]);
          } else {
#pragma unroll
            for (int pr = 0; pr < kGMC; ++pr) {
              if (q0 + pr < a.nA)
                two_sum_acc(sA, cA, x[pr]);
              else
                two_sum_acc(sB, cB, x[pr]);
            }
          }
          ssA += static_cast<double>(sA) + static_cast<double>(cA);
          ssB += static_cast<double>(sB) + static_cast<double>(cB);
        }
      } else {
        // large common offset: x - s_f in fp64 (fp64 pipe)
#pragma unroll
        for (int pr = 0; pr < kGMC; ++pr) {
          const int64_t p = q0 + pr;
          double v = f32_to_f64(src[pr * 128]) - sf;
          if (p >= p1) v = 0.0;
          dst[pr * kGLd] = v;
          if (own) {
            if (p < a.nA)
              ssA += v;
            else
              ssB += v;
          }
        }
      }
      named_arrive(1 + b, kGT);
    }
    // pair the MMA warps' last EMPTY arrivals (chunks nch - kGNB .. nch - 1) so no barrier is left open
    for (int c = (nch > kGNB ? nch - kGNB : 0); c < nch; ++c) named_sync(1 + kGNB + (c % kGNB), kGT);
    cp_wait<0>();
    if (slot < 4) {
      double* sp = a.Spart + (static_cast<int64_t>(blockIdx.x) * 4 + slot) * 64;
      sp[lane] = ssA;
      sp[32 + lane] = ssB;
    }
  } else {
    // ------------------------------------------------------------------ DMMA warps
    const bool active = warp < G.ntiles;
    const int sI = active ? G.si[warp] : 0, sJ = active ? G.sj[warp] : 0;
    const int fr = lane >> 2, fk = lane & 3;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    // fragments double-buffered in registers: the loads of k-step k + 1 (the next chunk's first
    // k-step after its FULL barrier) are issued before the 16 DMMAs of k-step k
    double af[2][4], bf[2][4];
    const int oI = sI * 32 + fr, oJ = sJ * 32 + fr;
    auto ldfrag = [&](const double* row, double (&A_)[4], double (&B_)[4]) {
      if (active) {
#pragma unroll
        for (int i = 0; i < 4; ++i) A_[i] = row[oI + i * 8];
#pragma unroll
        for (int j = 0; j < 4; ++j) B_[j] = row[oJ + j * 8];
      }
    };
    if (nch > 0) {
      named_sync(1, kGT);
      ldfrag(tile + fk * kGLd, af[0], bf[0]);
    }
    for (int c = 0; c < nch; ++c) {
      const int b = c % kGNB;
      const double* t = tile + b * kGMC * kGLd;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int cur = ks & 1, nxt = cur ^ 1;
        if (ks < 3) {
          ldfrag(t + ((ks + 1) * 4 + fk) * kGLd, af[nxt], bf[nxt]);
        } else if (c + 1 < nch) {
          const int bn = (c + 1) % kGNB;
          named_sync(1 + bn, kGT);
          ldfrag(tile + bn * kGMC * kGLd + fk * kGLd, af[nxt], bf[nxt]);
        }
        if (active) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[cur][i], bf[cur][j]);
        }
      }
      named_arrive(1 + kGNB + b, kGT);
    }
    double* out = a.Gpart + (static_cast<int64_t>(blockIdx.x) * 4 + warp) * 1024;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        *reinterpret_cast<double2*>(out + (i * 8 + fr) * 32 + j * 8 + 2 * fk) =
            make_double2(acc[i][j][0], acc[i][j][1]);
  }
}

// G (full symmetric D x D) and S_A, S_B from the per-CTA partials; ranges summed in order.
__global__ void __launch_bounds__(256) gram_reduce_kernel(const __grid_constant__ GramArgs a, double* __restrict__ Gout,
                                                          double* __restrict__ SA, double* __restrict__ SB) {
  const int D = a.D;
  const int64_t total = static_cast<int64_t>(a.ngroups) * 4 * 1024;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(e / 4096), w = static_cast<int>((e / 1024) % 4), x = static_cast<int>(e % 1024);
    const GramGroup& G = a.grp[g];
    if (w >= G.ntiles) continue;
    const int I = G.fb[G.si[w]], J = G.fb[G.sj[w]];
    const int ii = x / 32, jj = x % 32;
    if (I == J && ii > jj) continue;  // diagonal tiles: upper triangle is authoritative
    const int i = I * 32 + ii, j = J * 32 + jj;
    if (i >= D || j >= D) continue;
    double acc = 0.0;
    for (int r = 0; r < a.rpg; ++r) acc += a.Gpart[(static_cast<int64_t>(r * a.ngroups + g) * 4 + w) * 1024 + x];
    Gout[static_cast<int64_t>(i) * D + j] = acc;
    Gout[static_cast<int64_t>(j) * D + i] = acc;
  }
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < D; f += gridDim.x * blockDim.x) {
    const int og = a.owner[2 * (f / 32)], os = a.owner[2 * (f / 32) + 1];
    double sa = 0.0, sb = 0.0;
    for (int r = 0; r < a.rpg; ++r) {
      const double* sp = a.Spart + (static_cast<int64_t>(r * a.ngroups + og) * 4 + os) * 64;
      sa += sp[f % 32];
      sb += sp[32 + f % 32];
    }
    SA[f] = sa;
    SB[f] = sb;
  }
}

}  // namespace

// Host-side grouping of the upper-triangle 32x32 tiles (see the file header).
bool plan_gram(int64_t nA, int64_t nB, int D, int num_sms, GramPlan& p) {
  const int nb32 = (D + 31) / 32;
  if (nb32 > kGramMaxFb) return false;
  const int nb64 = (nb32 + 1) / 2;
  p.ngroups = 0;
  auto add_group = [&](const int (*tiles)[2], int nt) -> bool {
    if (p.ngroups >= kGramMaxGroups) return false;
    GramGroup& G = p.grp[p.ngroups++];
    G = GramGroup{};
    for (int t = 0; t < nt; ++t) {
      const int blk[2] = {tiles[t][0], tiles[t][1]};
      int sl[2];
      for (int q = 0; q < 2; ++q) {
        int s = 0;
        while (s < G.nfb && G.fb[s] != blk[q]) ++s;
        if (s == G.nfb) G.fb[G.nfb++] = static_cast<unsigned char>(blk[q]);
        sl[q] = s;
      }
      G.si[t] = static_cast<unsigned char>(sl[0]);
      G.sj[t] = static_cast<unsigned char>(sl[1]);
    }
    G.ntiles = static_cast<unsigned char>(nt);
    return true;
  };
  // off-diagonal 64x64 blocks: one group each
  for (int a = 0; a < nb64; ++a)
    for (int b = a + 1; b < nb64; ++b) {
      int tl[4][2], nt = 0;
      for (int i = 2 * a; i < 2 * a + 2; ++i)
        for (int j = 2 * b; j < 2 * b + 2; ++j)
          if (i < nb32 && j < nb32) {
            tl[nt][0] = i;
            tl[nt][1] = j;
            ++nt;
          }
      if (nt > 0 && !add_group(tl, nt)) return false;
    }
  // diagonal 64x64 blocks: their upper 32x32 tiles, packed <= 4 tiles / <= 4 feature blocks
  {
    int tl[4][2], nt = 0, fbs[8], nfb = 0;
    for (int a = 0; a < nb64; ++a) {
      const int cand[3][2] = {{2 * a, 2 * a}, {2 * a, 2 * a + 1}, {2 * a + 1, 2 * a + 1}};
      for (int c = 0; c < 3; ++c) {
        const int i = cand[c][0], j = cand[c][1];
        if (i >= nb32 || j >= nb32) continue;
        int extra = 0;
        for (int q = 0; q < 2; ++q) {
          const int blk = q == 0 ? i : j;
          bool seen = (q == 1 && j == i);
          for (int s = 0; s < nfb && !seen; ++s) seen = fbs[s] == blk;
          extra += seen ? 0 : 1;
        }
        if (nt == 4 || nfb + extra > 4) {
          if (!add_group(tl, nt)) return false;
          nt = 0;
          nfb = 0;
        }
        for (int q = 0; q < 2; ++q) {
          const int blk = q == 0 ? i : j;
          bool seen = false;
          for (int s = 0; s < nfb; ++s) seen = seen || fbs[s] == blk;
          if (!seen) fbs[nfb++] = blk;
        }
        tl[nt][0] = i;
        tl[nt][1] = j;
        ++nt;
      }
    }
    if (nt > 0 && !add_group(tl, nt)) return false;
  }
  // owner of each feature block's column sums: the group holding its diagonal tile
  for (int fb = 0; fb < nb32; ++fb) {
    p.owner[2 * fb] = -1;
    for (int g = 0; g < p.ngroups; ++g)
      for (int t = 0; t < p.grp[g].ntiles; ++t)
        if (p.grp[g].fb[p.grp[g].si[t]] == fb && p.grp[g].fb[p.grp[g].sj[t]] == fb) {
          p.owner[2 * fb] = g;
          p.owner[2 * fb + 1] = p.grp[g].si[t];
          p.grp[g].own[p.grp[g].si[t]] = 1;
        }
    if (p.owner[2 * fb] < 0) return false;
  }
  const int64_t N = nA + nB;
  const int64_t chunks = N > 0 ? (N + kGMC - 1) / kGMC : 1;
  int rpg = (2 * (num_sms > 0 ? num_sms : 148)) / p.ngroups;
  if (rpg < 1) rpg = 1;
  if (rpg > chunks) rpg = static_cast<int>(chunks);
  p.rpg = rpg;
  p.per = ((N + rpg - 1) / rpg + kGMC - 1) / kGMC * kGMC;
  p.nctas = p.ngroups * rpg;
  p.gpart_doubles = static_cast<int64_t>(p.nctas) * 4 * 1024;
  p.spart_doubles = static_cast<int64_t>(p.nctas) * 4 * 64;
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
  a.rpg = p.rpg;
  a.per = p.per;
  a.Gpart = Gpart;
  a.Spart = Spart;
  for (int g = 0; g < p.ngroups; ++g) a.grp[g] = p.grp[g];
  for (int q = 0; q < 2 * kGramMaxFb; ++q) a.owner[q] = static_cast<short>(p.owner[q]);
  cudaError_t e;
  const bool vec = (D % 4) == 0;
  auto kern = vec ? gram_kernel<true> : gram_kernel<false>;
  if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kGSmem))) !=
      cudaSuccess)
    return e;
  count_launch();
  kern<<<p.nctas, kGT, kGSmem, st>>>(a);
  count_launch();
  gram_reduce_kernel<<<148 * 2, 256, 0, st>>>(a, Gout, SA, SB);
  return cudaGetLastError();
}

}  // namespace prohd
