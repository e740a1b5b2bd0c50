// prohd_steps.cuh — the ProHD (Alg. 3) orchestration entry points.
#pragma once
#include "../../include/prohd.h"

#include <cstddef>
#include <cstdint>

namespace prohd {
// Workspace bytes for prohd_run at these sizes.
size_t estimate_workspace_bytes(int64_t nA, int64_t nB, int D, int k, int64_t m, bool host_inputs,
                                bool certified = false);
}  // namespace prohd

// Alg. 3 end to end. If `dirs_in` is non-null it holds n_dirs_in fp64 directions
// (host, D x n_dirs_in, column 0 = centroid axis) that replace steps 1a-1b.
// mode 0: Alg. 3 as written (subset-subset HD); mode 1: certified subset-full estimate.
int prohd_run(prohd_ctx* ctx, const float* A, int64_t nA, const float* B, int64_t nB, int32_t D, int32_t k,
              int64_t m, const double* dirs_in, int32_t n_dirs_in, prohd_est* out, double* dirs_out,
              int64_t* idxA_out, int64_t* idxB_out, int mode = 0, const int64_t* counts = nullptr);
// counts (optional, HOST, 4 values): per-tail counts {A: centroid axis, A: PCs, B: centroid
// axis, B: PCs} for the paper-literal parameterisation;
// `m` must then be their maximum (it sizes the workspace).
