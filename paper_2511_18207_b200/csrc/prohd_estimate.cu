// prohd_estimate.cu — ProHD Alg. 3 orchestration (filled in by the K1-K5 kernels).
#include "api_common.cuh"
#include "prohd_steps.cuh"

namespace prohd {
size_t estimate_workspace_bytes(int64_t, int64_t, int, int, int64_t, bool) { return 0; }
}  // namespace prohd

int prohd_run(prohd_ctx* ctx, const float*, int64_t, const float*, int64_t, int32_t, int32_t, int64_t,
              const double*, int32_t, prohd_est*, double*, int64_t*, int64_t*) {
  int rc = enter(ctx);
  if (rc) return rc;
  return fail(ctx, PROHD_E_NOTIMPL, "prohd_estimate not built yet");
}
