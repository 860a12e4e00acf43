// k_score_tc.cu -- tcgen05 (5th-gen tensor core) path of ns_score_plans:
// the fwd/bwd comm MLPs as split-TF32 GEMM chains.  (Not built yet.)
#include "ns_internal.cuh"

namespace ns {
struct ScoreArgs;
ns_status run_score_plans_tf32x3(ns_ctx* ctx, const ScoreArgs&, double*) {
    return set_err(ctx, NS_ERR_STATE, "NS_SCORE_TF32X3 is not available in this build");
}
}  // namespace ns
