// ko_score_d128_tbl.cu — head_dim 128 instantiations of the scoring kernel, table packing
// (every routed launch; grid launches that need fewer tiles this way).
#include "ko_score.cuh"

namespace ko {

cudaError_t launch_score_d128_tbl(const ScoreParams& p, int CPR0, int tnt, int64_t max_units,
                                  cudaStream_t s) {
#define KO_DISPATCH_TBL(C0, T) \
  if (CPR0 == C0 && tnt == T) return launch_score_t<128, C0, 0, false, T>(p, max_units, s);
  KO_DISPATCH_TBL(1, 1) KO_DISPATCH_TBL(1, 2) KO_DISPATCH_TBL(1, 4) KO_DISPATCH_TBL(2, 1)
  KO_DISPATCH_TBL(2, 2) KO_DISPATCH_TBL(2, 4) KO_DISPATCH_TBL(4, 2) KO_DISPATCH_TBL(4, 4)
  KO_DISPATCH_TBL(4, 8) KO_DISPATCH_TBL(8, 4) KO_DISPATCH_TBL(8, 8)
#undef KO_DISPATCH_TBL
  return cudaErrorInvalidValue;
}

}  // namespace ko
