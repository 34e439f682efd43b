// ko_score_d64.cu — head_dim 64 instantiations of the scoring kernel (both packings).
#include "ko_score.cuh"

namespace ko {

cudaError_t launch_score_d64(const ScoreParams& p, int CPR0, int CPR1, bool nolo, int tnt,
                             int64_t max_units, cudaStream_t s) {
#define KO_DISPATCH(C0, C1) \
  if (tnt == 0 && CPR0 == C0 && CPR1 == C1 && !nolo) return launch_score_t<64, C0, C1, false, 0>(p, max_units, s);
#define KO_DISPATCH_NOLO(C0, C1) \
  if (tnt == 0 && CPR0 == C0 && CPR1 == C1 && nolo) return launch_score_t<64, C0, C1, true, 0>(p, max_units, s);
#define KO_DISPATCH_TBL(C0, T) \
  if (CPR0 == C0 && tnt == T) return launch_score_t<64, C0, 0, false, T>(p, max_units, s);
  KO_DISPATCH(1, 0) KO_DISPATCH(1, 1) KO_DISPATCH(2, 0) KO_DISPATCH(2, 1) KO_DISPATCH(2, 2)
  KO_DISPATCH(4, 0) KO_DISPATCH(4, 1) KO_DISPATCH(4, 2) KO_DISPATCH(4, 4) KO_DISPATCH(8, 0)
  KO_DISPATCH(8, 1) KO_DISPATCH(8, 2) KO_DISPATCH(8, 4) KO_DISPATCH(8, 8)
  KO_DISPATCH_NOLO(2, 0) KO_DISPATCH_NOLO(4, 0) KO_DISPATCH_NOLO(8, 0) KO_DISPATCH_NOLO(2, 1)
  KO_DISPATCH_NOLO(4, 1) KO_DISPATCH_NOLO(8, 1)
  KO_DISPATCH_TBL(1, 1) KO_DISPATCH_TBL(1, 2) KO_DISPATCH_TBL(1, 4) KO_DISPATCH_TBL(2, 1)
  KO_DISPATCH_TBL(2, 2) KO_DISPATCH_TBL(2, 4) KO_DISPATCH_TBL(4, 2) KO_DISPATCH_TBL(4, 4)
  KO_DISPATCH_TBL(4, 8) KO_DISPATCH_TBL(8, 4) KO_DISPATCH_TBL(8, 8)
#undef KO_DISPATCH_TBL
#undef KO_DISPATCH_NOLO
#undef KO_DISPATCH
  return cudaErrorInvalidValue;
}

}  // namespace ko
