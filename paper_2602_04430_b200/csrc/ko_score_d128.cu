// ko_score_d128.cu — head_dim 128 instantiations of the scoring kernel.
#include "ko_score.cuh"

namespace ko {

cudaError_t launch_score_d128(const ScoreParams& p, int CPR, int NT, int64_t max_units,
                             cudaStream_t s) {
#define KO_DISPATCH(C, T) \
  if (CPR == C && NT == T) return launch_score_t<128, C, T>(p, max_units, s);
  // (class stride, tiles) pairs the table packing can produce: a C-class row has C (bf16) or 2C
  // (fp32) entries, at most 2·NT of them per lane group
  KO_DISPATCH(1, 1) KO_DISPATCH(1, 2) KO_DISPATCH(1, 4) KO_DISPATCH(2, 1) KO_DISPATCH(2, 2)
  KO_DISPATCH(2, 4) KO_DISPATCH(4, 2) KO_DISPATCH(4, 4) KO_DISPATCH(4, 8) KO_DISPATCH(8, 4)
  KO_DISPATCH(8, 8)
#undef KO_DISPATCH
  return cudaErrorInvalidValue;
}

cudaError_t launch_grid_final(const ScoreParams& p, int CPR, cudaStream_t s) {
  switch (CPR) {
    case 1: return launch_grid_final_t<1>(p, s);
    case 2: return launch_grid_final_t<2>(p, s);
    case 4: return launch_grid_final_t<4>(p, s);
    case 8: return launch_grid_final_t<8>(p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace ko
