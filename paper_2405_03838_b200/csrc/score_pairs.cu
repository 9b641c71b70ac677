// score_pairs.cu -- the fast pair scorer (placeholder: routes to the generic scorer).
#include "cosched_internal.h"

namespace cosched {
int launch_score_pairs_fast(const SpaceParams& sp, int64_t n_jobs, const float* ka, const float* kb, int64_t first,
                            int64_t count, float* obj, int32_t* cfg, unsigned long long* best_key,
                            const unsigned long long* err, cudaStream_t st) {
  return launch_score(sp, n_jobs, ka, kb, first, count, obj, cfg, best_key, err, 0, st);
}
}  // namespace cosched
