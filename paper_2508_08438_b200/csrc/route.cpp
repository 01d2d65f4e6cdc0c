// route.cpp -- multi-GPU request router (host): skv_route / skv_route_depth of include/safekv_b200.h.
#include "../../include/safekv_b200.h"
#include "route.hpp"

extern "C" {

int skv_route_depth(const uint32_t* tokens, const uint64_t* offsets, uint32_t n_prompts, uint32_t block_tokens,
                    uint32_t depth, const uint64_t* prompt_ids, uint32_t world, uint32_t* rank_out) {
  if (!offsets || !rank_out || (n_prompts && !tokens) || block_tokens == 0 || world == 0) return SKV_ERR_ARG;
  for (uint32_t p = 0; p < n_prompts; ++p) {
    if (offsets[p + 1] < offsets[p]) return SKV_ERR_ARG;
    rank_out[p] = skvroute::route_one(tokens + offsets[p], offsets[p + 1] - offsets[p], block_tokens, depth,
                                       prompt_ids ? prompt_ids[p] : p, world);
  }
  return SKV_OK;
}

int skv_route(const uint32_t* tokens, const uint64_t* offsets, uint32_t n_prompts, uint32_t block_tokens,
              const uint64_t* prompt_ids, uint32_t world, uint32_t* rank_out) {
  return skv_route_depth(tokens, offsets, n_prompts, block_tokens, 0, prompt_ids, world, rank_out);
}

}  // extern "C"
