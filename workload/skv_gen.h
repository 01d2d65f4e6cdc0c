/* skv_gen.h -- deterministic synthetic prompt batches for the bench configs and the tests
 * (SURVEY.md section 8(d)).  BENCH / TEST INFRASTRUCTURE: this is not part of the product
 * library (paper_2508_08438_b200/libsafekv_b200.so).  The same source is compiled into
 * workload/libskv_gen.so (our bench arm, tests) and into oracle/_ref/libsafekv_ref.so (the
 * reference arm), so both arms admit byte-identical inputs without the reference arm ever
 * loading the product library.  Built from the reference's generator primitives, restated:
 * SplitMix64 / derive_seed (util.hpp:14-55), detail::filler (workload.hpp:256-266),
 * detail::make_secret (workload.hpp:182-241). */
#ifndef SKV_GEN_H_
#define SKV_GEN_H_
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint64_t n_prompts, prompt_tokens;  /* prompt length (all prompts equal) */
  uint64_t n_users;                   /* user = first_user + prompt_id % n_users */
  uint64_t first_user;
  uint64_t pool_size, pool_tokens;    /* shared-prefix pool                */
  double shared_fraction;             /* fraction of prompts that start with a pool prefix */
  double pii_per_kib;                 /* PII phrases per KiB of unique body */
  uint32_t pii_mix;                   /* 1: config-3 mix (60% none, 30% one per 2 KiB, 10% one per 256 B) */
  uint32_t pad0_;
  uint64_t seed;
  uint64_t prompt_id_base;            /* global id of prompt 0 (sharding)  */
  /* routed generation: with route_world > 1 the batch is the first n_prompts global ids
   * >= prompt_id_base whose prompt skv_route_depth(..., route_depth, ...)s to route_rank */
  uint32_t route_world, route_rank, route_block_tokens, route_depth;
  uint64_t* prompt_ids_out;           /* optional: global id of each generated prompt */
} skvgen_spec;

/* Writes n_prompts*prompt_tokens tokens and n_prompts+1 offsets; users/owners may be NULL.
 * Returns 0, 1 (bad argument) or 4 (bad spec). */
int skvgen_generate(const skvgen_spec* spec, uint32_t* tokens, uint64_t* offsets, uint64_t* users,
                    uint8_t* owners, int nthreads);
/* The pool prefixes themselves (pool_size prompts of pool_tokens). */
int skvgen_generate_pool(const skvgen_spec* spec, uint32_t* tokens, uint64_t* offsets, uint64_t* users,
                         uint8_t* owners);
/* The router's rank per prompt (the same arithmetic as the product's skv_route_depth). */
int skvgen_route(const uint32_t* tokens, const uint64_t* offsets, uint32_t n_prompts, uint32_t block_tokens,
                 uint32_t depth, const uint64_t* prompt_ids, uint32_t world, uint32_t* rank_out);

#ifdef __cplusplus
}
#endif
#endif
