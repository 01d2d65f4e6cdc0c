/* safekv_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference algorithm for the SafeKV admission path, used
 * as the parity checker of the CUDA implementation.  It never links the product and
 * is never called by it.  Only tests/, __graft_entry__.smoke() and bench.py's CPU
 * baseline load it.  Parity of this restatement is pinned against the reference
 * itself (oracle/_ref/libsafekv_ref.so, built from the unmodified reference headers)
 * and against the reference's own known-answer tests (tests/test_oracle.py).
 */
#ifndef SAFEKV_ORACLE_H_
#define SAFEKV_ORACLE_H_
#include <stddef.h>
#include <stdint.h>

/* rules: kinds 0 = regex (ECMAScript subset), 1 = whole-token blacklist term.
 * Returns NULL on a pattern error (message in err).  Rule masks use bit i = rule i. */
void* orc_rules_create(uint32_t n, const char* const* patterns, const uint32_t* lens, const uint8_t* kinds,
                       const uint8_t* enabled, char* err, size_t errcap);
void orc_rules_free(void* r);
uint64_t orc_rules_mask(void* r, const uint8_t* text, size_t len);

uint64_t orc_fnv1a64(const uint8_t* p, size_t n);
uint64_t orc_token_seq_digest(const uint32_t* t, size_t n);
uint64_t orc_chain(uint64_t prev_h, uint64_t d);

void* orc_engine_create(void* rules, uint32_t B, uint32_t W, double jump, uint64_t u_pre_max);
void orc_engine_free(void* e);
int orc_engine_admit(void* e, const uint32_t* tok, const uint64_t* off, const uint64_t* users,
                     const uint8_t* owners, uint32_t n_prompts, uint64_t* out_h, uint64_t* out_d,
                     uint64_t* out_mask, uint8_t* out_label, uint8_t* out_decision, uint32_t* out_matched,
                     uint8_t* out_tier);
int orc_engine_commit(void* e);
int orc_engine_ttft(void* e, const uint64_t* request_ids, double t_base, double c_prefill, double pen_dram,
                    double pen_ssd, double sigma, uint64_t seed, double* out_ttft, uint32_t* out_intra,
                    uint32_t* out_inter);
int orc_engine_set_tiers(void* e, const uint32_t* tok, const uint64_t* off, uint32_t n_prompts,
                         const uint8_t* tiers);
int orc_engine_epoch(void* e, uint64_t* out_epoch, size_t cap, uint64_t* ev_h, uint64_t* ev_d, uint8_t* ev_action,
                     double* ev_now, double* ev_prev, uint64_t* ev_upre, size_t* n_events);
size_t orc_engine_export(void* e, size_t cap, uint64_t* h, uint64_t* d, uint64_t* creator, uint8_t* label,
                         uint8_t* owner, uint8_t* tier, uint64_t* hit_cur, uint64_t* u_cnt, uint64_t* hit_pre,
                         uint64_t* u_pre);
#endif
