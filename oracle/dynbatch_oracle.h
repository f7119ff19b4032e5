/* oracle/dynbatch_oracle.h — CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load liboracle.so, and
 * only as the checker or the timed CPU baseline — never as a product path.
 *
 * Parity status:
 *   - RNG, workloads, labels, improved schedule, dense (Tier A) execute, top-k
 *     gate and MoE forward are PINNED: tests compare them bit-for-bit against
 *     the compiled reference (oracle/_ref/libdbref.so) and the SURVEY §8(c)
 *     golden fingerprints.
 *   - The Tier-B residual conv module body has NO reference implementation
 *     (SPEC.md:268-269 names it): its arithmetic is
 *     "parity unpinned"; only the executor semantics around it are pinned.
 *
 * Batch CSR: prog_off[b+1] node offsets, fid[N], child0[N], child1[N]
 * (program-local child ids, -1 absent), root[b] (program-local).
 * Schedule arrays: step_group_off[steps+1], group_fid[G],
 * group_member_off[G+1], member_example[M], member_node[M].
 */
#ifndef DYNBATCH_ORACLE_H
#define DYNBATCH_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint64_t mt[312];
  int idx;
} orc_rng;

void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_u64(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
uint64_t orc_mix_seed(uint64_t seed, uint64_t stream);
void orc_random_batch(int64_t rows, int64_t width, uint64_t seed, double* out);
void orc_random_rows(const int64_t* rows, int64_t n, int64_t width, uint64_t seed, double* out);
uint64_t orc_fnv1a64(const void* data, int64_t bytes, uint64_t h);

int64_t orc_gen_batch(int kind, int64_t b, int p, int depth, int length, double branch_prob,
                      uint64_t seed, int32_t* prog_off, int32_t* fid, int32_t* child0,
                      int32_t* child1, int32_t* root);

int orc_labels(int64_t b, const int32_t* prog_off, const int32_t* child0, const int32_t* child1,
               const int32_t* root, int32_t* labels, int32_t* d_max);

int orc_schedule_improved(int64_t b, int p, const int32_t* prog_off, const int32_t* fid,
                          const int32_t* child0, const int32_t* child1, const int32_t* root,
                          int64_t* counts, int32_t* step_group_off, int32_t* group_fid,
                          int32_t* group_member_off, int32_t* member_example,
                          int32_t* member_node);

void orc_dense_weights(int arity, int width, uint64_t seed, int fid, double* w, double* bias);

/* module_kind 0 = dense (Tier A, width W); 1 = residual conv block (Tier B,
 * width C*H*W, CHW element order). trace = [expensive_calls, peak_group_rows,
 * steps]. */
int orc_execute(int module_kind, int64_t b, int p, int width, int C, int H, int W,
                const int32_t* prog_off, const int32_t* fid, const int32_t* child0,
                const int32_t* child1, const int32_t* root, int64_t n_steps,
                const int32_t* step_group_off, const int32_t* group_fid,
                const int32_t* group_member_off, const int32_t* member_example,
                const int32_t* member_node, const double* inputs, uint64_t module_seed,
                double* outputs, int64_t* trace, int64_t* per_function_calls, double* seconds);

void orc_resblock_weights(int arity, int C, uint64_t seed, int fid, double* w0, double* b0,
                          double* w1, double* b1, double* w2, double* b2);

int orc_topk(const double* scores, int64_t T, int64_t n, int64_t k, int32_t* ids,
             double* weights);
void orc_expert_weights(int64_t d, int64_t h, uint64_t seed, int64_t id, double* w1, double* w2);
int orc_moe_forward(const double* inputs, int64_t T, int64_t d, int64_t h, int64_t n, int64_t k,
                    const int32_t* ids, const double* weights, uint64_t expert_seed,
                    const int32_t* expert_subset, int64_t n_subset, double* out, int64_t* trace,
                    double* seconds);

/* IEP classifier head (beyond the reference). */
void orc_head_weights(int C, int P, int F, int A, uint64_t seed, double* wp, double* bp, double* w1,
                      double* b1, double* w2, double* b2);
int orc_head_forward(int64_t b, const double* roots, int C, int P, int F, int A, uint64_t seed,
                     double* logits);

#ifdef __cplusplus
}
#endif
#endif
