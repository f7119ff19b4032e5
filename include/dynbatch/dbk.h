/* dbk.h — thin internal host→CUDA C-ABI of the dynbatch B200 library.
 *
 * Raw device pointers, sizes and a cudaStream_t (passed as void*); every
 * launcher returns 0 or a cudaError_t value and never synchronizes. Device
 * scalars (d_max, group counts, error flags) stay in device memory so one
 * forward needs a single tiny device→host read (the step count).
 *
 * Node numbering: "global" node g = prog_off[e] + local id (CSR order =
 * (example, node) order, which is the reference's member order).
 */
#ifndef DYNBATCH_DBK_H
#define DYNBATCH_DBK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- scheduler
 * Replaces max_root_distance_labels + schedule_improved/make_step
 * (src/program.cpp:239-272, src/schedule.cpp:66-79,135-164). */

/* Per-node step labels, one thread per program; strategy (db_strategy):
 *   2 improved: labels[g] = longest root→g distance (Kahn from the root);
 *   1 standard: labels[g] = g's position in postorder_flatten
 *               (src/program.cpp:274-303; schedule_standard's column);
 *   3 online:   labels[g] = g's height (schedule_online_full's round).
 * dev_scalars[0] = largest label (atomicMax), dev_scalars[1] |= 1 on a
 * cycle / unreachable node. scratch: 2·N int32. child*: global ids or -1. */
int dbk_sched_labels(int64_t b, int64_t N, const int32_t* prog_off, const int32_t* child_off,
                     const int32_t* child_list, const int32_t* root_g, int32_t* labels,
                     int32_t* scratch, int32_t* dev_scalars, int32_t strategy, void* stream);

/* Labels of a batch whose programs all share one tree shape (programs of n
 * nodes, shape labels table[n], depth dmax): the balanced-tree static
 * schedule (SURVEY.md §3 balanced_static_schedule); sets dev_scalars[0] = dmax. */
int dbk_sched_labels_static(int64_t N, int32_t n, const int32_t* table, int32_t dmax, int32_t* labels,
                            int32_t* dev_scalars, void* stream);

/* Stable counting sort of all N nodes by key = step·p + fid over CSR
 * order, step = label (ascending: standard, online) or d_max − label
 * (improved); writes member_g[N] (sorted global ids), and the group
 * tables: group_fid[G], group_begin[G+1], step_group_begin[S+1] (and empty
 * steps up to steps_cap, so a host may launch per-step work for an upper
 * bound of S) with dev_scalars[2] = G. seg_hist must hold max_keys ·
 * n_segments ints with max_keys ≥ (d_max+1)·p; size from
 * dbk_bucket_sort_scratch(N, max_keys). */
int dbk_sched_bucket_sort(int64_t N, int32_t p, int32_t max_keys, const int32_t* fid,
                          const int32_t* labels, int32_t* dev_scalars, int32_t* seg_hist,
                          int32_t* member_g, int32_t* group_fid, int32_t* group_begin,
                          int32_t* step_group_begin, int32_t steps_cap, int32_t ascending, void* stream);

/* build_program_from_prefix (src/program.cpp:95-142) for b concatenated
 * prefix sequences (tokens, seq_off[b+1]), one thread per program: writes
 * the CSR (prog_off, fid, child_off[N+1], child_list, child0/1, example,
 * root_g) and fwd_ok (expensive non-root node). stack: N int2 scratch.
 * *err (first error wins): 1 empty sequence, 2 unknown function,
 * 3 underfull, 4 overfull. */
int dbk_build_prefix(int64_t b, const int32_t* tokens, const int32_t* seq_off, int32_t p, const int32_t* arity_of,
                     int32_t* prog_off, int32_t* fid, int32_t* child_off, int32_t* child_list, int32_t* child0,
                     int32_t* child1, int32_t* example, int32_t* root_g, int32_t* fwd_ok, void* stack,
                     int32_t* err, void* stream);

/* Scratch (int32 count) the bucket sorts need in seg_hist. */
int64_t dbk_bucket_sort_scratch(int64_t n_items, int32_t max_keys);

/* Generic stable counting sort by an explicit key in [0, n_keys): order[]
 * receives item indices sorted by key, stable in index order; offsets[n_keys+1]
 * the bucket starts. Used for the MoE expert dispatch (group_by_function). */
int dbk_stable_bucket_sort(int64_t n_items, int32_t n_keys, const int32_t* keys,
                           int32_t* seg_hist, int32_t* order, int32_t* offsets, void* stream);

/* ------------------------------------------------------ dense (Tier A) step
 * One step of execute() (src/executor.cpp:117-166) with apply_module
 * (src/modules.cpp:52-108): for every expensive member of step s,
 * out = relu(bias + Σ_k Σ_i x_k[i]·W[(kW+i)W + j]) in fp64 with the
 * reference's ascending fused multiply-add order. Leaves alias inputs. */
int dbk_dense_step(int32_t step, int32_t width, const int32_t* step_group_begin,
                   const int32_t* group_fid, const int32_t* group_begin, const int32_t* member_g,
                   const int32_t* arity_of, const int32_t* child_off, const int32_t* child_list,
                   const int32_t* example, const double* inputs, double* values,
                   int32_t* present, const double* const* weights,
                   const double* const* biases, int32_t* err, int32_t max_arity,
                   int32_t blocks, void* stream);

/* root rows → out[b × width] (fp64). */
/* apply_module (src/modules.cpp:52-108) on stacked rows: x [rows][arity·width]
 * (operand k of a row at column k·width), w [arity·width][width], bias
 * [width] → out [rows][width]; the fp64 fma chain of dbk_dense_step. */
int dbk_dense_apply(int64_t rows, int32_t arity, int32_t width, const double* x, const double* w,
                    const double* bias, double* out, void* stream);
int dbk_dense_gather_roots(int64_t b, int32_t width, const int32_t* root_g,
                           const int32_t* present, const double* values, double* out,
                           int32_t* err, void* stream);

/* ------------------------------------------------------- resblock (Tier B)
 * Maps are C=128 × 14 × 14. Node values / inputs are fp32 "plane maps"
 * [16 planes][196 px][8 ch]; per-step staging is fp16 planes over a packed,
 * zero-padded 15×15 position grid (rb_conv.cu header). */

/* Per step: segment starts (seg_start[g], -1 for leaf groups), tile lists
 * (all expensive groups; binary groups only) and their per-step offsets.
 * training != 0 (here and in dbk_rb_step): a training forward — every
 * expensive node also keeps its fp32 value and the mid / block-input images
 * stay in place, since the backward reads them. */
int dbk_rb_plan(int32_t n_steps, const int32_t* step_group_begin, const int32_t* group_fid,
                const int32_t* group_begin, const int32_t* arity_of, int32_t* seg_start,
                int32_t* group_tile0, int32_t* group_bintile0, int32_t* step_tile_begin,
                int32_t* step_bintile_begin, int32_t* step_positions, int32_t* tile_group,
                int32_t* tile_q0, int32_t* bin_group, int32_t* bin_q0, int64_t n_nodes,
                const int32_t* member_g, const int32_t* child0, const int32_t* child1,
                const int32_t* fwd_ok, int32_t* fwd_pos, int32_t* fwd_slot, int32_t* fwd_parent,
                int32_t* need, int32_t tile_m, int32_t training, void* stream);
/* Gather of operands no child epilogue forwards, from the task lists that
 * dbk_rb_memtab emits (32-byte tasks, list 0 = leaves of every step, list 1
 * = children shared by several parents, processed for `step` only): fp32
 * plane maps → staged fp16 images (hi; plus the lo image, the block's
 * residual, in stage_lo for unary members); plane_stride in rows. */
int dbk_rb_gather(const void* tasks, const int32_t* n_tasks, int32_t list, int32_t step, int64_t task_cap,
                  void* stage_x, void* stage_lo, void* stage_cat, int64_t plane_stride, int32_t* err,
                  int32_t blocks, void* stream);
/* One persistent launch (one CTA per SM, CTA pairs) for steps [step,
 * step_end) over a device work queue of their tiles, step s + 1's after
 * all of step s (step_done[s] counts step s's finished conv3x3 #2 tiles): conv1x1 over [x; y] → z hi/lo (stage_x / stage_lo),
 * conv3x3 #1 → mid (stage_mid), conv3x3 #2 + residual (accumulated on the
 * tensor cores from the hi/lo images through the identity blocks `ident`) →
 * hi/lo images of the parent's call and fp32 values where a reader needs
 * them. Tile-level dependencies through done flags (done0 per bin tile,
 * done1 per tile; == epoch means done); queue[step] and step_done[step ..
 * step_end) must be 0 at launch.
 * D[128 channels][tile_m positions] per tile (tcgen05.mma M = 128, N =
 * tile_m, 256 or 128; the plan must have used the same tile_m). *err gets
 * the first of 9 (a module output is non-finite, src/executor.cpp:156-159)
 * or 10 (a value exceeds the fp16 operand range, |x| > 65504); the gather
 * flags its input maps the same way. */
/* Sets the step kernel's attributes; call before capturing a forward. */
int dbk_rb_configure(void);
int dbk_rb_step(int32_t step, int32_t step_end, int32_t epoch, const int32_t* step_tile_begin,
                const int32_t* tile_group,
                const int32_t* tile_q0, const int32_t* step_bintile_begin, const int32_t* bin_group,
                const int32_t* bin_q0, const int32_t* group_fid, const int32_t* group_begin,
                const int32_t* seg_start, const int32_t* group_tile0, const int32_t* group_bintile0,
                const void* memtab, void* stage_x, void* stage_lo, void* stage_cat, void* stage_mid,
                int64_t plane_stride, const void* const* w0, const void* const* w1, const void* const* w2,
                const float* const* b0, const float* const* b1, const float* const* b2, const void* ident,
                int32_t* done0, int32_t* done1, int32_t* step_done, int32_t* queue, int32_t* err,
                int32_t* ready, const int32_t* need, const int32_t* member_g, const int32_t* order, const float* values,
                int64_t values_floats, int32_t tile_m, int32_t num_sms, int32_t training,
                void* stream);
/* Zeroes stage_x rows between each segment's last image and its tile end
 * (read as top / left pads by the next segment's first image), every
 * forward, so a new layout needs no full re-zeroing. */
int dbk_rb_zero_gaps(int32_t n_steps, const int32_t* step_group_begin, const int32_t* group_begin,
                     const int32_t* seg_start, void* stage_x, int64_t plane_stride, int32_t tile_m, void* stream);
/* Per-member epilogue table (32 bytes per member, schedule order: own fp32
 * slot, forwarding target row / buffer, keep-fp32 flag) and the gather task
 * lists (n_tasks[2] counters, reset here; capacity task_cap per list), built
 * after dbk_rb_plan from its forwarding tables. */
/* Claim order of every step's work units (conv1x1 tiles DYNBATCH_BIN_LEAD SM-rows ahead of the conv3x3 #1
 * tiles that read them); order[(bintile_begin[s] + 2·tile_begin[s]) / 2 + k] = (kind << 28) | unit. */
int dbk_rb_order(int32_t n_steps, const int32_t* step_tile_begin, const int32_t* step_bintile_begin,
                 const int32_t* tile_group, const int32_t* group_tile0, const int32_t* group_bintile0,
                 int32_t num_sms, int32_t* prefix, int32_t* order, void* stream);
int dbk_rb_memtab(int32_t n_steps, const int32_t* step_group_begin, const int32_t* group_fid,
                  const int32_t* group_begin, const int32_t* seg_start, const int32_t* member_g,
                  const int32_t* fwd_pos, const int32_t* fwd_slot, const int32_t* arity_of, const int32_t* fid,
                  const int32_t* child0, const int32_t* child1, const int32_t* example, const int32_t* fwd_ok,
                  const float* inputs, float* values, void* memtab, void* tasks, int32_t* n_tasks,
                  int64_t task_cap, const int32_t* fwd_parent, int32_t* need, int32_t tile_m, void* stream);
int dbk_rb_debug(unsigned long long* out64, int32_t reset, int32_t enable);
/* Whether the wait-counter (debug) step kernel is selected (a launch-time choice). */
int dbk_rb_debug_enabled(void);
int dbk_rb_inputs_from_chw(int64_t rows, const float* chw, float* planes, void* stream);
int dbk_rb_outputs_to_chw(int64_t b, const int32_t* root_g, const int32_t* fid,
                          const int32_t* arity_of, const int32_t* example, const float* inputs,
                          const float* values, float* chw, void* stream);

/* --------------------------------------------------------------------- MoE */
/* top_k_gate (src/moe.cpp:36-69), one warp per token, fp64. */
int dbk_moe_topk(int64_t T, int32_t n, int32_t k, const double* scores, int32_t* ids,
                 double* weights, int32_t* err, void* stream);
/* fp64 expert apply + staging (src/moe.cpp:98-145, 244-251), reference order. */
int dbk_moe_expert_fp64(int64_t T, int32_t n, int32_t k, int32_t d, int32_t h,
                        const int32_t* order, const int32_t* offsets, const double* x,
                        const double* const* w1, const double* const* w2, double* hidden,
                        double* staged, int32_t* tile_scratch /* n+1 */, void* stream);
/* combine (src/moe.cpp:254-264): out[t] = Σ_slot w·y in slot order. */
int dbk_moe_combine_fp64(int64_t T, int32_t k, int32_t d, const double* weights,
                         const double* staged, double* out, void* stream);

/* Tensor-core experts (moe_gemm.cu). fmt selects the 16-bit operand format
 * of the dispatched rows, weights, H and Y: DBK_FMT_F16 (fp16, the precise
 * mode) or DBK_FMT_BF16; tcgen05 kind::f16 with fp32 accumulation either way.
 * Per-expert 256-row padded layout and tile list; dispatch of x rows (fp32 →
 * 16-bit, pre-tiled operand); grouped GEMM (epi 0: ReLU → tiled H, epi 1: Y
 * rows); slot-order combine. */
enum { DBK_FMT_BF16 = 0, DBK_FMT_F16 = 1 };
int dbk_moe_tc_layout(int32_t n, const int32_t* offsets, int32_t* pstart, int32_t* tile_expert,
                      int32_t* tile_rb, int32_t* n_tiles, void* stream);
/* dispatch: row_of_item[item] = the item's padded row, then one warp per
 * token writes its 16-bit x row into its k rows of the SWIZZLE_128B tiled A
 * (k ≤ 8, d a multiple of 256). */
int dbk_moe_tc_dispatch(int32_t fmt, int64_t T, int32_t k, int32_t d, const int32_t* order, const int32_t* ids,
                        const int32_t* offsets, const int32_t* pstart, const float* x, void* A,
                        int32_t* row_of_item, int32_t blocks, void* stream);
/* row tiles [tile_begin, tile_end) of the tile list (tile_end < 0: all
 * *n_tiles); EP chunks run one contiguous expert range at a time. epi 1:
 * padded row r's output goes to Y row out_row[r] (skipped when < 0; out_row
 * NULL = row r) — the EP receive order directly, no unpack pass. */
int dbk_moe_tc_gemm(int32_t fmt, int32_t epi, int32_t n, int32_t K, int32_t N, const int32_t* n_tiles,
                    const int32_t* tile_expert, const int32_t* tile_rb, const void* A,
                    const void* const* W, void* H, void* Y, int32_t tile_begin, int32_t tile_end,
                    const int32_t* out_row, int32_t sms, void* stream);
/* Training (train.cu). PI = per-member padded image:
 * 257 rows (16 zero guard rows, the 225 packed positions, 16 guard rows) ×
 * channels, fp32. */
int dbk_tr_stage_to_pi(int32_t n, const int64_t* rows, const void* hi, const void* lo, int64_t ps, int32_t plane0,
                       int32_t planes, float* out, void* stream);
/* bias gradients of 128 channels: slab i = rows [slab_row[2i], slab_row[2i+1]) into dst[i] */
int dbk_tr_colsum_seg(int32_t slabs, const int64_t* slab_row, float* const* dst, const float* a, void* stream);
/* absmax (nullable): atomicMax of |DA2| (float bits) for the fp16 gradient scale */
int dbk_tr_da_out(int32_t n, const int32_t* nodes, const float* dy_nodes, const float* values, float* out,
                  uint32_t* absmax, void* stream);
int dbk_tr_im2col(int64_t rows, int32_t ch, const float* x, float* cols, void* stream);
int dbk_tr_col2im(int32_t n, int32_t ch, const float* g, const float* res, const float* mask, float* out,
                  void* stream);
int dbk_tr_mask(int64_t count, const float* g, const float* act, float* out, void* stream);
int dbk_tr_colsum(int64_t rows, int32_t cols, const float* a, float* db, void* stream);
int dbk_tr_route(int32_t n, const int32_t* nodes, const int32_t* child, const int32_t* fid, const int32_t* arity_of,
                 const int32_t* example, const float* src, int32_t ch, int32_t c0, float* dy_nodes, float* d_inputs,
                 void* stream);
/* loss holds 1 + b floats: [1 + e] = program e's cross-entropy, [0] = their
 * mean summed in a fixed order (bit-reproducible); dlogits [b][A] */
int dbk_tr_softmax_ce(int64_t b, int32_t A, int32_t ld, const float* logits, const int32_t* labels, float* dlogits,
                      float* loss, void* stream);
/* Data gradient of a 3×3 conv as a tf32 implicit GEMM (bwd_conv.cu): packed
 * dA (dbk_tr_pack_sw128f: PI rows → 32-channel SW128 chunk rows, `lead` zero
 * rows first), tiles of 256 PI rows within one group (tile_row0 a multiple of
 * 8; rows [tile_lo, tile_hi) written), transposed tap weights per function
 * (dbk_tr_pack_dgrad_weights: 9 × 4 blocks of 16 KB); out = D ⊙ (mask > 0)
 * and / or + resid at real positions, 0 at pads and guard rows. */
int dbk_tr_pack_sw128f(int64_t rows, int64_t rows_alloc, int32_t lead, const float* pi, void* out, void* stream);
int dbk_tr_pack_dgrad_weights(const float* w, void* out, void* stream);
/* fp16 variant (f16 != 0 in dbk_tr_dgrad): dA packed by dbk_tr_pack_sw128h
 * with its absmax scale, weights by dbk_tr_pack_dgrad_weights_h (9 × 2 blocks) */
int dbk_tr_pack_dgrad_weights_h(const float* w, void* out, void* stream);
int dbk_tr_dgrad(const void* packed, int32_t f16, const uint32_t* absmax, int64_t rows_alloc, int32_t lead,
                 int32_t n_tiles, const int32_t* tile_row0, const int32_t* tile_lo, const int32_t* tile_hi,
                 const int32_t* tile_fn, const void* const* wpack, const float* mask, const void* mask_h,
                 const float* resid, float* out, uint32_t* out_absmax, int32_t sms, void* stream);
/* The forward's staged fp16 rows of n members (staging row of member k's
 * position 0: srows[k]) → packed backward rows, as dbk_tr_pack_sw128h lays
 * them out (the weight gradient's activations, the data gradient's mask_h);
 * and the binary blocks' mask from such packed rows. */
int dbk_tr_stage_to_pack(int32_t n, const int64_t* srows, const void* hi, int64_t plane_stride, int64_t rows_alloc,
                         int32_t lead, void* out, void* stream);
int dbk_tr_mask_h(int64_t r0, int64_t n, const float* g, const void* packed, int64_t rows_alloc, int32_t lead,
                  float* out, void* stream);
/* Weight gradient of a 3×3 conv (bwd_conv.cu): items [4][item_stride] = K
 * range [k0, k1) of PI rows (multiples of 16, inside one call group or its
 * zero guard rows), kernel row dr, function; gw[function] += Σ x[r + s_t] ⊗
 * dA[r] for the three taps of row dr. x and dA are packed to fp16 by
 * dbk_tr_pack_sw128h, dA scaled from its |max| (dbk_tr_absmax). */
int dbk_tr_absmax(int64_t n, const float* x, uint32_t* out, void* stream);
int dbk_tr_pack_sw128h(int64_t rows, int64_t rows_alloc, int32_t lead, const float* pi, const uint32_t* absmax,
                       void* out, void* stream);
int dbk_tr_wgrad(const void* x_packed, const void* da_packed, const uint32_t* absmax, int64_t rows_alloc, int32_t lead,
                 int32_t n_items, const int32_t* items, int64_t item_stride, float* const* gw, int32_t sms,
                 void* stream);
/* SGD update and the forward's weight layouts rebuilt from fp32 masters:
 * w -= lr·g; the step kernel's fp16 blocks (pack_blocks layout); the grouped
 * GEMM's fp16 B tiles of a K × N_src matrix padded to N columns. */
int dbk_tr_sgd(int64_t n, float* w, const float* g, float lr, void* stream);
int dbk_tr_pack_conv_weights(const float* w, int32_t cin, int32_t taps, void* out, void* stream);
int dbk_tr_tile_weights(const float* w, int32_t K, int32_t N_src, int32_t N, void* out, void* stream);
int dbk_tr_unpack_h(int64_t rows, int32_t K, const void* h, float* out, void* stream);
int dbk_tr_unpack_sw128(int64_t rows, int32_t K, const void* a, float* out, void* stream);
int dbk_tr_pool_bwd(int64_t b, int32_t P, const float* proj, const float* dpooled, float* dproj, void* stream);
int dbk_tr_droots(int64_t b, const int32_t* root_g, const int32_t* fid, const int32_t* arity_of,
                  const int32_t* example, const float* droots, float* dy_nodes, float* d_inputs, void* stream);
/* IEP classifier head operand moves (head.cu): roots → fp16 SW128 tiled
 * rows (program·196 + px) × 128; projection output (tiled H, P columns) →
 * 2×2 max pool → fp16 SW128 tiled rows (program) × 49·P. */
int dbk_head_pack(int64_t b, const int32_t* root_g, const int32_t* fid, const int32_t* arity_of,
                  const int32_t* example, const float* inputs, const float* values, void* A, void* stream);
int dbk_head_pool(int64_t b, int32_t P, const void* H, void* A, void* stream);
/* The same grouped GEMM with an optional per-expert fp32 bias [N] added in
 * the epilogue, and epi 2 = fp32 row-major output (Y is then float*). */
int dbk_tc_gemm_bias(int32_t fmt, int32_t epi, int32_t n, int32_t K, int32_t N, const int32_t* n_tiles,
                     const int32_t* tile_expert, const int32_t* tile_rb, const void* A,
                     const void* const* W, const float* const* bias, void* H, void* Y, int32_t tile_begin,
                     int32_t tile_end, const int32_t* out_row, int32_t sms, void* stream);
int dbk_moe_tc_combine(int32_t fmt, int64_t T, int32_t k, int32_t d, const double* weights,
                       const int32_t* row_of_item, const void* Y, float* out, void* stream);

/* Expert-parallel MoE (moe_gemm.cu): pack the rank's rows in sorted order
 * (16-bit, fmt) with pos_of_item[item] = row; receiver layout from the count
 * matrix cnt[G][E] (source × local expert); scatter received rows into the
 * tiled GEMM operand (expert-major, source-rank order within an expert) with
 * recv_of_row[padded row] = receive row (−1: padding), which GEMM2's
 * epilogue uses to write its rows back in receive order (out_row). */
int dbk_moe_ep_pack(int32_t fmt, int64_t items, int32_t k, int32_t d, const int32_t* order, const float* x,
                    void* send, int32_t* pos_of_item, int32_t blocks, void* stream);
/* counts[e] = offsets[e+1] − offsets[e]: rows per global expert (sends). */
int dbk_moe_ep_counts(int32_t n, const int32_t* offsets, int32_t* counts, void* stream);
int dbk_moe_ep_layout(int32_t G, int32_t E, const int32_t* cnt, int32_t* pstart, int32_t* tile_expert,
                      int32_t* tile_rb, int32_t* n_tiles, int32_t* src_row, int32_t* cum, void* stream);
int dbk_moe_ep_scatter(int32_t G, int32_t E, int32_t d, const int32_t* pstart, const int32_t* tile_expert,
                       const int32_t* src_row, const int32_t* cum, const void* recv, void* A,
                       int32_t* recv_of_row, int32_t row_begin, int32_t row_end, int32_t blocks, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DYNBATCH_DBK_H */
