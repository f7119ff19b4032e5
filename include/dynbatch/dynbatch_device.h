/* dynbatch_device.h — device extensions of the drop-in C ABI.
 *
 * Added beside (never instead of) the reference's 27 entry points, as
 * SURVEY.md §8(b) recommends. Sessions keep a batch, its module weights and
 * all scratch resident in HBM so that the forward pass — device scheduler
 * (labels → stable (level, function) bucket sort → group/tile tables) plus
 * the per-step gather / module / scatter kernels — can be timed alone, with
 * host↔device traffic accounted separately (…_forward_host does both).
 *
 * Module kinds:
 *   DB_MODULE_DENSE    — the reference module body (src/modules.cpp:52-108):
 *                        relu(W·concat(operands) + b), fp64, same fused
 *                        multiply-add order ⇒ bit-identical to the reference.
 *   DB_MODULE_RESBLOCK — the north-star IEP residual block on C×H×W maps
 *                        (C = 128, 14×14): unary y = relu(x + conv3(relu(conv3(x)))),
 *                        binary z = relu(conv1x1([x;y])) then the unary block;
 *                        tcgen05/TMEM implicit-GEMM kernels, fp16 operands,
 *                        fp32 accumulation and fp32 node values.
 * MoE precisions:
 *   DB_MOE_FP64 — reference arithmetic order (src/moe.cpp:98-145, 254-264).
 *   DB_MOE_BF16 — tcgen05 grouped GEMMs, bf16 operands, H and expert outputs,
 *                 fp32 accumulation (≈4e-3 max-norm vs fp64).
 *   DB_MOE_FP16 — the same kernels with fp16 operands, H and expert outputs
 *                 (≤ 1e-3 max-norm vs fp64, same tensor-core rate).
 */
#ifndef DYNBATCH_DYNBATCH_DEVICE_H
#define DYNBATCH_DYNBATCH_DEVICE_H

#include "dynbatch/dynbatch.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { DB_MODULE_DENSE = 0, DB_MODULE_RESBLOCK = 1 } db_module_kind;
typedef enum { DB_MOE_FP64 = 0, DB_MOE_BF16 = 1, DB_MOE_FP16 = 2 } db_moe_precision;

typedef struct {
  int32_t module_kind; /* db_module_kind */
  int32_t channels;    /* RESBLOCK: C (must be 128) */
  int32_t height;      /* RESBLOCK: H (must be 14)  */
  int32_t width_px;    /* RESBLOCK: W (must be 14)  */
  /* Capacity for later db_iep_session_set_programs batches (0: the initial
   * batch's size): programs, total nodes, longest program. */
  int64_t program_capacity;
  int64_t node_capacity;
  int32_t length_capacity;
  int32_t reserved;
} db_module_opts;

/* Session statistics (db_iep_session_stats / db_moe_session_stats). */
typedef struct {
  int64_t steps;
  int64_t groups;
  int64_t expensive_calls;
  int64_t peak_group_rows;
  int64_t members;
  int64_t kernel_launches; /* kernels enqueued by the last forward */
  int64_t h2d_bytes;       /* per …_forward_host call */
  int64_t d2h_bytes;
  double algorithmic_flops; /* module FLOPs of one forward (2·MAC) */
  double algorithmic_bytes; /* minimum HBM bytes of one forward */
} db_session_stats_t;

/* Per-kernel-class device time of a timed loop (CUDA events on the session
 * stream around every launch of the class). Classes: 0 scheduler, 1 plan,
 * 2 gather, 3 moe gate+sort, 4 fused conv step (conv1x1 + conv3x3 ×2) / moe
 * GEMM1, 5 moe GEMM2, 6 layout / combine, 7 dense step. */
typedef struct {
  double ms[8];
  int64_t launches[8];
  double flops[8]; /* algorithmic FLOPs of those launches */
  double bytes[8]; /* algorithmic HBM bytes of those launches */
} db_kernel_times_t;

DYNBATCH_API int32_t db_device_count(void);
/* Pinned (page-locked) host memory for end-to-end transfers. */
DYNBATCH_API void* db_host_alloc(int64_t bytes);
DYNBATCH_API void db_host_free(void* p);
/* Programs [first, last) of gen_batch(opts), bit-identical to those rows of
 * db_batch_generate (for data-parallel shards). */
DYNBATCH_API db_status db_batch_generate_range(const db_workload_opts* opts, int64_t first,
                                               int64_t last, db_batch** out);
/* Diagnostics: cycle accounting of the conv step kernel (64 counters):
 * [12..15] MMA thread [accumulator, window, weight waits, loop total];
 * [16..19] window producer [item ring, dependencies, free slot, total];
 * [20..21] MMA-loop cycles and nanoseconds (the kernel's own clock);
 * [24 + 4k ..] per tile kind k (0 conv1x1, 1 conv3x3 #1, 2 conv3x3 #2):
 * item cycles, window, weight, accumulator waits; [36 + 2k] epilogue
 * cycles and tiles; [42 + k] producer dependency waits. enable != 0 turns
 * accounting on for later launches. */
DYNBATCH_API db_status db_debug_conv_waits(uint64_t* out64, int32_t reset, int32_t enable);
/* Borrowing view of the batch's b × width input rows (valid until free). */
DYNBATCH_API db_status db_batch_inputs(const db_batch* batch, const double** data, int64_t* rows,
                                       int64_t* width);
/* Binds the calling thread to `device` and checks it is sm_100. */
DYNBATCH_API db_status db_device_open(int32_t device);

/* ---- IEP sessions ---- */
typedef struct db_iep_session db_iep_session;

/* Uploads programs [first, last) of `batch` (the whole batch when
 * last <= first), their inputs and the module set ModuleSet(vocab, seed). */
DYNBATCH_API db_status db_iep_session_create(const db_batch* batch, int64_t first, int64_t last,
                                             uint64_t module_seed, const db_module_opts* opts,
                                             db_iep_session** out);
/* Executes a host-built schedule (any strategy) instead of the device
 * scheduler; NULL restores the device improved scheduler. */
DYNBATCH_API db_status db_iep_session_set_schedule(db_iep_session* s, const db_schedule* schedule);
/* Strategy of the device scheduler run by every forward: IMPROVED (the
 * default), STANDARD or ONLINE (same schedules as db_schedule_build, built
 * on the device); NAIVE is DB_ERR_INVALID_ARG (load it with set_schedule). */
DYNBATCH_API db_status db_iep_session_set_strategy(db_iep_session* s, db_strategy strategy);
/* Enqueues one forward on the session stream (schedule + execute). */
DYNBATCH_API db_status db_iep_session_forward(db_iep_session* s);
/* End-to-end: pinned-host fp32 inputs (rows × width, reference row layout,
 * CHW for RESBLOCK) → H2D → forward → D2H of the root outputs (fp32). */
DYNBATCH_API db_status db_iep_session_forward_host(db_iep_session* s, const float* inputs,
                                                   float* outputs);
/* Pipelined form of …_forward_host: returns once the call is enqueued. The
 * upload of this call and the download of the previous one overlap the
 * forward (copy streams, triple-buffered device rows). The host buffers must
 * stay valid, and should be pinned, until db_iep_session_synchronize. */
DYNBATCH_API db_status db_iep_session_forward_host_async(db_iep_session* s, const float* inputs,
                                                         float* outputs);
DYNBATCH_API db_status db_iep_session_synchronize(db_iep_session* s);
/* RESBLOCK sessions: replace the programs by b prefix function sequences
 * (build_program_from_prefix order; tokens concatenated, seq_off[b+1]),
 * built into the CSR on the device. Within the session
 * capacity; an empty sequence is reported at once (DB_ERR_INVALID_ARGUMENT),
 * the device build's errors (unknown function / underfull / overfull) at the
 * next synchronize. tokens may be NULL only when seq_off[b] == 0. The next forward uses them; its inputs
 * are the next …_forward_host(_async) call's rows (b of them). */
DYNBATCH_API db_status db_iep_session_set_programs(db_iep_session* s, const int32_t* tokens,
                                                   const int32_t* seq_off, int64_t b);
DYNBATCH_API void* db_iep_session_stream(db_iep_session* s);
DYNBATCH_API db_status db_iep_session_stats(db_iep_session* s, db_session_stats_t* out);
/* Copies the device schedule of the last forward into a host handle. */
DYNBATCH_API db_status db_iep_session_schedule(db_iep_session* s, db_schedule** out);
/* Root outputs (as double, reference row layout) + integer trace. */
DYNBATCH_API db_status db_iep_session_run(db_iep_session* s, db_run** out);
/* Device level labels of the last forward (total_nodes int32, CSR order). */
DYNBATCH_API db_status db_iep_session_labels(db_iep_session* s, int32_t* labels, int64_t n);
/* Runs `iters` forwards between two CUDA events on the session stream and
 * returns the elapsed device milliseconds. profile 1 also fills per-kernel-
 * class times (direct launches, events around every launch); profile 2 runs
 * the forwards as unprofiled ones do (CUDA-graph replays) with event-record
 * nodes around the fused step kernel and fills class 4 (conv step) with that
 * kernel's own time inside the same loop (RESBLOCK sessions whose forward is
 * one step launch; launches[4] = 0 otherwise). */
DYNBATCH_API db_status db_iep_session_time(db_iep_session* s, int32_t iters, int32_t profile,
                                           double* ms, db_kernel_times_t* kt);
/* IEP classifier head on the root maps (RESBLOCK sessions; SURVEY.md §8(f)4,
 * beyond the reference, whose path ends at the root feature maps):
 * conv1x1 128 → 512 + ReLU, 2×2 max pool, FC 25088 → 1024 + ReLU,
 * FC 1024 → `answers` (≤ 256), fp16 tensor-core operands, fp32 logits.
 * Weights Rng(mix_seed(seed, 0x4ead)) as oracle/dynbatch_oracle.c
 * orc_head_weights. set_head creates (or replaces) it; head_forward enqueues
 * it on the current roots (after a forward); logits downloads b × answers
 * fp32; forward_logits_host = H2D rows → forward → head → D2H logits;
 * time_head returns device ms per head forward (CUDA events). */
DYNBATCH_API db_status db_iep_session_set_head(db_iep_session* s, int32_t answers, uint64_t seed);
DYNBATCH_API db_status db_iep_session_head_forward(db_iep_session* s);
DYNBATCH_API db_status db_iep_session_logits(db_iep_session* s, float* out, int64_t n);
DYNBATCH_API db_status db_iep_session_forward_logits_host(db_iep_session* s, const float* inputs,
                                                          float* logits);
DYNBATCH_API db_status db_iep_session_time_head(db_iep_session* s, int32_t iters, double* ms,
                                                double* flops);
/* Training (RESBLOCK sessions with a head, beyond the
 * reference's forward-only path): set_training(1) keeps every node's fp32
 * value during training forwards. train_step runs forward → head → mean
 * softmax cross-entropy over labels[b] (in [0, answers)) → backward through
 * the head and the module groups in reverse step order, and returns the
 * loss. grad downloads one fp32 gradient of that step: which 0-5 = module
 * w0, b0, w1, b1, w2, b2 of function fid (input-major like the weights),
 * 6-11 = head wp, bp, w1, b1, w2, b2, 12 = the input maps (CHW rows);
 * grad_size gives its element count. time_train = device ms per step. */
DYNBATCH_API db_status db_iep_session_set_training(db_iep_session* s, int32_t on);
DYNBATCH_API db_status db_iep_session_train_step(db_iep_session* s, const int32_t* labels, float* loss);
DYNBATCH_API db_status db_iep_session_grad_size(db_iep_session* s, int32_t which, int32_t fid, int64_t* n);
DYNBATCH_API db_status db_iep_session_grad(db_iep_session* s, int32_t which, int32_t fid, float* out, int64_t n);
/* SGD with the last train_step's gradients: every module weight and bias and
 * the head's, w -= lr·g on fp32 masters, then the forward's fp16 operand
 * layouts rebuilt on the device (the next forward / train_step uses them). */
DYNBATCH_API db_status db_iep_session_sgd(db_iep_session* s, float lr);
DYNBATCH_API db_status db_iep_session_time_train(db_iep_session* s, int32_t iters, const int32_t* labels,
                                                 double* ms);
DYNBATCH_API void db_iep_session_free(db_iep_session* s);

/* db_schedule_build on the device scheduler: IMPROVED, STANDARD or ONLINE
 * (bit-identical to the host builders; sched.cu); NAIVE is DB_ERR_INVALID_ARG. */
DYNBATCH_API db_status db_schedule_build_device(const db_batch* batch, db_strategy strategy, db_schedule** out);
/* db_execute with a module kind; schedule NULL = device improved scheduler. */
DYNBATCH_API db_status db_execute_device(const db_batch* batch, const db_schedule* schedule,
                                         uint64_t module_seed, const db_module_opts* opts,
                                         db_run** out);

/* ---- MoE sessions ---- */
typedef struct db_moe_session db_moe_session;

/* Generates inputs/scores (gen_moe_inputs) and experts (ExpertSet with
 * mix_seed(seed, 0xe4be27)) exactly as db_moe_run does and uploads them.
 * Tokens [first, last) are kept (all when last <= first). */
DYNBATCH_API db_status db_moe_session_create(const db_moe_opts* opts, int32_t precision,
                                             int64_t first, int64_t last, db_moe_session** out);
DYNBATCH_API db_status db_moe_session_forward(db_moe_session* s);
/* End-to-end: host fp32 inputs [T×d] and fp64 scores [T×n] → outputs fp32. */
DYNBATCH_API db_status db_moe_session_forward_host(db_moe_session* s, const float* inputs,
                                                   const double* scores, float* outputs);
/* Pipelined form (pinned host buffers, three calls in flight, uploads and
 * downloads on their own streams overlapping the neighbouring calls'
 * forwards); the buffers stay in use until db_moe_session_synchronize. */
DYNBATCH_API db_status db_moe_session_forward_host_async(db_moe_session* s, const float* inputs,
                                                         const double* scores, float* outputs);
DYNBATCH_API db_status db_moe_session_synchronize(db_moe_session* s);
DYNBATCH_API void* db_moe_session_stream(db_moe_session* s);
DYNBATCH_API db_status db_moe_session_stats(db_moe_session* s, db_session_stats_t* out);
/* Routing of the last forward: ids[T×k], weights[T×k], expert_offsets[n+1],
 * sorted items[T×k] (token·k + slot in per-expert (token, slot) order). */
DYNBATCH_API db_status db_moe_session_routing(db_moe_session* s, int32_t* ids, double* weights,
                                              int32_t* expert_offsets, int32_t* items);
DYNBATCH_API db_status db_moe_session_run(db_moe_session* s, db_run** out);
/* Output rows rows[0..n_rows) of the last forward as fp32 [n_rows×d] (rows
 * NULL: the first n_rows) — a sample of a layer too large to download. */
DYNBATCH_API db_status db_moe_session_outputs(db_moe_session* s, const int64_t* rows, int64_t n_rows,
                                              float* out);
DYNBATCH_API db_status db_moe_session_time(db_moe_session* s, int32_t iters, int32_t profile,
                                           double* ms, db_kernel_times_t* kt);
DYNBATCH_API void db_moe_session_free(db_moe_session* s);

/* ---- expert-parallel MoE (one rank of G) ----
 * Tokens [rank·T/G, (rank+1)·T/G) and experts [rank·n/G, (rank+1)·n/G) of
 * the db_moe_run fixtures; tcgen05 grouped GEMMs with 16-bit operands
 * (precision DB_MOE_FP16 or DB_MOE_BF16; rows exchanged in that format).
 * One forward:
 *   dispatch: gate → stable expert sort → the rank's k·T/G rows packed in
 *             sorted order into send_rows (device 16-bit [items][d]);
 *             expert_counts[n] (host) = rows per global expert, so the rows
 *             for rank q are the contiguous block of q's experts;
 *   (caller) all-to-all of the counts and an all-to-allv of the rows;
 *   experts:  recv_rows = every source's block in rank order, recv_counts
 *             [G][n/G] (host; source × local expert); ret_rows (device 16-bit)
 *             receives the expert outputs in receive order;
 *   (caller) the reverse all-to-allv (ret_rows → the senders);
 *   combine:  ret_rows = this rank's rows back in its sorted order → the
 *             slot-order weighted sum (outputs fp32 [T/G][d]).
 * Kernels run on db_moe_ep_stream(). */
typedef struct db_moe_ep_session db_moe_ep_session;
DYNBATCH_API db_status db_moe_ep_create(const db_moe_opts* opts, int32_t precision, int32_t rank,
                                        int32_t world, db_moe_ep_session** out);
DYNBATCH_API db_status db_moe_ep_sizes(db_moe_ep_session* s, int64_t* tokens, int64_t* items,
                                       int32_t* local_experts);
DYNBATCH_API db_status db_moe_ep_dispatch(db_moe_ep_session* s, void* send_rows, int32_t* expert_counts);
DYNBATCH_API db_status db_moe_ep_experts(db_moe_ep_session* s, const void* recv_rows, const int32_t* recv_counts,
                                         void* ret_rows);
/* db_moe_ep_experts in pieces, for exchanges chunked by expert: the layout
 * from recv_counts once, then contiguous local-expert ranges [e_begin,
 * e_end) as their rows arrive (recv_rows / ret_rows as for _experts; each
 * call reads and writes only its experts' rows). */
DYNBATCH_API db_status db_moe_ep_layout(db_moe_ep_session* s, const int32_t* recv_counts);
/* World 1 only: the whole layer in one device pass (gate, sort, dispatch,
 * grouped GEMMs, combine), no exchange buffers. */
DYNBATCH_API db_status db_moe_ep_forward_local(db_moe_ep_session* s);
DYNBATCH_API db_status db_moe_ep_experts_range(db_moe_ep_session* s, const void* recv_rows, void* ret_rows,
                                               int32_t e_begin, int32_t e_end);
DYNBATCH_API db_status db_moe_ep_combine(db_moe_ep_session* s, const void* ret_rows);
/* The whole layer with the exchange inside the library, on NCCL over
 * NVLink: rank 0 makes a 128-byte id (db_moe_ep_nccl_id), the caller passes
 * it to every rank out of band, each rank joins (db_moe_ep_comm_init), then
 * db_moe_ep_forward runs gate → sort → count all-to-all → pack → per
 * expert range: rows out, grouped GEMMs, rows back → combine, the exchange
 * of range c+1 overlapping the GEMMs of range c (chunks ranges; 1 = no
 * overlap). At world 1 without a communicator it is forward_local.
 * NCCL (libnccl.so.2) is loaded at the first of these calls. */
DYNBATCH_API db_status db_moe_ep_nccl_id(void* unique_id /* 128 bytes */);
DYNBATCH_API db_status db_moe_ep_comm_init(db_moe_ep_session* s, const void* unique_id);
DYNBATCH_API db_status db_moe_ep_forward(db_moe_ep_session* s, int32_t chunks);
/* Rows this rank's experts received in the last forward. */
DYNBATCH_API db_status db_moe_ep_recv_rows(db_moe_ep_session* s, int64_t* rows);
/* The exchange plan (host only): send_counts[G·E] (rows this rank sends per
 * global expert), recv_counts[G][E] (rows each source sends per local
 * expert) → *n_chunks = C expert ranges and, per range c and peer q
 * ([C][G], caller-sized for min(chunks, E) ranges), the row offset and
 * count of the send piece and of the receive piece. */
DYNBATCH_API db_status db_moe_ep_plan(int32_t G, int32_t E, const int32_t* send_counts, const int32_t* recv_counts,
                                      int32_t chunks, int32_t* n_chunks, int64_t* send_off, int64_t* send_rows,
                                      int64_t* recv_off, int64_t* recv_rows);
DYNBATCH_API db_status db_moe_ep_outputs(db_moe_ep_session* s, float* out);
DYNBATCH_API db_status db_moe_ep_synchronize(db_moe_ep_session* s);
DYNBATCH_API void* db_moe_ep_stream(db_moe_ep_session* s);
DYNBATCH_API void db_moe_ep_free(db_moe_ep_session* s);

/* db_moe_run with a precision (batched only). */
DYNBATCH_API db_status db_moe_run_device(const db_moe_opts* opts, int32_t precision,
                                         db_run** out);

#ifdef __cplusplus
}
#endif

#endif /* DYNBATCH_DYNBATCH_DEVICE_H */
