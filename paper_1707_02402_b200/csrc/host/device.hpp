// device.hpp — host-side orchestration of the device path (internal).
//
// Owns device memory, the session stream and the per-forward launch
// sequence. Everything crosses into CUDA through the dbk_* C-ABI
// (include/dynbatch/dbk.h); no CUDA types leak into the public headers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <span>
#include <vector>

#include "dynbatch.hpp"

namespace dynbatch::dev {

// Throws std::runtime_error (→ DB_ERR_INTERNAL) with the CUDA error text.
void check(cudaError_t e, const char* what);
inline void check(int e, const char* what) { check(static_cast<cudaError_t>(e), what); }
// Verifies a CUDA device is present and is an sm_100 part; there is no CPU
// fallback, so every compute entry point calls this first.
void require_device();
int sm_count();

template <class T>
class Buf {
 public:
  Buf() = default;
  explicit Buf(size_t n) { alloc(n); }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  Buf(Buf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  Buf& operator=(Buf&& o) noexcept {
    if (this != &o) { release(); p_ = o.p_; n_ = o.n_; o.p_ = nullptr; o.n_ = 0; }
    return *this;
  }
  ~Buf() { release(); }
  void alloc(size_t n) {
    release();
    if (n == 0) n = 1;
    check(cudaMalloc(reinterpret_cast<void**>(&p_), n * sizeof(T)), "cudaMalloc");
    n_ = n;
  }
  void ensure(size_t n) { if (n > n_ || !p_) alloc(n); }
  void upload(const T* src, size_t n, cudaStream_t s) {
    ensure(n);
    if (n) check(cudaMemcpyAsync(p_, src, n * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
  }
  void upload(const std::vector<T>& v, cudaStream_t s) { upload(v.data(), v.size(), s); }
  void zero(cudaStream_t s) { if (p_) check(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s), "memset"); }
  std::vector<T> download(size_t n, cudaStream_t s) const {
    std::vector<T> out(n);
    if (n) check(cudaMemcpyAsync(out.data(), p_, n * sizeof(T), cudaMemcpyDeviceToHost, s), "D2H");
    check(cudaStreamSynchronize(s), "sync");
    return out;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* p_ = nullptr;
  size_t n_ = 0;
};

// Page-locked host array (grow-only), for copies that overlap compute.
template <typename T>
class Pinned {
 public:
  Pinned() = default;
  Pinned(const Pinned&) = delete;
  Pinned& operator=(const Pinned&) = delete;
  ~Pinned() {
    if (p_) cudaFreeHost(p_);
  }
  void ensure(size_t n) {
    if (n <= n_) return;
    if (p_) cudaFreeHost(p_);
    p_ = nullptr;
    n_ = 0;
    check(cudaHostAlloc(reinterpret_cast<void**>(&p_), sizeof(T) * std::max<size_t>(n, 1), cudaHostAllocPortable),
          "cudaHostAlloc");
    n_ = n;
  }
  T* get() const { return p_; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

// Per-kernel-class timing with CUDA events around launches (mirrors
// db_kernel_times_t). Events are pooled; results are read after a sync.
struct KernelTimes {
  double ms[8] = {};
  std::int64_t launches[8] = {};
  double flops[8] = {};
  double bytes[8] = {};
};

class Profiler {
 public:
  ~Profiler();
  bool on = false;
  void reset() { recs_.clear(); used_ = 0; }
  void begin(int cls, cudaStream_t s);
  void end(cudaStream_t s);
  void add_work(int cls, double flops, double bytes) { work_flops_[cls] += flops; work_bytes_[cls] += bytes; }
  KernelTimes collect();

 private:
  cudaEvent_t next_event();
  struct Rec { int cls; cudaEvent_t a, b; };
  std::vector<Rec> recs_;
  std::vector<cudaEvent_t> pool_;
  size_t used_ = 0;
  double work_flops_[8] = {};
  double work_bytes_[8] = {};
};

// Batch in CSR form (global node g = prog_off[e] + local id).
struct HostCSR {
  std::int64_t b = 0, N = 0;
  int p = 0, max_arity = 0, s_max = 0;
  // Allocation capacities (≥ b, N, s_max): a session can take later batches
  // up to these sizes (IepSession::set_programs).
  std::int64_t cap_b = 0, cap_N = 0;
  int cap_s = 0;
  std::vector<std::int32_t> prog_off, fid, child_off, child_list, child0, child1, example, root_g;
  std::vector<std::int32_t> arity_of, expensive_of;
};
HostCSR make_csr(std::span<const Program> programs, const FunctionVocab& vocab);

// Device copy of the CSR plus the device scheduler (labels + stable bucket
// sort) and the schedule tables it writes (or that a host schedule fills).
class DeviceProgramBatch {
 public:
  DeviceProgramBatch(const HostCSR& csr, cudaStream_t s);
  const HostCSR& csr() const { return csr_; }

  // Replaces the programs by b prefix function sequences (host arrays),
  // built into the CSR on the device (dbk_build_prefix); within capacity.
  // Build errors surface at the next resolve(). The host CSR arrays go stale
  // (sizes stay current) until replace_host_csr().
  void set_prefix_programs(const std::int32_t* tokens, const std::int32_t* seq_off, std::int64_t b, cudaStream_t s);
  // The same in two halves, for callers that upload the sequences
  // themselves: host checks + new sizes (returns the node count), then the
  // device build from device copies of the sequences.
  std::int64_t begin_prefix_programs(const std::int32_t* seq_off, std::int64_t b);
  void build_prefix_programs(const std::int32_t* tokens_dev, const std::int32_t* seq_off_dev, cudaStream_t s);
  void replace_host_csr(const HostCSR& csr);
  Buf<std::int32_t> fwd_ok;  // expensive node with one parent (written by the prefix build)

  // Device improved scheduler; returns the step count (one small D2H), or,
  // with upper_bound, s_max without a host sync (empty trailing steps).
  // strategy: improved (default), standard or online — the same bucket
  // sort over per-strategy labels; naive stays host-built.
  int run_scheduler(cudaStream_t s, bool upper_bound = false, Strategy strategy = Strategy::improved);
  void check_scheduler_error(cudaStream_t s) const;
  // Installs a host-built schedule in the same table format.
  int load_schedule(const Schedule& schedule, cudaStream_t s);
  Schedule download_schedule(Strategy strategy, cudaStream_t s) const;
  std::vector<std::int32_t> download_labels(cudaStream_t s) const { return labels.download(csr_.N, s); }
  ExecutionTrace trace_counts(cudaStream_t s) const;

  // Group count of the last schedule (the device scheduler's value is read
  // lazily: a static-shape schedule needs no host sync).
  std::int64_t group_count(cudaStream_t s) const;
  bool static_shape() const { return shape_n_ > 0; }

  void resolve(cudaStream_t s) const;

  // Host bookkeeping a forward leaves behind (step count, pending reads):
  // restored when a captured forward is replayed.
  struct SchedState {
    int steps;
    std::int64_t groups;
    bool groups_pending, errors_pending;
  };
  SchedState sched_state() const { return {steps, groups, groups_pending_, errors_pending_}; }
  void set_sched_state(const SchedState& st) const {
    steps = st.steps;
    groups = st.groups;
    groups_pending_ = st.groups_pending;
    errors_pending_ = st.errors_pending;
  }

  mutable int steps = 0;
  mutable std::int64_t groups = 0;
  Buf<std::int32_t> prog_off, fid, child_off, child_list, child0, child1, example, root_g;
  Buf<std::int32_t> arity_of, labels, scratch, scalars, seg_hist;
  Buf<std::int32_t> member_g, group_fid, group_begin, step_group_begin;

 private:
  void detect_static_shape(cudaStream_t s);
  HostCSR csr_;
  int max_keys_ = 0;
  mutable bool groups_pending_ = false;
  mutable bool errors_pending_ = false;
  mutable bool build_pending_ = false;  // a device prefix build's error flag is unread
  Buf<std::int32_t> tokens_dev_, seq_off_dev_, build_err_;
  Buf<std::int64_t> build_stack_;
  int shape_n_ = 0, shape_dmax_ = 0;  // programs share one tree shape (static schedule)
  Buf<std::int32_t> shape_labels_;
};

enum class ModuleKind { dense = 0, resblock = 1 };

class IepHead;

class IepSession {
 public:
  // cap_* (0: the initial batch's size) bound the batches set_programs accepts.
  IepSession(const FunctionVocab& vocab, std::span<const Program> programs,
             const TensorBatch& inputs, std::uint64_t module_seed, ModuleKind kind,
             std::int64_t cap_programs = 0, std::int64_t cap_nodes = 0, int cap_length = 0);
  ~IepSession();

  // Resblock sessions: replace the programs by b prefix function sequences
  // (concatenated tokens, seq_off[b+1]), built into the CSR on the device;
  // the next forward schedules and executes them. Inputs come with the next
  // forward_host / forward_host_async call.
  void set_programs(const std::int32_t* tokens, const std::int32_t* seq_off, std::int64_t b);

  void set_schedule(const Schedule* schedule);
  void set_strategy(Strategy strategy);  // device scheduler strategy (improved / standard / online)
  void forward();
  void forward_host(const float* inputs, float* outputs);
  void forward_host_async(const float* inputs, float* outputs);
  void sync_pipeline();
  void ensure_host_mirror();  // host CSR arrays of programs set on the device
  void synchronize();
  cudaStream_t stream() const { return stream_; }

  Schedule download_schedule();
  std::vector<std::int32_t> download_labels();
  TensorBatch download_outputs();
  // Output rows rows[0..n_rows) (rows NULL: 0..n_rows) as fp32.
  void download_rows(const std::int64_t* rows, std::int64_t n_rows, float* out);
  ExecutionTrace trace();
  std::int64_t launches() const { return launches_; }
  double algorithmic_flops() const;
  double algorithmic_bytes() const;
  const HostCSR& csr() const { return batch_->csr(); }
  int width() const { return width_; }
  ModuleKind kind() const { return kind_; }
  std::int64_t h2d_bytes() const;
  std::int64_t d2h_bytes() const;
  // profile 0: elapsed only; 1: events around every launch (direct
  // launches, per-class times); 2: the forwards as they run unprofiled
  // (graph replays) with event-record nodes around the fused step kernel, so
  // class 4 holds that kernel's own time inside the same loop.
  double time_forwards(int iters, int profile, KernelTimes* kt);
  // IEP classifier head on the root maps (iep_head.hpp; resblock sessions).
  void set_head(int answers, std::uint64_t seed);
  void head_forward();                                   // logits of the current roots
  void download_logits(float* out, std::int64_t n);      // n = b · answers
  void forward_logits_host(const float* inputs, float* logits);  // H2D rows → forward → head → D2H logits
  double time_head(int iters);                           // ms per head forward (events, session stream)
  double head_flops() const;                             // per head forward of the current batch
  int head_answers() const;
  // Training (iep_train.cpp; resblock sessions with a head): one step =
  // training forward (every node value kept) → head → mean softmax
  // cross-entropy over labels[b] → backward through the head and the module
  // groups in reverse step order. Gradients are fp32, input-major like the
  // weights; they are overwritten by every step.
  struct Train;  // iep_train.hpp
  void set_training(bool on);
  float train_step(const std::int32_t* labels);
  // which: 0-5 = module w0, b0, w1, b1, w2, b2 of function fid; 6-11 = head
  // wp, bp, w1, b1, w2, b2; 12 = input maps (CHW rows [b][C·196]).
  void download_grad(int which, int fid, float* out, std::int64_t n);
  std::int64_t grad_size(int which, int fid) const;
  double time_train(int iters, const std::int32_t* labels);
  // SGD with the last train_step's gradients: every module and head weight
  // and bias (fp32 masters) w -= lr·g, then the forward's fp16 operand
  // layouts rebuilt from them on the device.
  void sgd_update(float lr);

 private:
  FunctionVocab vocab_;
  std::vector<std::int32_t> host_tokens_, host_seq_off_;
  bool mirror_stale_ = false;
  void forward_dense();
  void forward_resblock();
  void check_errors();
  void flush_programs();                       // builds sequences staged by a pipelined set_programs
  void forward_direct();                       // enqueue one forward launch by launch
  // CUDA graphs of whole resblock forwards, keyed by what their launches
  // depend on (sizes, strategy, tile size, kernel variant): a replay costs one
  // launch instead of ~20 dependent ones.
  struct GraphKey {
    std::int64_t b, N, n_shared;
    int s_max, strategy, host_schedule, tile_m, static_shape, debug, kevents;
    std::uint64_t gen;
    bool operator==(const GraphKey&) const = default;
  };
  struct CachedGraph {
    GraphKey key;
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;                 // kept when kb / ke are set
    cudaGraphNode_t kb = nullptr, ke = nullptr;  // event records around the step kernel
    DeviceProgramBatch::SchedState sched;
    std::int64_t launches = 0;
    std::uint64_t used = 0;
  };
  std::vector<CachedGraph> graphs_;
  std::uint64_t graph_clock_ = 0, schedule_gen_ = 0;
  // time_forwards(profile 2): events recorded around the one-launch step
  // kernel of each forward (kev_cur_, set per forward; placeholders kev_mark_
  // while a graph is captured, then the exec's nodes are pointed at kev_cur_)
  bool kevents_ = false, kev_recorded_ = false;
  cudaEvent_t kev_cur_[2] = {nullptr, nullptr}, kev_mark_[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> kev_pool_;
  void release_graph(CachedGraph& g);
  bool graphs_enabled() const;
  void forward_graph();
  void programs_built();                       // session state that follows a device prefix build
  void init_resblock(const TensorBatch& inputs, std::uint64_t module_seed);
  void upload_resblock_inputs(const float* chw_rows);
  void download_resblock_outputs(float* chw_rows);

  ModuleKind kind_;
  int width_ = 0;
  cudaStream_t stream_ = nullptr;
  std::unique_ptr<DeviceProgramBatch> batch_;
  bool host_schedule_ = false;
  Strategy strategy_ = Strategy::improved;
  std::int64_t launches_ = 0;
  Buf<std::int32_t> err_;
  Buf<std::int32_t> present_;
  // dense
  Buf<double> in64_, values64_, out64_;
  std::vector<Buf<double>> w64_;
  Buf<const double*> wtab_, btab_;
  // resblock
  struct RB;
  std::unique_ptr<RB> rb_;
  std::unique_ptr<IepHead> head_;
  std::unique_ptr<Train> train_;
  bool train_fwd_ = false;  // the forward in flight is a training step's (dbk_rb_plan / dbk_rb_step training)
  std::uint64_t module_seed_ = 0;
  void backward(float* loss_dev);
  void require_head() const;
  Profiler prof_;
  void add_forward_work();
};

// MoE session (fp64 reference order, or fp16 / bf16 tensor-core grouped GEMMs).
class MoeSession {
 public:
  MoeSession(const MoeConfig& cfg, std::uint64_t seed, int precision, std::int64_t first,
             std::int64_t last);
  ~MoeSession();
  void forward();
  void forward_host(const float* inputs, const double* scores, float* outputs);
  // Pipelined host call: returns once queued; the pinned buffers must stay
  // untouched until synchronize() (three calls in flight, copies on their
  // own streams overlapping the neighbouring calls' forwards).
  void forward_host_async(const float* inputs, const double* scores, float* outputs);
  void synchronize();
  cudaStream_t stream() const { return stream_; }
  void routing(std::int32_t* ids, double* weights, std::int32_t* offsets, std::int32_t* items);
  TensorBatch download_outputs();
  // Output rows rows[0..n_rows) (rows NULL: 0..n_rows) as fp32.
  void download_rows(const std::int64_t* rows, std::int64_t n_rows, float* out);
  ExecutionTrace trace();
  std::int64_t launches() const { return launches_; }
  double algorithmic_flops() const;
  double algorithmic_bytes() const;
  std::int64_t tokens() const { return T_; }
  std::int64_t h2d_bytes() const;
  std::int64_t d2h_bytes() const;
  double time_forwards(int iters, bool profile, KernelTimes* kt);
  Profiler prof_;

 private:
  void forward_from(const float* x, const double* scores, float* out);   // a cached graph replay when enabled
  void forward_direct(const float* x, const double* scores, float* out);
  struct Impl;
  std::unique_ptr<Impl> impl_;
  cudaStream_t stream_ = nullptr;
  std::int64_t T_ = 0;
  std::int64_t launches_ = 0;
};

// Expert-parallel MoE rank: tokens [rank·T/G, (rank+1)·T/G),
// experts [rank·n/G, (rank+1)·n/G), 16-bit tcgen05 grouped GEMMs. forward()
// runs the whole layer with the exchange on the library's own NCCL
// communicator; the staged calls (dispatch / experts / combine) leave the
// exchange to the caller.
class MoeEp {
 public:
  MoeEp(const MoeConfig& cfg, std::uint64_t seed, int precision, int rank, int world);
  ~MoeEp();
  std::int64_t tokens() const { return T_; }
  std::int64_t items() const;
  int local_experts() const;
  // gate → stable expert sort → rows packed in sorted order into `send`
  // (device bf16 [items][d]); expert_counts[n] (host) = rows per expert.
  void dispatch(void* send, std::int32_t* expert_counts);
  // recv = rows received from every source (rank order, expert-major),
  // cnt[G][E_local] (host); ret (device bf16) gets the expert outputs in
  // receive order.
  void experts(const void* recv, const std::int32_t* cnt, void* ret);
  // The same in pieces, for exchanges chunked by expert: layout(cnt) once,
  // then experts_range for contiguous local-expert ranges, each as soon as
  // its rows have arrived (rows of other experts may still be in flight).
  void layout(const std::int32_t* cnt);
  // World 1: the whole layer in one device pass (no exchange, no pack).
  void forward_local();
  // NCCL communicator of the G ranks (ncclCommInitRank; the 128-byte unique
  // id comes from rank 0's nccl_unique_id, passed out of band).
  void comm_init(const void* unique_id);
  // One forward with the exchange on NCCL, local experts cut into `chunks`
  // ranges whose transfers overlap the GEMMs (world 1 without a
  // communicator: forward_local).
  void forward(int chunks);
  std::int64_t last_recv_rows() const { return last_recv_rows_; }
  void experts_range(const void* recv, void* ret, int e_begin, int e_end);
  // ret_recv = the rank's own rows back, in its sorted order → outputs.
  void combine(const void* ret_recv);
  void download_outputs(float* out);
  void synchronize();
  cudaStream_t stream() const { return stream_; }
  Profiler prof_;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
  cudaStream_t stream_ = nullptr;
  std::int64_t T_ = 0;
  std::int64_t last_recv_rows_ = 0;
};

}  // namespace dynbatch::dev
