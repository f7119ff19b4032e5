// moe_device.cpp — MoE layer on the device (host orchestration).
//
// Forward = top-k gate (dbk_moe_topk) → stable expert sort of the k·T
// assignments in (token, slot) order (dbk_stable_bucket_sort; the reference
// group_by_function, src/schedule.cpp:166-169 via src/moe.cpp:214-224) →
// grouped expert application → slot-order combine.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <thread>

#include "device.hpp"
#include "dynbatch/dbk.h"
#include "ep_nccl.hpp"
#include "moe_bf16.hpp"

namespace dynbatch {
namespace dev {

struct MoeDev {
  std::int64_t T = 0;
  int n = 0, k = 0, d = 0, h = 0;
  Buf<double> x, scores, wts, hidden, staged, out;
  Buf<std::int32_t> ids, order, offsets, seg_hist, tiles, err;
  std::vector<Buf<double>> w;  // per expert: w1 | w2
  Buf<const double*> w1tab, w2tab;

  void alloc(std::int64_t T_, int n_, int k_, int d_, int h_) {
    T = T_; n = n_; k = k_; d = d_; h = h_;
    const size_t items = static_cast<size_t>(T) * static_cast<size_t>(k);
    scores.alloc(static_cast<size_t>(T) * n);
    wts.alloc(items);
    ids.alloc(items);
    order.alloc(items);
    offsets.alloc(static_cast<size_t>(n) + 1);
    seg_hist.alloc(static_cast<size_t>(dbk_bucket_sort_scratch(static_cast<std::int64_t>(items), n)));
    tiles.alloc(static_cast<size_t>(n) + 1);
    err.alloc(4);
    // read by check_err (synchronize) before the first gate resets it: a
    // fresh allocation can hold a freed buffer's bytes
    check(cudaMemset(err.get(), 0, 16), "memset");
  }
  void alloc_fp64_work() {
    const size_t items = static_cast<size_t>(T) * static_cast<size_t>(k);
    x.alloc(static_cast<size_t>(T) * d);
    hidden.alloc(items * static_cast<size_t>(h));
    staged.alloc(items * static_cast<size_t>(d));
    out.alloc(static_cast<size_t>(T) * d);
  }
  void upload_experts(const ExpertSet& experts, cudaStream_t s) {
    w.resize(static_cast<size_t>(n));
    std::vector<const double*> t1(static_cast<size_t>(n)), t2(static_cast<size_t>(n));
    for (int e = 0; e < n; ++e) {
      const Expert& ex = experts.expert(e);
      Buf<double>& b = w[static_cast<size_t>(e)];
      b.alloc(ex.w1.size() + ex.w2.size());
      check(cudaMemcpyAsync(b.get(), ex.w1.data(), ex.w1.size() * 8, cudaMemcpyHostToDevice, s), "H2D w1");
      check(cudaMemcpyAsync(b.get() + ex.w1.size(), ex.w2.data(), ex.w2.size() * 8, cudaMemcpyHostToDevice, s), "H2D w2");
      t1[static_cast<size_t>(e)] = b.get();
      t2[static_cast<size_t>(e)] = b.get() + ex.w1.size();
    }
    w1tab.upload(t1, s);
    w2tab.upload(t2, s);
  }
  void gate(cudaStream_t s, const double* sc = nullptr) {
    check(cudaMemsetAsync(err.get(), 0, 16, s), "memset");
    check(dbk_moe_topk(T, n, k, sc ? sc : scores.get(), ids.get(), wts.get(), err.get(), s), "dbk_moe_topk");
  }
  void sort(cudaStream_t s) {
    check(dbk_stable_bucket_sort(T * k, n, ids.get(), seg_hist.get(), order.get(), offsets.get(), s),
          "dbk_stable_bucket_sort");
  }
  void experts_fp64(cudaStream_t s) {
    check(dbk_moe_expert_fp64(T, n, k, d, h, order.get(), offsets.get(), x.get(), w1tab.get(),
                              w2tab.get(), hidden.get(), staged.get(), tiles.get(), s),
          "dbk_moe_expert_fp64");
  }
  void combine_fp64(cudaStream_t s) {
    check(dbk_moe_combine_fp64(T, k, d, wts.get(), staged.get(), out.get(), s), "dbk_moe_combine_fp64");
  }
  void check_err(cudaStream_t s) {
    std::int32_t e = 0;
    check(cudaMemcpyAsync(&e, err.get(), 4, cudaMemcpyDeviceToHost, s), "D2H");
    check(cudaStreamSynchronize(s), "sync");
    if (e == 9) throw_error(Errc::non_finite_value, "non-finite gate score");
    if (e) throw std::runtime_error("device MoE error " + std::to_string(e));
  }
  ExecutionTrace trace(cudaStream_t s) {
    ExecutionTrace t;
    t.per_function_calls.assign(static_cast<size_t>(n), 0);
    const auto off = offsets.download(static_cast<size_t>(n) + 1, s);
    for (int e = 0; e < n; ++e) {
      const std::int64_t rows = off[static_cast<size_t>(e) + 1] - off[static_cast<size_t>(e)];
      if (rows == 0) continue;
      ++t.expensive_calls;
      ++t.per_function_calls[static_cast<size_t>(e)];
      t.peak_group_rows = std::max(t.peak_group_rows, rows);
    }
    t.per_step_seconds.assign(1, 0.0);
    return t;
  }
};

namespace {
cudaStream_t make_stream() {
  cudaStream_t s = nullptr;
  check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  return s;
}
struct StreamGuard {
  cudaStream_t s;
  ~StreamGuard() { if (s) { cudaStreamSynchronize(s); cudaStreamDestroy(s); } }
};

// Rows [first, last) of random_batch(·, width, seed) (src/workload.cpp:207-212)
// generated straight into device memory in 32 MB host chunks, as V: the
// values are the reference's doubles (fp32 inputs are their rounding), and
// no full-size host copy exists (cfg5: 17 GB of fp64 inputs).
template <typename V>
void upload_random_rows(V* dst, std::int64_t first, std::int64_t last, std::int64_t width, std::uint64_t seed) {
  if (last <= first) return;
  Rng rng(seed);
  rng.discard(static_cast<std::uint64_t>(first) * static_cast<std::uint64_t>(width));
  const std::int64_t chunk = std::max<std::int64_t>(1, (std::int64_t{32} << 20) / (width * static_cast<std::int64_t>(sizeof(V))));
  std::vector<V> buf(static_cast<size_t>(std::min(chunk, last - first) * width));
  for (std::int64_t r = first; r < last; r += chunk) {
    const std::int64_t nr = std::min(chunk, last - r);
    const size_t n = static_cast<size_t>(nr * width);
    for (size_t i = 0; i < n; ++i) buf[i] = static_cast<V>(rng.uniform(-1.0, 1.0));
    check(cudaMemcpy(dst + (r - first) * width, buf.data(), n * sizeof(V), cudaMemcpyHostToDevice), "H2D rows");
  }
}

// gen_moe_inputs (src/workload.cpp:248-254) for tokens [first, last): scores
// (fp64) and inputs (fp64 or fp32) on two host threads (independent streams).
template <typename X>
void upload_moe_inputs(const MoeConfig& cfg, std::uint64_t seed, std::int64_t first, std::int64_t last,
                       double* scores, X* x) {
  std::exception_ptr err;
  std::thread t([&] {
    try {
      upload_random_rows(scores, first, last, cfg.experts, mix_seed(seed, 0x11ULL));
    } catch (...) {
      err = std::current_exception();
    }
  });
  upload_random_rows(x, first, last, cfg.data_dim, mix_seed(seed, 0x10ULL));
  t.join();
  if (err) std::rethrow_exception(err);
}
}  // namespace

// ------------------------------------------------------------ MoeSession
struct MoeSession::Impl {
  MoeConfig cfg;
  int precision = 0;
  MoeDev dev;
  std::unique_ptr<MoeBf16> bf16;
  // Pipelined host calls (forward_host_async): kDepth calls in flight, each
  // with its own device input / score / output slots; uploads on h2d,
  // downloads on d2h, so call i's forward overlaps call i+1's upload and
  // call i−1's download (full-duplex PCIe).
  struct Pipe {
    static constexpr int kDepth = 3;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    Buf<float> x[kDepth], out[kDepth];
    Buf<double> sc[kDepth];
    cudaEvent_t h2d_done[kDepth] = {}, in_free[kDepth] = {}, out_ready[kDepth] = {}, out_free[kDepth] = {};
    std::uint64_t calls = 0;
    ~Pipe() {
      if (h2d) cudaStreamSynchronize(h2d);
      if (d2h) cudaStreamSynchronize(d2h);
      for (int k = 0; k < kDepth; ++k)
        for (cudaEvent_t e : {h2d_done[k], in_free[k], out_ready[k], out_free[k]})
          if (e) cudaEventDestroy(e);
      if (h2d) cudaStreamDestroy(h2d);
      if (d2h) cudaStreamDestroy(d2h);
    }
  };
  std::unique_ptr<Pipe> pipe;
  // CUDA graphs of whole forwards (the ~12 dependent launches replay as one),
  // keyed by the device input / score / output pointers (the pipeline's
  // slots); a small LRU
  struct Graph {
    const float* x;
    const double* sc;
    float* out;
    cudaGraphExec_t exec = nullptr;
    std::int64_t launches = 0;
    std::uint64_t used = 0;
  };
  std::vector<Graph> graphs;
  std::uint64_t clock = 0;
  ~Impl() {
    for (Graph& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
  }
};

MoeSession::MoeSession(const MoeConfig& cfg_in, std::uint64_t seed, int precision,
                       std::int64_t first, std::int64_t last)
    : impl_(std::make_unique<Impl>()) {
  require_device();
  cfg_in.check();
  MoeConfig cfg = cfg_in;
  if (last <= first) { first = 0; last = cfg.batch; }
  if (first < 0 || last > cfg.batch) throw_error(Errc::invalid_argument, "token range out of bounds");
  T_ = last - first;
  impl_->cfg = cfg;
  if (precision < 0 || precision > 2) throw_error(Errc::invalid_argument, "unknown MoE precision");
  impl_->precision = precision;
  stream_ = make_stream();
  MoeDev& D = impl_->dev;
  D.alloc(T_, static_cast<int>(cfg.experts), static_cast<int>(cfg.active_per_example),
          static_cast<int>(cfg.data_dim), static_cast<int>(cfg.hidden));
  // Fixture generation exactly as db_moe_run (src/c_api.cpp:270-290); the
  // token slice keeps rows [first, last) of the full-batch generators.
  const std::uint64_t expert_seed = mix_seed(seed, 0xe4be27ULL);
  if (precision == 0) {
    D.alloc_fp64_work();
    upload_moe_inputs(cfg, seed, first, last, D.scores.get(), D.x.get());
    const ExpertSet experts(cfg.experts, cfg.data_dim, cfg.hidden, expert_seed);
    D.upload_experts(experts, stream_);
  } else {
    impl_->bf16 = std::make_unique<MoeBf16>(cfg, T_, expert_seed,
                                            precision == 2 ? DBK_FMT_F16 : DBK_FMT_BF16, stream_);
    upload_moe_inputs(cfg, seed, first, last, D.scores.get(), impl_->bf16->inputs_device());
  }
  check(cudaStreamSynchronize(stream_), "upload");
}

MoeSession::~MoeSession() {
  impl_.reset();
  if (stream_) {
    cudaStreamSynchronize(stream_);
    cudaStreamDestroy(stream_);
  }
}

void MoeSession::forward() { forward_from(nullptr, nullptr, nullptr); }

// DYNBATCH_GRAPH=0: direct launches (as the profiled forwards always are)
static bool moe_graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DYNBATCH_GRAPH");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

void MoeSession::forward_from(const float* x, const double* scores, float* out) {
  Impl& I = *impl_;
  if (prof_.on || !moe_graphs_enabled()) {
    forward_direct(x, scores, out);
    return;
  }
  ++I.clock;
  for (Impl::Graph& g : I.graphs) {
    if (g.x != x || g.sc != scores || g.out != out) continue;
    g.used = I.clock;
    launches_ = g.launches;
    check(cudaGraphLaunch(g.exec, stream_), "graph launch");
    return;
  }
  cudaGraph_t graph = nullptr;
  check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "begin capture");
  try {
    forward_direct(x, scores, out);
  } catch (...) {
    cudaStreamEndCapture(stream_, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  check(cudaStreamEndCapture(stream_, &graph), "end capture");
  Impl::Graph g{x, scores, out};
  const cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  check(e, "graph instantiate");
  g.launches = launches_;
  g.used = I.clock;
  constexpr size_t kMaxGraphs = 4;  // the pipeline's slots and the plain forward
  if (I.graphs.size() >= kMaxGraphs) {
    auto lru = std::min_element(I.graphs.begin(), I.graphs.end(),
                                [](const Impl::Graph& a, const Impl::Graph& b) { return a.used < b.used; });
    cudaGraphExecDestroy(lru->exec);
    I.graphs.erase(lru);
  }
  I.graphs.push_back(g);
  check(cudaGraphLaunch(g.exec, stream_), "graph launch");
}

void MoeSession::forward_direct(const float* x, const double* scores, float* out) {
  MoeDev& D = impl_->dev;
  launches_ = 0;
  prof_.begin(3, stream_);
  D.gate(stream_, scores);
  D.sort(stream_);
  prof_.end(stream_);
  launches_ += 1 + 6;  // top-k; histogram, 3-pass scan, offsets, stable scatter
  if (impl_->precision == 0) {
    prof_.begin(4, stream_);
    D.experts_fp64(stream_);
    prof_.end(stream_);
    prof_.begin(6, stream_);
    D.combine_fp64(stream_);
    prof_.end(stream_);
    launches_ += 3 + 1;
  } else {
    launches_ += impl_->bf16->forward(D.ids.get(), D.wts.get(), D.order.get(), D.offsets.get(), stream_,
                                      &prof_, x, out);
  }
  if (prof_.on) {
    const MoeConfig& c = impl_->cfg;
    const double T = static_cast<double>(T_), k = static_cast<double>(c.active_per_example);
    const double es = impl_->precision == 0 ? 8.0 : 2.0;
    const double gemm = 2.0 * T * k * c.data_dim * static_cast<double>(c.hidden);
    // class 3: scores read + routing written; the bf16 path also dispatches
    // (fp32 x rows read once, k bf16 rows written per token)
    const double dispatch = impl_->precision == 0 ? 0.0 : T * c.data_dim * 4.0 + T * k * c.data_dim * es;
    prof_.add_work(3, 0.0, T * c.experts * 8.0 + T * k * 12.0 + dispatch);
    prof_.add_work(4, gemm, T * k * c.data_dim * es + c.experts * c.data_dim * static_cast<double>(c.hidden) * es +
                                T * k * c.hidden * es);
    // GEMM2 writes Y rows (fp64 path: 8 B, bf16 path: 2 B per element)
    prof_.add_work(5, gemm, T * k * c.hidden * es + c.experts * c.data_dim * static_cast<double>(c.hidden) * es +
                                T * k * c.data_dim * es);
    // combine: k Y rows read and one fp32 (fp64) output row written per token
    prof_.add_work(6, 0.0, T * k * c.data_dim * es + T * c.data_dim * (impl_->precision == 0 ? 8.0 : 4.0));
  }
}

double MoeSession::time_forwards(int iters, bool profile, KernelTimes* kt) {
  synchronize();
  prof_.on = profile;
  prof_.reset();
  cudaEvent_t a, b;
  check(cudaEventCreate(&a), "event");
  check(cudaEventCreate(&b), "event");
  check(cudaEventRecord(a, stream_), "event");
  for (int i = 0; i < iters; ++i) forward();
  check(cudaEventRecord(b, stream_), "event");
  check(cudaEventSynchronize(b), "event sync");
  float ms = 0.f;
  check(cudaEventElapsedTime(&ms, a, b), "elapsed");
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  synchronize();
  if (profile && kt) *kt = prof_.collect();
  prof_.on = false;
  return ms;
}

void MoeSession::forward_host(const float* inputs, const double* scores, float* outputs) {
  MoeDev& D = impl_->dev;
  check(cudaMemcpyAsync(D.scores.get(), scores, sizeof(double) * static_cast<size_t>(T_) * D.n,
                        cudaMemcpyHostToDevice, stream_), "H2D scores");
  if (impl_->precision == 0) throw_error(Errc::invalid_argument, "forward_host needs a tensor-core session (DB_MOE_BF16 or DB_MOE_FP16)");
  impl_->bf16->upload_inputs(inputs, stream_);
  forward();
  impl_->bf16->download_outputs(outputs, stream_);
}

void MoeSession::forward_host_async(const float* inputs, const double* scores, float* outputs) {
  Impl& I = *impl_;
  if (I.precision == 0) throw_error(Errc::invalid_argument, "forward_host needs a tensor-core session (DB_MOE_BF16 or DB_MOE_FP16)");
  const MoeConfig& c = I.cfg;
  const size_t xb = sizeof(float) * static_cast<size_t>(T_) * c.data_dim;
  const size_t sb = sizeof(double) * static_cast<size_t>(T_) * c.experts;
  if (!I.pipe) {
    I.pipe = std::make_unique<Impl::Pipe>();
    Impl::Pipe& Q = *I.pipe;
    check(cudaStreamCreateWithFlags(&Q.h2d, cudaStreamNonBlocking), "stream");
    check(cudaStreamCreateWithFlags(&Q.d2h, cudaStreamNonBlocking), "stream");
    for (int k = 0; k < Impl::Pipe::kDepth; ++k) {
      Q.x[k].alloc(static_cast<size_t>(T_) * c.data_dim);
      Q.out[k].alloc(static_cast<size_t>(T_) * c.data_dim);
      Q.sc[k].alloc(static_cast<size_t>(T_) * c.experts);
      for (cudaEvent_t* e : {&Q.h2d_done[k], &Q.in_free[k], &Q.out_ready[k], &Q.out_free[k]}) {
        check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
        check(cudaEventRecord(*e, stream_), "event");
      }
    }
  }
  Impl::Pipe& Q = *I.pipe;
  const int k = static_cast<int>(Q.calls++ % Impl::Pipe::kDepth);
  check(cudaStreamWaitEvent(Q.h2d, Q.in_free[k]), "wait");
  check(cudaMemcpyAsync(Q.sc[k].get(), scores, sb, cudaMemcpyHostToDevice, Q.h2d), "H2D scores");
  check(cudaMemcpyAsync(Q.x[k].get(), inputs, xb, cudaMemcpyHostToDevice, Q.h2d), "H2D inputs");
  check(cudaEventRecord(Q.h2d_done[k], Q.h2d), "event");
  check(cudaStreamWaitEvent(stream_, Q.h2d_done[k]), "wait");
  check(cudaStreamWaitEvent(stream_, Q.out_free[k]), "wait");
  forward_from(Q.x[k].get(), Q.sc[k].get(), Q.out[k].get());
  check(cudaEventRecord(Q.in_free[k], stream_), "event");
  check(cudaEventRecord(Q.out_ready[k], stream_), "event");
  check(cudaStreamWaitEvent(Q.d2h, Q.out_ready[k]), "wait");
  check(cudaMemcpyAsync(outputs, Q.out[k].get(), xb, cudaMemcpyDeviceToHost, Q.d2h), "D2H outputs");
  check(cudaEventRecord(Q.out_free[k], Q.d2h), "event");
}

void MoeSession::synchronize() {
  check(cudaStreamSynchronize(stream_), "sync");
  if (impl_->pipe) {
    check(cudaStreamSynchronize(impl_->pipe->h2d), "sync");
    check(cudaStreamSynchronize(impl_->pipe->d2h), "sync");
  }
  impl_->dev.check_err(stream_);
}

void MoeSession::routing(std::int32_t* ids, double* weights, std::int32_t* offsets, std::int32_t* items) {
  synchronize();
  MoeDev& D = impl_->dev;
  const size_t nk = static_cast<size_t>(T_) * D.k;
  if (ids) check(cudaMemcpyAsync(ids, D.ids.get(), nk * 4, cudaMemcpyDeviceToHost, stream_), "D2H");
  if (weights) check(cudaMemcpyAsync(weights, D.wts.get(), nk * 8, cudaMemcpyDeviceToHost, stream_), "D2H");
  if (offsets) check(cudaMemcpyAsync(offsets, D.offsets.get(), (static_cast<size_t>(D.n) + 1) * 4, cudaMemcpyDeviceToHost, stream_), "D2H");
  if (items) check(cudaMemcpyAsync(items, D.order.get(), nk * 4, cudaMemcpyDeviceToHost, stream_), "D2H");
  check(cudaStreamSynchronize(stream_), "sync");
}

TensorBatch MoeSession::download_outputs() {
  synchronize();
  MoeDev& D = impl_->dev;
  TensorBatch out(T_, D.d);
  if (impl_->precision == 0) {
    check(cudaMemcpyAsync(out.data().data(), D.out.get(), sizeof(double) * out.data().size(),
                          cudaMemcpyDeviceToHost, stream_), "D2H");
    check(cudaStreamSynchronize(stream_), "sync");
  } else {
    std::vector<float> tmp(out.data().size());
    impl_->bf16->download_outputs(tmp.data(), stream_);
    check(cudaStreamSynchronize(stream_), "sync");
    for (size_t i = 0; i < tmp.size(); ++i) out.data()[i] = tmp[i];
  }
  if (!out.all_finite()) throw_error(Errc::non_finite_value, "non-finite output");
  return out;
}

void MoeSession::download_rows(const std::int64_t* rows, std::int64_t n_rows, float* out) {
  synchronize();
  MoeDev& D = impl_->dev;
  const size_t d = static_cast<size_t>(D.d);
  std::vector<double> tmp(impl_->precision == 0 ? d : 0);
  for (std::int64_t i = 0; i < n_rows; ++i) {
    const std::int64_t r = rows ? rows[i] : i;
    if (r < 0 || r >= T_) throw_error(Errc::invalid_argument, "output row out of range");
    if (impl_->precision == 0) {
      check(cudaMemcpy(tmp.data(), D.out.get() + static_cast<size_t>(r) * d, d * 8, cudaMemcpyDeviceToHost), "D2H");
      for (size_t j = 0; j < d; ++j) out[static_cast<size_t>(i) * d + j] = static_cast<float>(tmp[j]);
    } else {
      check(cudaMemcpy(out + static_cast<size_t>(i) * d, impl_->bf16->outputs_device() + static_cast<size_t>(r) * d,
                       d * 4, cudaMemcpyDeviceToHost), "D2H");
    }
  }
}

ExecutionTrace MoeSession::trace() { return impl_->dev.trace(stream_); }

double MoeSession::algorithmic_flops() const {
  const MoeConfig& c = impl_->cfg;
  return 4.0 * static_cast<double>(T_) * c.active_per_example * c.data_dim * static_cast<double>(c.hidden);
}

double MoeSession::algorithmic_bytes() const {
  const MoeConfig& c = impl_->cfg;
  const double es = impl_->precision == 0 ? 8.0 : 2.0;
  // scores read, inputs read, weights read once, outputs written (fp32/fp64)
  return static_cast<double>(T_) * c.experts * 8.0 + static_cast<double>(T_) * c.data_dim * es +
         2.0 * c.experts * c.data_dim * static_cast<double>(c.hidden) * es +
         static_cast<double>(T_) * c.data_dim * (impl_->precision == 0 ? 8.0 : 4.0);
}

std::int64_t MoeSession::h2d_bytes() const {
  return T_ * impl_->cfg.data_dim * 4 + T_ * impl_->cfg.experts * 8;
}
std::int64_t MoeSession::d2h_bytes() const { return T_ * impl_->cfg.data_dim * 4; }

// ----------------------------------------------------------------- MoeEp
struct MoeEp::Impl {
  MoeConfig cfg;
  int rank = 0, world = 1, E = 0, e_first = 0, sms = 148, fmt = DBK_FMT_F16;
  MoeDev dev;
  Buf<float> x, out;
  Buf<std::int32_t> pos_of_item, cnt, pstart, tile_expert, tile_rb, n_tiles, src_row, cum, recv_of_row;
  Buf<std::uint8_t> A, H;
  Buf<std::uint16_t> w1, w2, Y;  // 16-bit (fmt); Y: GEMM2 rows of the world-1 pass
  Buf<const void*> w1tab, w2tab;
  std::int64_t cap_rows = 0;  // padded-row capacity of A / H
  std::vector<std::int32_t> cnt_h;    // last layout's counts [G][E]
  std::vector<std::int64_t> pstart_h; // and its padded expert starts [E+1]
  // NCCL exchange (forward): communicator, its stream, counts, row buffers
  ncclComm_t comm = nullptr;
  cudaStream_t cs = nullptr;
  Buf<std::int32_t> send_cnt, recv_cnt;  // [n] rows per global expert sent; [G][E] received
  std::int32_t* h_cnt = nullptr;         // pinned: send [n] | recv [G·E]
  Buf<std::uint16_t> sendb, backb, recvb, retb;  // 16-bit rows: [items][d] ×2, [recv cap][d] ×2
  std::int64_t recv_cap = 0;
  std::vector<cudaEvent_t> ev;           // sorted, counts, packed, back, arrive[c]..., done[c]...

  cudaEvent_t event(size_t i) {
    while (ev.size() <= i) {
      cudaEvent_t e;
      check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      ev.push_back(e);
    }
    return ev[i];
  }
  ~Impl() {
    if (comm) Nccl::get().CommDestroy(comm);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    if (cs) cudaStreamDestroy(cs);
    if (h_cnt) cudaFreeHost(h_cnt);
  }

  void ensure_capacity(std::int64_t rows) {
    if (rows <= cap_rows) return;
    cap_rows = rows + rows / 4;
    const size_t r = static_cast<size_t>(cap_rows);
    A.alloc(r * cfg.data_dim * 2);
    H.alloc(r * cfg.hidden * 2);
    tile_expert.alloc(r / 128 + 1);
    tile_rb.alloc(r / 128 + 1);
    recv_of_row.alloc(r);
  }
};

MoeEp::MoeEp(const MoeConfig& cfg, std::uint64_t seed, int precision, int rank, int world)
    : impl_(std::make_unique<Impl>()) {
  require_device();
  cfg.check();
  if (precision != 1 && precision != 2)
    throw_error(Errc::invalid_argument, "expert parallel runs the tensor-core path (DB_MOE_BF16 or DB_MOE_FP16)");
  if (world < 1 || rank < 0 || rank >= world) throw_error(Errc::invalid_argument, "bad rank/world");
  if (cfg.experts % world != 0 || cfg.batch % world != 0)
    throw_error(Errc::invalid_argument, "expert parallel needs experts and tokens divisible by the world size");
  if (cfg.data_dim % 256 != 0 || cfg.hidden % 256 != 0)
    throw_error(Errc::invalid_argument, "tensor-core MoE path needs data_dim and hidden multiples of 256");
  Impl& I = *impl_;
  I.cfg = cfg;
  I.fmt = precision == 2 ? DBK_FMT_F16 : DBK_FMT_BF16;
  I.rank = rank;
  I.world = world;
  I.E = static_cast<int>(cfg.experts / world);
  I.e_first = rank * I.E;
  I.sms = sm_count();
  T_ = cfg.batch / world;
  const std::int64_t first = rank * T_, last = first + T_;
  stream_ = make_stream();
  MoeDev& D = I.dev;
  const int n = static_cast<int>(cfg.experts), k = static_cast<int>(cfg.active_per_example);
  D.alloc(T_, n, k, static_cast<int>(cfg.data_dim), static_cast<int>(cfg.hidden));
  // the rank's token slice of the db_moe_run fixtures (src/c_api.cpp:270-290)
  I.x.alloc(static_cast<size_t>(T_) * cfg.data_dim);
  upload_moe_inputs(cfg, seed, first, last, D.scores.get(), I.x.get());
  I.out.alloc(static_cast<size_t>(T_) * cfg.data_dim);
  I.pos_of_item.alloc(static_cast<size_t>(T_) * k);
  I.cnt.alloc(static_cast<size_t>(world) * I.E);
  I.pstart.alloc(static_cast<size_t>(I.E) + 1);
  I.n_tiles.alloc(1);
  I.src_row.alloc(static_cast<size_t>(I.E) * world);
  I.cum.alloc(static_cast<size_t>(I.E) * (world + 1));
  I.ensure_capacity(T_ * k + static_cast<std::int64_t>(I.E) * 256);
  upload_expert_weights(cfg, mix_seed(seed, 0xe4be27ULL), I.e_first, I.E, I.fmt, I.w1, I.w2, I.w1tab, I.w2tab, stream_);
  check(cudaStreamSynchronize(stream_), "upload");
}

MoeEp::~MoeEp() {
  impl_.reset();
  if (stream_) {
    cudaStreamSynchronize(stream_);
    cudaStreamDestroy(stream_);
  }
}

std::int64_t MoeEp::items() const { return T_ * impl_->cfg.active_per_example; }
int MoeEp::local_experts() const { return impl_->E; }

void MoeEp::dispatch(void* send, std::int32_t* expert_counts) {
  Impl& I = *impl_;
  MoeDev& D = I.dev;
  prof_.begin(3, stream_);
  D.gate(stream_);
  D.sort(stream_);
  check(dbk_moe_ep_pack(I.fmt, items(), D.k, D.d, D.order.get(), I.x.get(), send, I.pos_of_item.get(), I.sms * 8, stream_),
        "ep pack");
  prof_.end(stream_);
  const auto off = D.offsets.download(static_cast<size_t>(D.n) + 1, stream_);  // synchronises
  for (int e = 0; e < D.n; ++e) expert_counts[e] = off[static_cast<size_t>(e) + 1] - off[static_cast<size_t>(e)];
}

// World 1: no exchange, so the layer runs as one device pass — gate, sort,
// token-major dispatch straight into the tiled operand, the two grouped
// GEMMs, slot-order combine (the single-GPU bf16 layer's kernels, on this
// session's experts).
void MoeEp::forward_local() {
  Impl& I = *impl_;
  MoeDev& D = I.dev;
  if (I.world != 1) throw_error(Errc::invalid_argument, "forward_local needs world 1");
  const int d = static_cast<int>(I.cfg.data_dim), h = static_cast<int>(I.cfg.hidden);
  prof_.begin(3, stream_);
  D.gate(stream_);
  D.sort(stream_);
  check(dbk_moe_tc_layout(D.n, D.offsets.get(), I.pstart.get(), I.tile_expert.get(), I.tile_rb.get(),
                            I.n_tiles.get(), stream_), "moe layout");
  check(dbk_moe_tc_dispatch(I.fmt, T_, D.k, d, D.order.get(), D.ids.get(), D.offsets.get(), I.pstart.get(), I.x.get(),
                              I.A.get(), I.pos_of_item.get(), I.sms * 8, stream_),
        "moe dispatch");  // pos_of_item holds each item's padded row here
  prof_.end(stream_);
  if (I.Y.size() < static_cast<size_t>(I.cap_rows) * d) I.Y.alloc(static_cast<size_t>(I.cap_rows) * d);
  prof_.begin(4, stream_);
  check(dbk_moe_tc_gemm(I.fmt, 0, D.n, d, h, I.n_tiles.get(), I.tile_expert.get(), I.tile_rb.get(), I.A.get(),
                          I.w1tab.get(), I.H.get(), nullptr, 0, -1, nullptr, I.sms, stream_), "moe gemm1");
  check(dbk_moe_tc_gemm(I.fmt, 1, D.n, h, d, I.n_tiles.get(), I.tile_expert.get(), I.tile_rb.get(), I.H.get(),
                          I.w2tab.get(), nullptr, I.Y.get(), 0, -1, nullptr, I.sms, stream_), "moe gemm2");
  prof_.end(stream_);
  prof_.begin(6, stream_);
  check(dbk_moe_tc_combine(I.fmt, T_, D.k, d, D.wts.get(), I.pos_of_item.get(), I.Y.get(), I.out.get(), stream_),
        "moe combine");
  prof_.end(stream_);
  last_recv_rows_ = items();
}

void MoeEp::comm_init(const void* unique_id) {
  Impl& I = *impl_;
  const Nccl& nc = Nccl::get();
  if (I.comm) {
    nc.CommDestroy(I.comm);
    I.comm = nullptr;
  }
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  nc.check(nc.CommInitRank(&I.comm, I.world, id, I.rank), "ncclCommInitRank");
  if (!I.cs) check(cudaStreamCreateWithFlags(&I.cs, cudaStreamNonBlocking), "stream");
  const int n = I.dev.n;
  I.send_cnt.alloc(static_cast<size_t>(n));
  I.recv_cnt.alloc(static_cast<size_t>(I.world) * I.E);
  if (!I.h_cnt)
    check(cudaHostAlloc(reinterpret_cast<void**>(&I.h_cnt), sizeof(std::int32_t) * (static_cast<size_t>(n) * 2),
                        cudaHostAllocDefault), "pinned counts");
  I.sendb.alloc(static_cast<size_t>(items()) * I.cfg.data_dim);
  I.backb.alloc(static_cast<size_t>(items()) * I.cfg.data_dim);
}

// One expert-parallel forward with the exchange on NCCL, all
// of it issued from here on the session stream (kernels) and the exchange
// stream (NCCL), ordered by events:
//   1. gate, stable sort, per-expert send counts               (stream)
//   2. count all-to-all as grouped ncclSend/ncclRecv of the [q·E, (q+1)·E)
//      slices, then their copy to pinned host memory           (exchange)
//      — meanwhile the stream packs the rows in sorted order;
//   3. the host waits for the counts alone (the pack keeps running), plans
//      the pieces (make_ep_plan) and lays out the received experts;
//   4. per local-expert range c: the rows' grouped send/recv (exchange),
//      the range's grouped GEMMs once they arrived (stream), its outputs
//      back to their senders once computed (exchange), so range c+1's
//      transfer overlaps range c's GEMMs;
//   5. the slot-order combine once every output is back       (stream).
// Receivers concatenate by source rank, which keeps every expert's rows in
// the reference's (token, slot) order (src/moe.cpp:214-251).
void MoeEp::forward(int chunks) {
  Impl& I = *impl_;
  MoeDev& D = I.dev;
  if (!I.comm) {
    if (I.world != 1) throw_error(Errc::invalid_argument, "expert parallel forward needs db_moe_ep_comm_init");
    forward_local();
    return;
  }
  const Nccl& nc = Nccl::get();
  const int G = I.world, E = I.E, n = D.n;
  const size_t row_bytes = static_cast<size_t>(I.cfg.data_dim) * 2;
  prof_.begin(3, stream_);
  D.gate(stream_);
  D.sort(stream_);
  check(dbk_moe_ep_counts(n, D.offsets.get(), I.send_cnt.get(), stream_), "ep counts");
  cudaEvent_t ev_sorted = I.event(0), ev_counts = I.event(1), ev_packed = I.event(2), ev_back = I.event(3);
  check(cudaEventRecord(ev_sorted, stream_), "event");
  check(cudaStreamWaitEvent(I.cs, ev_sorted, 0), "wait");
  nc.check(nc.GroupStart(), "ncclGroupStart");
  for (int q = 0; q < G; ++q) {
    nc.check(nc.Send(I.send_cnt.get() + static_cast<size_t>(q) * E, static_cast<size_t>(E), ncclInt32, q, I.comm, I.cs),
             "ncclSend counts");
    nc.check(nc.Recv(I.recv_cnt.get() + static_cast<size_t>(q) * E, static_cast<size_t>(E), ncclInt32, q, I.comm, I.cs),
             "ncclRecv counts");
  }
  nc.check(nc.GroupEnd(), "ncclGroupEnd");
  std::int32_t* h_send = I.h_cnt;
  std::int32_t* h_recv = I.h_cnt + n;
  check(cudaMemcpyAsync(h_send, I.send_cnt.get(), sizeof(std::int32_t) * static_cast<size_t>(n), cudaMemcpyDeviceToHost,
                        I.cs), "D2H counts");
  check(cudaMemcpyAsync(h_recv, I.recv_cnt.get(), sizeof(std::int32_t) * static_cast<size_t>(G) * E,
                        cudaMemcpyDeviceToHost, I.cs), "D2H counts");
  check(cudaEventRecord(ev_counts, I.cs), "event");
  check(dbk_moe_ep_pack(I.fmt, items(), D.k, D.d, D.order.get(), I.x.get(), I.sendb.get(), I.pos_of_item.get(),
                        I.sms * 8, stream_), "ep pack");
  check(cudaEventRecord(ev_packed, stream_), "event");
  prof_.end(stream_);
  check(cudaEventSynchronize(ev_counts), "counts");  // the GPU keeps packing meanwhile
  const EpPlan plan = make_ep_plan(G, E, h_send, h_recv, chunks);
  if (plan.recv_total > I.recv_cap) {
    check(cudaStreamSynchronize(stream_), "sync");  // the old buffers may still be read
    check(cudaStreamSynchronize(I.cs), "sync");
    I.recv_cap = plan.recv_total + plan.recv_total / 4 + 1;
    I.recvb.alloc(static_cast<size_t>(I.recv_cap) * I.cfg.data_dim);
    I.retb.alloc(static_cast<size_t>(I.recv_cap) * I.cfg.data_dim);
  }
  // layout of the received experts from the device copy of the counts
  I.cnt_h.assign(h_recv, h_recv + static_cast<size_t>(G) * E);
  I.pstart_h.assign(static_cast<size_t>(E) + 1, 0);
  for (int e = 0; e < E; ++e) {
    std::int64_t tot = 0;
    for (int r = 0; r < G; ++r) tot += h_recv[r * E + e];
    I.pstart_h[static_cast<size_t>(e) + 1] = I.pstart_h[static_cast<size_t>(e)] + (tot + 255) / 256 * 256;
  }
  I.ensure_capacity(I.pstart_h[static_cast<size_t>(E)]);
  check(cudaStreamWaitEvent(stream_, ev_counts, 0), "wait");
  check(dbk_moe_ep_layout(G, E, I.recv_cnt.get(), I.pstart.get(), I.tile_expert.get(), I.tile_rb.get(),
                          I.n_tiles.get(), I.src_row.get(), I.cum.get(), stream_), "ep layout");
  // rows out, per expert range
  auto* sb = reinterpret_cast<std::uint8_t*>(I.sendb.get());
  auto* rb = reinterpret_cast<std::uint8_t*>(I.recvb.get());
  auto* tb = reinterpret_cast<std::uint8_t*>(I.retb.get());
  auto* bb = reinterpret_cast<std::uint8_t*>(I.backb.get());
  auto exchange = [&](int c, const std::uint8_t* src, const std::vector<std::int64_t>& src_off,
                      const std::vector<std::int64_t>& src_rows, std::uint8_t* dst,
                      const std::vector<std::int64_t>& dst_off, const std::vector<std::int64_t>& dst_rows) {
    nc.check(nc.GroupStart(), "ncclGroupStart");
    for (int q = 0; q < G; ++q) {
      const size_t i = static_cast<size_t>(c) * G + q;
      if (src_rows[i])
        nc.check(nc.Send(src + src_off[i] * row_bytes, src_rows[i] * row_bytes, ncclUint8, q, I.comm, I.cs),
                 "ncclSend rows");
      if (dst_rows[i])
        nc.check(nc.Recv(dst + dst_off[i] * row_bytes, dst_rows[i] * row_bytes, ncclUint8, q, I.comm, I.cs),
                 "ncclRecv rows");
    }
    nc.check(nc.GroupEnd(), "ncclGroupEnd");
  };
  check(cudaStreamWaitEvent(I.cs, ev_packed, 0), "wait");
  const int C = plan.C;
  for (int c = 0; c < C; ++c) {
    exchange(c, sb, plan.s_off, plan.s_rows, rb, plan.r_off, plan.r_rows);
    check(cudaEventRecord(I.event(4 + static_cast<size_t>(c)), I.cs), "event");
  }
  for (int c = 0; c < C; ++c) {
    check(cudaStreamWaitEvent(stream_, I.event(4 + static_cast<size_t>(c)), 0), "wait");
    experts_range(rb, tb, plan.bounds[static_cast<size_t>(c)].first, plan.bounds[static_cast<size_t>(c)].second);
    check(cudaEventRecord(I.event(4 + static_cast<size_t>(C + c)), stream_), "event");
  }
  for (int c = 0; c < C; ++c) {  // outputs back: the reverse pieces
    check(cudaStreamWaitEvent(I.cs, I.event(4 + static_cast<size_t>(C + c)), 0), "wait");
    exchange(c, tb, plan.r_off, plan.r_rows, bb, plan.s_off, plan.s_rows);
  }
  check(cudaEventRecord(ev_back, I.cs), "event");
  check(cudaStreamWaitEvent(stream_, ev_back, 0), "wait");
  combine(bb);
  last_recv_rows_ = plan.recv_total;
}

void MoeEp::layout(const std::int32_t* cnt) {
  Impl& I = *impl_;
  const int G = I.world, E = I.E;
  I.cnt_h.assign(cnt, cnt + static_cast<size_t>(G) * E);
  I.pstart_h.assign(static_cast<size_t>(E) + 1, 0);
  for (int e = 0; e < E; ++e) {
    std::int64_t tot = 0;
    for (int r = 0; r < G; ++r) tot += cnt[r * E + e];
    I.pstart_h[static_cast<size_t>(e) + 1] = I.pstart_h[static_cast<size_t>(e)] + (tot + 255) / 256 * 256;
  }
  I.ensure_capacity(I.pstart_h[static_cast<size_t>(E)]);
  check(cudaMemcpyAsync(I.cnt.get(), cnt, sizeof(std::int32_t) * static_cast<size_t>(G) * E, cudaMemcpyHostToDevice,
                        stream_), "H2D counts");
  check(dbk_moe_ep_layout(G, E, I.cnt.get(), I.pstart.get(), I.tile_expert.get(), I.tile_rb.get(), I.n_tiles.get(),
                          I.src_row.get(), I.cum.get(), stream_), "ep layout");
}

// Local experts [e_begin, e_end): their padded rows are one contiguous
// range, their row tiles too (the layout is expert-major).
void MoeEp::experts_range(const void* recv, void* ret, int e_begin, int e_end) {
  Impl& I = *impl_;
  const int G = I.world, E = I.E, d = static_cast<int>(I.cfg.data_dim), h = static_cast<int>(I.cfg.hidden);
  if (I.pstart_h.size() != static_cast<size_t>(E) + 1) throw_error(Errc::invalid_argument, "db_moe_ep_layout first");
  if (e_begin < 0 || e_end > E || e_begin > e_end) throw_error(Errc::invalid_argument, "expert range out of bounds");
  if (e_begin == e_end) return;
  const std::int32_t r0 = static_cast<std::int32_t>(I.pstart_h[static_cast<size_t>(e_begin)]);
  const std::int32_t r1 = static_cast<std::int32_t>(I.pstart_h[static_cast<size_t>(e_end)]);
  if (r0 == r1) return;
  prof_.begin(4, stream_);
  check(dbk_moe_ep_scatter(G, E, d, I.pstart.get(), I.tile_expert.get(), I.src_row.get(), I.cum.get(), recv,
                           I.A.get(), I.recv_of_row.get(), r0, r1, I.sms * 8, stream_), "ep scatter");
  check(dbk_moe_tc_gemm(I.fmt, 0, E, d, h, I.n_tiles.get(), I.tile_expert.get(), I.tile_rb.get(), I.A.get(),
                          I.w1tab.get(), I.H.get(), nullptr, r0 / 128, r1 / 128, nullptr, I.sms, stream_),
        "ep gemm1");
  // GEMM2 writes each output row straight to its receive-order row of ret
  check(dbk_moe_tc_gemm(I.fmt, 1, E, h, d, I.n_tiles.get(), I.tile_expert.get(), I.tile_rb.get(), I.H.get(),
                          I.w2tab.get(), nullptr, ret, r0 / 128, r1 / 128, I.recv_of_row.get(), I.sms, stream_),
        "ep gemm2");
  prof_.end(stream_);
  if (prof_.on) {
    std::int64_t rows = 0;
    for (int r = 0; r < G; ++r)
      for (int e = e_begin; e < e_end; ++e) rows += I.cnt_h[static_cast<size_t>(r) * E + e];
    prof_.add_work(4, 4.0 * static_cast<double>(rows) * d * h, 0.0);
  }
}

void MoeEp::experts(const void* recv, const std::int32_t* cnt, void* ret) {
  layout(cnt);
  experts_range(recv, ret, 0, impl_->E);
}

void MoeEp::combine(const void* ret_recv) {
  Impl& I = *impl_;
  prof_.begin(6, stream_);
  check(dbk_moe_tc_combine(I.fmt, T_, I.dev.k, I.dev.d, I.dev.wts.get(), I.pos_of_item.get(), ret_recv, I.out.get(),
                             stream_), "ep combine");
  prof_.end(stream_);
}

void MoeEp::download_outputs(float* out) {
  check(cudaMemcpyAsync(out, impl_->out.get(), sizeof(float) * static_cast<size_t>(T_) * impl_->cfg.data_dim,
                        cudaMemcpyDeviceToHost, stream_), "D2H outputs");
  synchronize();
}

void MoeEp::synchronize() {
  check(cudaStreamSynchronize(stream_), "sync");
  impl_->dev.check_err(stream_);
}

}  // namespace dev

// ------------------------------------------------------- C++ operator API
GateAssignment top_k_gate(const TensorBatch& scores, std::int64_t k) {
  const std::int64_t n = scores.width();
  if (k < 1 || k > n) throw_error(Errc::k_too_large, "k=" + std::to_string(k) + " with n=" + std::to_string(n));
  if (!scores.all_finite()) throw_error(Errc::non_finite_value, "non-finite gate score");
  GateAssignment g;
  g.per_example.resize(static_cast<size_t>(scores.rows()));
  if (scores.rows() == 0) return g;
  dev::require_device();
  dev::StreamGuard sg{dev::make_stream()};
  dev::MoeDev D;
  D.alloc(scores.rows(), static_cast<int>(n), static_cast<int>(k), 1, 1);
  D.scores.upload(scores.data().data(), scores.data().size(), sg.s);
  D.gate(sg.s);
  D.check_err(sg.s);
  const auto ids = D.ids.download(static_cast<size_t>(scores.rows() * k), sg.s);
  const auto w = D.wts.download(static_cast<size_t>(scores.rows() * k), sg.s);
  for (std::int64_t t = 0; t < scores.rows(); ++t) {
    auto& e = g.per_example[static_cast<size_t>(t)];
    for (std::int64_t s = 0; s < k; ++s) {
      e.push_back({ids[static_cast<size_t>(t * k + s)], w[static_cast<size_t>(t * k + s)]});
    }
  }
  return g;
}

namespace {
void check_moe_args(const TensorBatch& inputs, const ExpertSet& experts, const GateAssignment& gates) {
  if (inputs.width() != experts.data_dim()) throw_error(Errc::width_mismatch, "inputs width " + std::to_string(inputs.width()));
  if (gates.per_example.size() != static_cast<size_t>(inputs.rows())) {
    throw_error(Errc::row_count_mismatch, "gate assignment rows do not match inputs");
  }
  if (!inputs.all_finite()) throw_error(Errc::non_finite_value, "non-finite input");
}

MoeResult moe_forward(const TensorBatch& inputs, const ExpertSet& experts, const GateAssignment& gates,
                      bool batched) {
  check_moe_args(inputs, experts, gates);
  const std::int64_t T = inputs.rows();
  const std::int64_t d = experts.data_dim();
  MoeResult r;
  r.outputs = TensorBatch(T, d);
  r.trace.per_function_calls.assign(static_cast<size_t>(experts.size()), 0);
  std::int64_t k = 0;
  for (const auto& e : gates.per_example) k = std::max<std::int64_t>(k, static_cast<std::int64_t>(e.size()));
  if (T == 0 || k == 0) return r;
  // Ragged gate lists are padded with zero-weight slots on expert 0; the
  // padding rows are excluded from the trace below.
  std::vector<std::int32_t> ids(static_cast<size_t>(T * k), 0);
  std::vector<double> w(static_cast<size_t>(T * k), 0.0);
  std::vector<unsigned char> real(static_cast<size_t>(T * k), 0);
  for (std::int64_t t = 0; t < T; ++t) {
    const auto& es = gates.per_example[static_cast<size_t>(t)];
    for (size_t s = 0; s < es.size(); ++s) {
      if (es[s].expert < 0 || es[s].expert >= experts.size()) {
        throw_error(Errc::invalid_argument, "expert id " + std::to_string(es[s].expert));
      }
      ids[static_cast<size_t>(t * k) + s] = es[s].expert;
      w[static_cast<size_t>(t * k) + s] = es[s].weight;
      real[static_cast<size_t>(t * k) + s] = 1;
    }
  }
  dev::require_device();
  dev::StreamGuard sg{dev::make_stream()};
  dev::MoeDev D;
  D.alloc(T, static_cast<int>(experts.size()), static_cast<int>(k), static_cast<int>(d), static_cast<int>(experts.hidden()));
  D.alloc_fp64_work();
  D.x.upload(inputs.data().data(), inputs.data().size(), sg.s);
  D.ids.upload(ids, sg.s);
  D.wts.upload(w, sg.s);
  D.upload_experts(experts, sg.s);
  const auto t0 = std::chrono::steady_clock::now();
  if (batched) {
    D.sort(sg.s);
    D.experts_fp64(sg.s);
  } else {
    // One single-row expert call per (token, slot) in token-major order.
    const std::int64_t items = T * k;
    std::vector<std::int32_t> off(static_cast<size_t>(items) * static_cast<size_t>(experts.size() + 1));
    std::vector<std::int32_t> order(static_cast<size_t>(items));
    for (std::int64_t i = 0; i < items; ++i) {
      order[static_cast<size_t>(i)] = static_cast<std::int32_t>(i);
      for (std::int64_t e = 0; e <= experts.size(); ++e)
        off[static_cast<size_t>(i * (experts.size() + 1) + e)] = e <= ids[static_cast<size_t>(i)] ? 0 : 1;
    }
    dev::Buf<std::int32_t> doff, dord;
    doff.upload(off, sg.s);
    dord.upload(order, sg.s);
    for (std::int64_t i = 0; i < items; ++i) {
      if (!real[static_cast<size_t>(i)]) continue;
      // order[0] = item i → input row i / k, staged row i.
      dev::check(dbk_moe_expert_fp64(1, static_cast<std::int32_t>(experts.size()), static_cast<std::int32_t>(k),
                                     static_cast<std::int32_t>(d), static_cast<std::int32_t>(experts.hidden()),
                                     dord.get() + i, doff.get() + i * (experts.size() + 1), D.x.get(),
                                     D.w1tab.get(), D.w2tab.get(), D.hidden.get(), D.staged.get(),
                                     D.tiles.get(), sg.s),
                 "naive expert call");
    }
  }
  D.combine_fp64(sg.s);
  dev::check(cudaStreamSynchronize(sg.s), "sync");
  const auto t1 = std::chrono::steady_clock::now();
  dev::check(cudaMemcpy(r.outputs.data().data(), D.out.get(), sizeof(double) * r.outputs.data().size(),
                        cudaMemcpyDeviceToHost), "D2H");
  const double secs = std::chrono::duration<double>(t1 - t0).count();
  r.trace.module_seconds = secs;
  r.trace.total_seconds = secs;
  r.trace.per_step_seconds.push_back(secs);
  if (batched) {
    std::vector<std::int64_t> rows(static_cast<size_t>(experts.size()), 0);
    for (size_t i = 0; i < ids.size(); ++i) if (real[i]) ++rows[static_cast<size_t>(ids[i])];
    for (std::int64_t e = 0; e < experts.size(); ++e) {
      if (!rows[static_cast<size_t>(e)]) continue;
      ++r.trace.expensive_calls;
      ++r.trace.per_function_calls[static_cast<size_t>(e)];
      r.trace.peak_group_rows = std::max(r.trace.peak_group_rows, rows[static_cast<size_t>(e)]);
    }
  } else {
    for (size_t i = 0; i < ids.size(); ++i) {
      if (!real[i]) continue;
      ++r.trace.expensive_calls;
      ++r.trace.per_function_calls[static_cast<size_t>(ids[i])];
      r.trace.peak_group_rows = 1;
    }
  }
  if (!r.outputs.all_finite()) throw_error(Errc::non_finite_value, "non-finite output");
  return r;
}
}  // namespace

MoeResult moe_forward_naive(const TensorBatch& inputs, const ExpertSet& experts, const GateAssignment& gates) {
  return moe_forward(inputs, experts, gates, false);
}

MoeResult moe_forward_batched(const TensorBatch& inputs, const ExpertSet& experts, const GateAssignment& gates) {
  return moe_forward(inputs, experts, gates, true);
}

}  // namespace dynbatch
