// iep_head.cpp — IEP classifier head (iep_head.hpp, head.cu).
#include "iep_head.hpp"

#include <algorithm>
#include <cmath>

#include "dynbatch.hpp"
#include "moe_bf16.hpp"

#include "dynbatch/dbk.h"

namespace dynbatch::dev {

HeadWeights make_head_weights(int C, int P, int F, int A, std::uint64_t seed) {
  HeadWeights h;
  h.C = C;
  h.P = P;
  h.F = F;
  h.A = A;
  Rng rng(mix_seed(seed, 0x4eadULL));
  const auto fill = [&rng](std::vector<double>& v, size_t n, double fan_in) {
    const double scale = 1.0 / std::sqrt(fan_in);
    v.resize(n);
    for (double& x : v) x = rng.uniform(-0.5, 0.5) * scale;
  };
  const size_t K1 = static_cast<size_t>(49) * P;
  fill(h.wp, static_cast<size_t>(C) * P, C);
  fill(h.bp, static_cast<size_t>(P), C);
  fill(h.w1, K1 * F, static_cast<double>(K1));
  fill(h.b1, static_cast<size_t>(F), static_cast<double>(K1));
  fill(h.w2, static_cast<size_t>(F) * A, F);
  fill(h.b2, static_cast<size_t>(A), F);
  return h;
}

namespace {
constexpr int kC = 128, kPx = 196, kBM = 128, kPairRows = 256;
std::int64_t pad_rows(std::int64_t rows) { return (rows + kPairRows - 1) / kPairRows * kPairRows; }
}  // namespace

IepHead::IepHead(int answers, std::uint64_t seed, cudaStream_t s) : answers_(answers) {
  if (answers < 1 || answers > kPad) throw_error(Errc::invalid_argument, "head answers must be in [1, 256]");
  int dev = 0;
  check(cudaGetDevice(&dev), "device");
  check(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev), "SM count");
  const HeadWeights h = make_head_weights(kC, kP, kF, answers, seed);
  const int K1 = 49 * kP;
  // B operands (N × K) from the input-major weights; the logit columns are
  // padded to one 256-wide N tile with zero weights and biases
  std::vector<double> w2p(static_cast<size_t>(kF) * kPad, 0.0), b2p(kPad, 0.0);
  for (int k = 0; k < kF; ++k)
    for (int a = 0; a < answers; ++a) w2p[static_cast<size_t>(k) * kPad + a] = h.w2[static_cast<size_t>(k) * answers + a];
  for (int a = 0; a < answers; ++a) b2p[a] = h.b2[a];
  const auto up = [s](Buf<std::uint16_t>& dst, const std::vector<double>& w, int K, int N) {
    std::vector<std::uint16_t> t(static_cast<size_t>(K) * N);
    tile_weights(w, K, N, DBK_FMT_F16, t.data());
    dst.upload(t, s);
    check(cudaStreamSynchronize(s), "weights upload");
  };
  up(wp_, h.wp, kC, kP);
  up(w1_, h.w1, K1, kF);
  up(w2_, w2p, kF, kPad);
  const auto upf = [s](Buf<float>& dst, const std::vector<double>& v) {
    std::vector<float> f(v.begin(), v.end());
    dst.upload(f, s);
    check(cudaStreamSynchronize(s), "bias upload");
  };
  upf(wp32_, h.wp);
  upf(w132_, h.w1);
  upf(w232_, h.w2);
  upf(bp_, h.bp);
  upf(b1_, h.b1);
  upf(b2_, b2p);
  const std::vector<const void*> wt = {wp_.get(), w1_.get(), w2_.get()};
  const std::vector<const float*> bt = {bp_.get(), b1_.get(), b2_.get()};
  wtab_.upload(wt, s);
  btab_.upload(bt, s);
  check(cudaStreamSynchronize(s), "head tables");
}

double IepHead::flops_per_program() const {
  return 2.0 * (static_cast<double>(kPx) * kC * kP + 49.0 * kP * kF + static_cast<double>(kF) * answers_);
}

void IepHead::size_for(std::int64_t b, cudaStream_t s) {
  const std::int64_t r0 = pad_rows(b * kPx), r1 = pad_rows(b);
  if (b > cap_b_) {
    a0_.alloc(static_cast<size_t>(r0) * kC);
    h1_.alloc(static_cast<size_t>(r0) * kP);
    a1_.alloc(static_cast<size_t>(r1) * 49 * kP);
    h2_.alloc(static_cast<size_t>(r1) * kF);
    logits_.alloc(static_cast<size_t>(r1) * kPad);
    std::vector<std::int32_t> iota(static_cast<size_t>(r0 / kBM));
    for (size_t i = 0; i < iota.size(); ++i) iota[i] = static_cast<std::int32_t>(i);
    iota_.upload(iota, s);
    zeros_.alloc(iota.size());
    zeros_.zero(s);
    cap_b_ = b;
    tiles_b_ = -1;
  }
  if (tiles_b_ != b) {
    const std::vector<std::int32_t> nt = {static_cast<std::int32_t>(r0 / kBM), static_cast<std::int32_t>(r1 / kBM)};
    ntiles_.upload(nt, s);
    check(cudaStreamSynchronize(s), "head tiles");  // nt is a host temporary
    tiles_b_ = b;
  }
}

int IepHead::forward(std::int64_t b, const std::int32_t* root_g, const std::int32_t* fid,
                     const std::int32_t* arity_of, const std::int32_t* example, const float* inputs,
                     const float* values, cudaStream_t s) {
  if (b <= 0) return 0;
  size_for(b, s);
  const void* const* wt = wtab_.get();
  const float* const* bt = btab_.get();
  check(dbk_head_pack(b, root_g, fid, arity_of, example, inputs, values, a0_.get(), s), "head pack");
  check(dbk_tc_gemm_bias(DBK_FMT_F16, 0, 1, kC, kP, ntiles_.get(), zeros_.get(), iota_.get(), a0_.get(), wt,
                         bt, h1_.get(), nullptr, 0, -1, nullptr, sms_, s),
        "head projection");
  check(dbk_head_pool(b, kP, h1_.get(), a1_.get(), s), "head pool");
  check(dbk_tc_gemm_bias(DBK_FMT_F16, 0, 1, 49 * kP, kF, ntiles_.get() + 1, zeros_.get(), iota_.get(), a1_.get(),
                         wt + 1, bt + 1, h2_.get(), nullptr, 0, -1, nullptr, sms_, s),
        "head fc1");
  check(dbk_tc_gemm_bias(DBK_FMT_F16, 2, 1, kF, kPad, ntiles_.get() + 1, zeros_.get(), iota_.get(), h2_.get(),
                         wt + 2, bt + 2, nullptr, logits_.get(), 0, -1, nullptr, sms_, s),
        "head fc2");
  return 5;
}

void IepHead::sgd(float lr, const float* gwp, const float* gbp, const float* gw1, const float* gb1, const float* gw2,
                  const float* gb2, cudaStream_t s) {
  const std::int64_t K1 = 49LL * kP;
  check(dbk_tr_sgd(static_cast<std::int64_t>(kC) * kP, wp32_.get(), gwp, lr, s), "sgd");
  check(dbk_tr_sgd(K1 * kF, w132_.get(), gw1, lr, s), "sgd");
  check(dbk_tr_sgd(static_cast<std::int64_t>(kF) * answers_, w232_.get(), gw2, lr, s), "sgd");
  check(dbk_tr_sgd(kP, bp_.get(), gbp, lr, s), "sgd");
  check(dbk_tr_sgd(kF, b1_.get(), gb1, lr, s), "sgd");
  check(dbk_tr_sgd(answers_, b2_.get(), gb2, lr, s), "sgd");  // the padded logit columns stay 0
  check(dbk_tr_tile_weights(wp32_.get(), kC, kP, kP, wp_.get(), s), "tile");
  check(dbk_tr_tile_weights(w132_.get(), static_cast<std::int32_t>(K1), kF, kF, w1_.get(), s), "tile");
  check(dbk_tr_tile_weights(w232_.get(), kF, answers_, kPad, w2_.get(), s), "tile");
}

void IepHead::download(std::int64_t b, float* out, cudaStream_t s) const {
  check(cudaMemcpy2DAsync(out, sizeof(float) * answers_, logits_.get(), sizeof(float) * kPad,
                          sizeof(float) * answers_, static_cast<size_t>(b), cudaMemcpyDeviceToHost, s),
        "D2H logits");
  check(cudaStreamSynchronize(s), "sync");
}

}  // namespace dynbatch::dev
