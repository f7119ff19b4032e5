// moe_bf16.cpp — host side of the 16-bit tensor-core MoE expert path
// (fp16 or bf16 operands, DBK_FMT_*).
//
// Expert weights follow ExpertSet (src/moe.cpp:71-88): Rng(mix_seed(seed, e)),
// w1 [d × h] then w2 [h × d], uniform(-0.5, 0.5)/sqrt(fan_in); they are
// generated on host threads (one Rng stream per expert, so the split is
// exact), rounded to fp16 or bf16 and pre-tiled for the grouped tcgen05 GEMMs
// (moe_gemm.cu): B operand of GEMM1 = W1ᵀ [N = h][K = d], of GEMM2 = W2ᵀ
// [N = d][K = h], as 32 KB blocks per (256-column N tile, 64-wide K chunk).
#include "moe_bf16.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>

#include <cuda_fp16.h>

#include "device.hpp"

#include "dynbatch/dbk.h"

namespace dynbatch::dev {

namespace {

std::uint16_t bf16(double v) {
  float f = static_cast<float>(v);
  std::uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<std::uint16_t>(u >> 16);
}

std::uint16_t f16(double v) {
  const __half x = __double2half(v);  // round to nearest even, subnormals kept
  std::uint16_t u;
  std::memcpy(&u, &x, 2);
  return u;
}

}  // namespace

// Element (n, kk) of the N × K operand, stored input-major in `w` as
// w[kk * N + n], into [N/256][K/64] blocks of 32 KB, each two 16 KB halves
// (columns 0-127 and 128-255 of the N tile: one per CTA of a pair) of
// [8 k-groups][128 n][8] (moe_gemm.cu).
void tile_weights(const std::vector<double>& w, int K, int N, int fmt, std::uint16_t* out) {
  const int n_kc = K / 64;
  for (int kk = 0; kk < K; ++kk) {
    const int kc = kk / 64, k8 = (kk % 64) / 8, ke = kk % 8;
    for (int n = 0; n < N; ++n) {
      const int nt = n / 256, half = (n % 256) / 128, nn = n % 128;
      const size_t blk = static_cast<size_t>(nt) * n_kc + kc;
      out[blk * 256 * 64 + ((static_cast<size_t>(half) * 8 + k8) * 128 + nn) * 8 + ke] =
          fmt == DBK_FMT_F16 ? f16(w[static_cast<size_t>(kk) * N + n]) : bf16(w[static_cast<size_t>(kk) * N + n]);
    }
  }
}

void upload_expert_weights(const MoeConfig& cfg, std::uint64_t expert_seed, int e_first, int n_local, int fmt,
                           Buf<std::uint16_t>& w1, Buf<std::uint16_t>& w2, Buf<const void*>& w1tab,
                           Buf<const void*>& w2tab, cudaStream_t s) {
  const int d = static_cast<int>(cfg.data_dim), h = static_cast<int>(cfg.hidden);
  const size_t per = static_cast<size_t>(d) * h;
  w1.alloc(per * n_local);
  w2.alloc(per * n_local);
  // Experts are independent Rng streams → generate on host threads.
  const double s1 = 1.0 / std::sqrt(static_cast<double>(d)), s2 = 1.0 / std::sqrt(static_cast<double>(h));
  const int chunk = 16;
  std::vector<std::uint16_t> h1(per * chunk), h2(per * chunk);
  for (int e0 = 0; e0 < n_local; e0 += chunk) {
    const int ne = std::min(chunk, n_local - e0);
    std::vector<std::thread> pool;
    for (int j = 0; j < ne; ++j) {
      pool.emplace_back([&, j] {
        Rng rng(mix_seed(expert_seed, static_cast<std::uint64_t>(e_first + e0 + j)));
        std::vector<double> w(per);
        for (double& v : w) v = rng.uniform(-0.5, 0.5) * s1;  // w1 [d][h]
        tile_weights(w, d, h, fmt, h1.data() + per * j);
        for (double& v : w) v = rng.uniform(-0.5, 0.5) * s2;  // w2 [h][d]
        tile_weights(w, h, d, fmt, h2.data() + per * j);
      });
    }
    for (auto& t : pool) t.join();
    check(cudaMemcpy(w1.get() + per * e0, h1.data(), per * ne * 2, cudaMemcpyHostToDevice), "H2D w1");
    check(cudaMemcpy(w2.get() + per * e0, h2.data(), per * ne * 2, cudaMemcpyHostToDevice), "H2D w2");
  }
  std::vector<const void*> t1(static_cast<size_t>(n_local)), t2(static_cast<size_t>(n_local));
  for (int e = 0; e < n_local; ++e) {
    t1[static_cast<size_t>(e)] = w1.get() + per * e;
    t2[static_cast<size_t>(e)] = w2.get() + per * e;
  }
  w1tab.upload(t1, s);
  w2tab.upload(t2, s);
  check(cudaStreamSynchronize(s), "sync");
}

struct MoeBf16::Impl {
  std::int64_t T = 0;
  int n = 0, k = 0, d = 0, h = 0, sms = 148, fmt = DBK_FMT_F16;
  Buf<float> x, out;
  Buf<std::uint16_t> Y;  // 16-bit expert outputs, padded rows
  Buf<std::uint8_t> A, H;
  Buf<std::uint16_t> w1, w2;  // all experts, tiled
  Buf<const void*> w1tab, w2tab;
  Buf<std::int32_t> pstart, tile_expert, tile_rb, n_tiles, row_of_item;
};

MoeBf16::MoeBf16(const MoeConfig& cfg, std::int64_t T, std::uint64_t expert_seed, int fmt, cudaStream_t s)
    : impl_(std::make_unique<Impl>()) {
  Impl& I = *impl_;
  I.T = T;
  I.fmt = fmt;
  I.n = static_cast<int>(cfg.experts);
  I.k = static_cast<int>(cfg.active_per_example);
  I.d = static_cast<int>(cfg.data_dim);
  I.h = static_cast<int>(cfg.hidden);
  if (I.d % 256 != 0 || I.h % 256 != 0) {
    throw_error(Errc::invalid_argument, "tensor-core MoE path needs data_dim and hidden multiples of 256");
  }
  I.sms = sm_count();
  const std::int64_t rows = T * I.k + static_cast<std::int64_t>(I.n) * 256;  // experts padded to 256 rows
  I.x.alloc(static_cast<size_t>(T) * I.d);
  I.A.alloc(static_cast<size_t>(rows) * I.d * 2);
  I.H.alloc(static_cast<size_t>(rows) * I.h * 2);
  I.Y.alloc(static_cast<size_t>(rows) * I.d);
  I.out.alloc(static_cast<size_t>(T) * I.d);
  I.pstart.alloc(static_cast<size_t>(I.n) + 1);
  I.tile_expert.alloc(static_cast<size_t>(rows / 128 + 1));
  I.tile_rb.alloc(static_cast<size_t>(rows / 128 + 1));
  I.n_tiles.alloc(1);
  I.row_of_item.alloc(static_cast<size_t>(T) * I.k);
  upload_expert_weights(cfg, expert_seed, 0, I.n, fmt, I.w1, I.w2, I.w1tab, I.w2tab, s);
}

MoeBf16::~MoeBf16() = default;

void MoeBf16::upload_inputs(const float* x, cudaStream_t s) {
  check(cudaMemcpyAsync(impl_->x.get(), x, sizeof(float) * static_cast<size_t>(impl_->T) * impl_->d,
                        cudaMemcpyHostToDevice, s), "H2D inputs");
}

int MoeBf16::forward(const std::int32_t* ids, const double* wts, const std::int32_t* order,
                     const std::int32_t* offsets, cudaStream_t s, Profiler* prof, const float* x, float* out) {
  Impl& I = *impl_;
  if (!x) x = I.x.get();
  if (!out) out = I.out.get();
  const int blocks = I.sms * 8;
  if (prof) prof->begin(3, s);
  check(dbk_moe_tc_layout(I.n, offsets, I.pstart.get(), I.tile_expert.get(), I.tile_rb.get(), I.n_tiles.get(), s),
        "moe layout");
  check(dbk_moe_tc_dispatch(I.fmt, I.T, I.k, I.d, order, ids, offsets, I.pstart.get(), x, I.A.get(),
                              I.row_of_item.get(), blocks, s),
        "moe dispatch");
  if (prof) prof->end(s);
  if (prof) prof->begin(4, s);
  check(dbk_moe_tc_gemm(I.fmt, 0, I.n, I.d, I.h, I.n_tiles.get(), I.tile_expert.get(), I.tile_rb.get(), I.A.get(),
                          I.w1tab.get(), I.H.get(), nullptr, 0, -1, nullptr, I.sms, s),
        "moe gemm1");
  if (prof) prof->end(s);
  if (prof) prof->begin(5, s);
  check(dbk_moe_tc_gemm(I.fmt, 1, I.n, I.h, I.d, I.n_tiles.get(), I.tile_expert.get(), I.tile_rb.get(), I.H.get(),
                          I.w2tab.get(), nullptr, I.Y.get(), 0, -1, nullptr, I.sms, s),
        "moe gemm2");
  if (prof) prof->end(s);
  if (prof) prof->begin(6, s);
  check(dbk_moe_tc_combine(I.fmt, I.T, I.k, I.d, wts, I.row_of_item.get(), I.Y.get(), out, s), "moe combine");
  if (prof) prof->end(s);
  return 5;
}

float* MoeBf16::inputs_device() { return impl_->x.get(); }
const float* MoeBf16::outputs_device() const { return impl_->out.get(); }

void MoeBf16::download_outputs(float* out, cudaStream_t s) {
  check(cudaMemcpyAsync(out, impl_->out.get(), sizeof(float) * static_cast<size_t>(impl_->T) * impl_->d,
                        cudaMemcpyDeviceToHost, s), "D2H outputs");
  check(cudaStreamSynchronize(s), "sync");
}

}  // namespace dynbatch::dev
