// iep_head.hpp — the IEP classifier head on the root feature maps
// (head.cu has the definition). Host side: reference-style
// weight init, fp16 pre-tiled GEMM operands, device buffers, and the launch
// sequence pack → GEMM(proj) → pool → GEMM(FC1) → GEMM(FC2).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "device.hpp"

namespace dynbatch::dev {

// Weights as fp64, input-major (w[k·N + n]): the init the oracle restates
// (oracle/dynbatch_oracle.c orc_head_weights): Rng(mix_seed(seed, 0x4ead)),
// draws wp, bp, w1, b1, w2, b2, each uniform(-0.5, 0.5)/sqrt(fan_in)
// (src/modules.cpp:13-28 style).
struct HeadWeights {
  int C = 128, P = 512, F = 1024, A = 28;
  std::vector<double> wp, bp, w1, b1, w2, b2;
};
HeadWeights make_head_weights(int C, int P, int F, int A, std::uint64_t seed);

class IepHead {
 public:
  static constexpr int kP = 512, kF = 1024, kPad = 256;  // projection, hidden width, padded logit columns
  IepHead(int answers, std::uint64_t seed, cudaStream_t s);
  // Logits of b roots (root tables and maps as the resblock session keeps
  // them); returns kernels launched.
  int forward(std::int64_t b, const std::int32_t* root_g, const std::int32_t* fid, const std::int32_t* arity_of,
              const std::int32_t* example, const float* inputs, const float* values, cudaStream_t s);
  const float* logits() const { return logits_.get(); }  // [b][kPad] fp32, columns < answers valid
  int answers() const { return answers_; }
  // 2·(196·128·P + 49·P·F + F·A) per program
  double flops_per_program() const;
  void download(std::int64_t b, float* out, cudaStream_t s) const;  // [b][answers]
  // The backward's operands: the last forward's 16-bit activations (tiled as
  // the GEMMs read / wrote them) and fp32 input-major weights.
  const void* roots_tiled() const { return a0_.get(); }   // SW128 rows e·196 + px, K = 128
  const void* proj_tiled() const { return h1_.get(); }    // H layout rows e·196 + px, K = P
  const void* pooled_tiled() const { return a1_.get(); }  // SW128 rows e, K = 49·P
  const void* hidden_tiled() const { return h2_.get(); }  // H layout rows e, K = F
  const float* wp32() const { return wp32_.get(); }       // [C][P]
  const float* w1_32() const { return w132_.get(); }      // [49P][F]
  const float* w2_32() const { return w232_.get(); }      // [F][answers]
  // SGD on the head (fp32 masters, then the GEMMs' fp16 tiles rebuilt);
  // gradients as IepSession::download_grad's head entries
  void sgd(float lr, const float* gwp, const float* gbp, const float* gw1, const float* gb1, const float* gw2,
           const float* gb2, cudaStream_t s);

 private:
  void size_for(std::int64_t b, cudaStream_t s);
  int answers_;
  int sms_ = 148;
  std::int64_t cap_b_ = 0;
  Buf<std::uint16_t> wp_, w1_, w2_;
  Buf<float> bp_, b1_, b2_;
  Buf<float> wp32_, w132_, w232_;
  Buf<const void*> wtab_;        // [wp, w1, w2]
  Buf<const float*> btab_;       // [bp, b1, b2]
  Buf<std::uint16_t> a0_, h1_, a1_, h2_;
  Buf<float> logits_;
  Buf<std::int32_t> zeros_, iota_, ntiles_;  // tile lists (one group) and tile counts [proj, fc]
  std::int64_t tiles_b_ = -1;
};

}  // namespace dynbatch::dev
