// moe_bf16.hpp — 16-bit tensor-core MoE expert path (grouped tcgen05 GEMMs),
// fp16 (DBK_FMT_F16, the precise mode) or bf16 (DBK_FMT_BF16) operands.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "device.hpp"

namespace dynbatch::dev {

// An N × K GEMM operand stored input-major (w[kk·N + n]) → 16-bit (fmt)
// [N/256][K/64] tiles of 32 KB for the grouped tcgen05 GEMM (moe_gemm.cu).
void tile_weights(const std::vector<double>& w, int K, int N, int fmt, std::uint16_t* out);

// ExpertSet experts [e_first, e_first + n_local) (src/moe.cpp:71-88) as
// 16-bit (fmt) pre-tiled GEMM operands, with device tables of per-expert
// pointers.
void upload_expert_weights(const MoeConfig& cfg, std::uint64_t expert_seed, int e_first, int n_local, int fmt,
                           Buf<std::uint16_t>& w1, Buf<std::uint16_t>& w2, Buf<const void*>& w1tab,
                           Buf<const void*>& w2tab, cudaStream_t s);

class MoeBf16 {
 public:
  MoeBf16(const MoeConfig& cfg, std::int64_t T, std::uint64_t expert_seed, int fmt, cudaStream_t s);
  ~MoeBf16();
  void upload_inputs(const float* x, cudaStream_t s);
  // Dispatch → GEMM1+ReLU → GEMM2 → combine; returns kernels launched.
  // x / out: device rows to read / write instead of the session's own
  // (the pipelined host path's per-call slots); null = the session's.
  int forward(const std::int32_t* ids, const double* wts, const std::int32_t* order,
              const std::int32_t* offsets, cudaStream_t s, Profiler* prof, const float* x = nullptr,
              float* out = nullptr);
  void download_outputs(float* out, cudaStream_t s);
  float* inputs_device();
  const float* outputs_device() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

}  // namespace dynbatch::dev
