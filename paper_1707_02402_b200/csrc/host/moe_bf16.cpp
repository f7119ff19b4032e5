// moe_bf16.cpp — host side of the bf16 grouped-GEMM MoE path.
#include "moe_bf16.hpp"

#include "device.hpp"

namespace dynbatch::dev {

struct MoeBf16::Impl {};

MoeBf16::MoeBf16(const MoeConfig&, std::int64_t, std::uint64_t, cudaStream_t) {
  throw std::runtime_error("bf16 MoE path not built yet");
}
MoeBf16::~MoeBf16() = default;
void MoeBf16::upload_inputs(const float*, cudaStream_t) {}
int MoeBf16::forward(const std::int32_t*, const double*, const std::int32_t*, const std::int32_t*, cudaStream_t, Profiler*) { return 0; }
void MoeBf16::download_outputs(float*, cudaStream_t) {}

}  // namespace dynbatch::dev
