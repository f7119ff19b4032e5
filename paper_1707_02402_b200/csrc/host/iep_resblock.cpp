// iep_resblock.cpp — Tier-B residual conv module path of the IEP session.
#include "device.hpp"
#include "iep_rb.hpp"

namespace dynbatch::dev {


IepSession::~IepSession() {
  for (cudaEvent_t e : step_events_) cudaEventDestroy(e);
  if (stream_) {
    cudaStreamSynchronize(stream_);
    cudaStreamDestroy(stream_);
  }
}


void IepSession::init_resblock(const TensorBatch&, std::uint64_t) {
  throw std::runtime_error("resblock path not built yet");
}
void IepSession::forward_resblock() {}
void IepSession::upload_resblock_inputs(const float*) {}
void IepSession::download_resblock_outputs(float*) {}
void IepSession::forward_host(const float* inputs, float* outputs) {
  if (kind_ != ModuleKind::resblock) throw_error(Errc::invalid_argument, "forward_host needs a resblock session");
  upload_resblock_inputs(inputs);
  forward();
  download_resblock_outputs(outputs);
}

}  // namespace dynbatch::dev
