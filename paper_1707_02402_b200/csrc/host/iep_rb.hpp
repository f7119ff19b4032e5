// iep_rb.hpp — device state of the Tier-B residual-block IEP path.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <vector>

#include "device.hpp"

namespace dynbatch::dev {

struct IepSession::RB {
  static constexpr int kFmap = 25088;  // floats per 128×14×14 plane map
  static constexpr int kTileM = 256;
  static constexpr int kGuard = 32;
  static constexpr int kLead = 16;  // zero rows before each segment's first image (rb_conv.cu)
  std::int64_t plane_stride = 0;  // staging positions per plane
  Buf<float> inputs;              // [b][kFmap] plane maps
  Buf<float> values;              // [N][kFmap] node values (and parked z)
  Buf<float> chw_in, chw_out;     // reference-layout rows for host I/O
  Buf<std::uint16_t> stage_x, stage_lo, stage_cat, stage_mid;  // fp16 staging (hi, lo, [x; y], mid)
  Buf<std::uint16_t> ident;  // two 16 KB identity weight blocks (residual through the MMA)
  std::vector<Buf<std::uint16_t>> wbuf;              // packed fp16 weights
  std::vector<Buf<float>> bbuf;
  Buf<const void*> w0tab, w1tab, w2tab;
  Buf<const float*> b0tab, b1tab, b2tab;
  Buf<std::int32_t> seg_start, group_tile0, group_bintile0, step_tile_begin, step_bintile_begin,
      step_positions, tile_group, tile_q0, bin_group, bin_q0, fwd_ok, fwd_pos, fwd_slot;
  // cross-step dependencies: the parent a node's image is forwarded to, and
  // per node the conv3x3 #2 tiles its operand images need / have received
  Buf<std::int32_t> fwd_parent, need, ready;
  Buf<std::uint64_t> memtab;  // per-member epilogue metadata, 32 bytes each (rb_conv.cu MemberEntry)
  Buf<std::uint64_t> tasks;   // gather tasks, 32 bytes each: 2 lists × task_cap
  Buf<std::int32_t> n_tasks;
  std::int64_t task_cap = 0;
  Buf<std::int32_t> done0, done1, queue;  // fused step kernel: tile done flags, claim counters
  Buf<std::int32_t> order, order_prefix;  // per-step claim order of the work units (dbk_rb_order)
  Buf<std::int32_t> step_done;            // per step: conv3x3 #2 tiles finished (one-launch forwards)
  std::int32_t epoch = 1;                 // done-flag stamp (flags are cleared every forward)
  // forward_host_async: copy streams, triple-buffered CHW rows, events
  struct Pipe {
    cudaStream_t h2d = nullptr, d2h = nullptr;
#ifndef DYNBATCH_PIPE_DEPTH
#define DYNBATCH_PIPE_DEPTH 3
#endif
    static constexpr int kDepth = DYNBATCH_PIPE_DEPTH;  // calls in flight (slack for host and link jitter)
    Buf<float> in[kDepth], out[kDepth];
    cudaEvent_t h2d_done[kDepth] = {}, in_free[kDepth] = {}, out_ready[kDepth] = {}, out_free[kDepth] = {};
    std::uint64_t calls = 0;
    // set_programs while pipelined: the sequences wait in pinned staging
    // slot (calls % kDepth) and ride the next call's input upload on the h2d
    // stream; the build runs on the main stream after that upload
    Pinned<std::int32_t> tok_pin[kDepth], off_pin[kDepth];
    Buf<std::int32_t> tok[kDepth], off[kDepth];
    bool programs_pending = false;
    // DYNBATCH_PIPE_TRACE: timing events per call (h2d start/end, main
    // start/forward end, d2h start/end), printed by sync_pipeline()
    bool trace = false;
    std::vector<std::array<cudaEvent_t, 6>> tev;
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
  std::int64_t n_expensive = 0;
  std::int64_t n_shared = 0;  // expensive children with several parents (gathered per step)
  int tile_m = kTileM;  // positions per scheduled tile (256, or 128 for small batches)
};

}  // namespace dynbatch::dev
