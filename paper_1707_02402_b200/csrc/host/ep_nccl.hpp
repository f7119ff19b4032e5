// ep_nccl.hpp — NCCL for the expert-parallel MoE exchange:
// the library loads libnccl.so.2 at first use (the copy already in the
// process when a framework brought one, else the system's), so
// libdynbatch.so has no link-time NCCL dependency and single-GPU users never
// load it. Plus the exchange plan: which rows go to / come from each peer,
// per expert range, from the count matrices.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <utility>
#include <vector>

namespace dynbatch::dev {

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  // Loaded once per process; throws (→ DB_ERR_INTERNAL) when NCCL is absent.
  static const Nccl& get();
  void check(ncclResult_t r, const char* what) const;
};

// Exchange plan of one rank for one forward (the C++ twin of
// paper_1707_02402_b200/moe_ep.py pieces / chunk_bounds).
//   send side: this rank's rows in sorted order = blocks [destination q]
//              [q's local expert e] (send_counts[q·E + e]);
//   recv side: blocks [source q][local expert e] (recv_counts[q·E + e]).
// Local experts are cut into C contiguous ranges; piece (c, q) of either
// buffer is the contiguous slice of peer q's block covering range c.
struct EpPlan {
  int G = 1, E = 0, C = 1;
  std::vector<std::pair<int, int>> bounds;  // [C] local-expert ranges
  std::vector<std::int64_t> s_off, s_rows;  // [C·G] send pieces (rows)
  std::vector<std::int64_t> r_off, r_rows;  // [C·G] receive pieces (rows)
  std::int64_t send_total = 0, recv_total = 0;
};
std::vector<std::pair<int, int>> ep_chunk_bounds(int E, int chunks);
EpPlan make_ep_plan(int G, int E, const std::int32_t* send_counts, const std::int32_t* recv_counts, int chunks);

}  // namespace dynbatch::dev
