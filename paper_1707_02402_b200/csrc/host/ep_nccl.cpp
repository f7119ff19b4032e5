// ep_nccl.cpp — runtime-loaded NCCL and the expert-parallel exchange plan.
#include "ep_nccl.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>

#include "dynbatch.hpp"

namespace dynbatch::dev {

namespace {
template <typename F>
void bind(void* lib, F& fn, const char* name) {
  fn = reinterpret_cast<F>(dlsym(lib, name));
  if (!fn) throw std::runtime_error(std::string("NCCL symbol ") + name + " not found");
}
}  // namespace

const Nccl& Nccl::get() {
  static Nccl n;
  static std::once_flag once;
  static std::string error;
  std::call_once(once, [] {
    const char* env = std::getenv("DYNBATCH_NCCL_LIB");
    void* lib = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      error = std::string("cannot load NCCL (") + (env ? env : "libnccl.so.2") + "): " + dlerror();
      return;
    }
    try {
      bind(lib, n.GetUniqueId, "ncclGetUniqueId");
      bind(lib, n.CommInitRank, "ncclCommInitRank");
      bind(lib, n.CommDestroy, "ncclCommDestroy");
      bind(lib, n.Send, "ncclSend");
      bind(lib, n.Recv, "ncclRecv");
      bind(lib, n.GroupStart, "ncclGroupStart");
      bind(lib, n.GroupEnd, "ncclGroupEnd");
      bind(lib, n.GetErrorString, "ncclGetErrorString");
    } catch (const std::exception& e) {
      error = e.what();
    }
  });
  if (!error.empty()) throw std::runtime_error(error);
  return n;
}

void Nccl::check(ncclResult_t r, const char* what) const {
  if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + GetErrorString(r));
}

std::vector<std::pair<int, int>> ep_chunk_bounds(int E, int chunks) {
  const int C = std::max(1, std::min(chunks, E));
  std::vector<std::pair<int, int>> b;
  for (int c = 0; c < C; ++c) b.emplace_back(E * c / C, E * (c + 1) / C);
  return b;
}

EpPlan make_ep_plan(int G, int E, const std::int32_t* send_counts, const std::int32_t* recv_counts, int chunks) {
  EpPlan p;
  p.G = G;
  p.E = E;
  p.bounds = ep_chunk_bounds(E, chunks);
  p.C = static_cast<int>(p.bounds.size());
  const size_t cg = static_cast<size_t>(p.C) * G;
  p.s_off.assign(cg, 0);
  p.s_rows.assign(cg, 0);
  p.r_off.assign(cg, 0);
  p.r_rows.assign(cg, 0);
  auto fill = [&](const std::int32_t* cnt, std::vector<std::int64_t>& off, std::vector<std::int64_t>& rows) {
    std::int64_t peer0 = 0;
    for (int q = 0; q < G; ++q) {
      std::vector<std::int64_t> pre(static_cast<size_t>(E) + 1, 0);  // prefix over q's local experts
      for (int e = 0; e < E; ++e) pre[static_cast<size_t>(e) + 1] = pre[static_cast<size_t>(e)] + cnt[q * E + e];
      for (int c = 0; c < p.C; ++c) {
        const auto [e0, e1] = p.bounds[static_cast<size_t>(c)];
        off[static_cast<size_t>(c) * G + q] = peer0 + pre[static_cast<size_t>(e0)];
        rows[static_cast<size_t>(c) * G + q] = pre[static_cast<size_t>(e1)] - pre[static_cast<size_t>(e0)];
      }
      peer0 += pre[static_cast<size_t>(E)];
    }
    return peer0;
  };
  p.send_total = fill(send_counts, p.s_off, p.s_rows);
  p.recv_total = fill(recv_counts, p.r_off, p.r_rows);
  return p;
}

}  // namespace dynbatch::dev
