// rb_conv.cu — Tier-B IEP module bodies: residual conv blocks on 128×14×14
// feature maps as tcgen05/TMEM implicit-GEMM kernels (sm_100a).
//
// Module (north star; no reference implementation — SPEC.md:268-269):
//   unary  y = relu(x + conv3x3_2(relu(conv3x3_1(x) + b1)) + b2)
//   binary z = relu(conv1x1([x; y]) + b0), then the unary block on z.
// Executor semantics around it follow src/executor.cpp:117-166 (gather child
// k as operand k, apply, scatter to the member's slot); leaves alias the
// example's input map instead of being copied.
//
// Data layout:
//   * fp32 "plane maps" [16 planes][196 px][8 ch] (plane j = channels
//     8j..8j+7), 100,352 B per map: the inputs, and the values of roots and
//     of children shared by several parents (the only values read later);
//   * per-step staging: fp16 rows over a packed position axis. Each image
//     occupies a 15×15 grid (225 positions; row 14 and column 14 are zero
//     pads shared with the next image / row), so a 3×3 tap (dh, dw) is the
//     row shift dh·15 + dw of the same array. Images of one call group are
//     contiguous; each group's segment starts on a TILE_M boundary so a CTA
//     tile never mixes weights. A 64-channel chunk c of staging row
//     r = GUARD + q is one 128-byte row at (c·PS + r)·128, its 8 planes
//     (8 channels, 16 B each) XOR-swizzled: plane j at ((j ^ (r & 7))·16) —
//     the 128-byte-swizzle K-major canonical layout keyed to the row, so a
//     window of consecutive rows is ONE bulk copy that lands correctly
//     swizzled in shared memory (window starts are 8-row aligned). A block
//     input x is staged twice: hi = fp16(x) in stage_x (the conv3x3 #1
//     operand) and lo = fp16(x − hi) in stage_lo; hi + lo carries x to
//     ≈2^-22 relative (fp32-equivalent);
//   * tensor-core operands use SWIZZLE_128B K-major descriptors with base
//     offset 0: the swizzle is keyed to absolute shared-memory addresses, so
//     a descriptor may start at ANY row of the window (tools/sw128_test.cu)
//     and all nine taps read the same window at different row offsets — the
//     im2col never materialises.
//
// The residual is added on the tensor cores: conv3x3 #2 accumulates
// W2·mid + I·hi + I·lo (I = identity weight blocks, exact products, fp32
// accumulation), so every operand arrives by TMA and every epilogue is
// store-only: bias, ReLU, fp16 hi/lo images for the parent's call and fp32
// values only where a later reader needs them.
//
// One persistent launch per step (k_rb_step, one CTA per SM) runs the
// step's conv1x1, conv3x3 #1 and conv3x3 #2 tiles from a device work queue:
//   warp 0   — scheduler + window producer: claims items, waits for the
//              tiles an item's window reads (done flags), bulk-copies (TMA
//              engine) the activation window per 64-channel K chunk;
//   warp 1   — TMEM allocator + single-thread tcgen05.mma issuer:
//              D[128 out channels][256 positions] (M = 128, N = 256, K = 16),
//              A = weight stage, B = window at the tap's row shift;
//   warps 2-9 — epilogue: tcgen05.ld (lane = channel), 8×8 lane transposes
//              to position-major 16-byte vectors, bias, ReLU, stores;
//   warp 10  — fills each tile's per-position table (targets, validity)
//              ahead of the epilogue;
//   warp 11  — streams the weight stages, decoupled from the windows.
// Accumulators are double-buffered in TMEM (2 × 256 columns) so the epilogue
// of one tile overlaps the MMAs of the next.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <atomic>
#include <cstdlib>

#include "dynbatch/dbk.h"
#include "tc_common.cuh"

namespace {

using namespace dbk;

constexpr int kC = 128;                    // channels
constexpr int kPlanes = kC / 8;            // 16
constexpr int kImg = 225;                  // 15 × 15 packed grid per image
constexpr int kPx = 196;                   // 14 × 14
constexpr int kFmap = kPlanes * kPx * 8;   // 25,088 floats per node map
constexpr int kGuard = 32;                 // zero positions before position 0
constexpr int kTileM = 256;                // positions per CTA tile (MMA N); the kernel also runs 128 (TM)
constexpr int kHalo = 16;                  // 3×3 window halo (15 + 1 positions)
constexpr int kLead = 16;                  // zero rows before a segment's first image (its top / left pads)
#ifndef DYNBATCH_CLUSTER
#define DYNBATCH_CLUSTER 2
#endif
// CTAs per cluster: the two CTAs of a pair take the two tiles of one tile
// pair (same segment, same weights) and each loads half of every weight
// stage, multicast to both — half the L2→SM weight traffic per CTA.
constexpr int kCluster = DYNBATCH_CLUSTER;
static_assert(kCluster == 1 || kCluster == 2, "cluster of 1 or 2 CTAs");
constexpr int kWin = kTileM + 2 * kHalo;   // window rows (row stride of every A slot)
constexpr int kChunkPlanes = 8;            // K chunk = 64 input channels = 8 planes
constexpr int kASlot = kWin * 128;         // 36 KB activation window slot (rows of 128 B)
#ifndef DYNBATCH_ASLOTS
#define DYNBATCH_ASLOTS 4
#endif
#ifndef DYNBATCH_BSTAGES
#define DYNBATCH_BSTAGES 4
#endif
constexpr int kASlots = DYNBATCH_ASLOTS;   // window slots (short hi/lo and 1×1 chunks need depth)
constexpr int kBStage = 128 * 64 * 2;      // 16 KB: 128 out channels × K=64 fp16 weight block
constexpr int kBStages = DYNBATCH_BSTAGES;
#ifndef DYNBATCH_EPI_WARPS
#define DYNBATCH_EPI_WARPS 8
#endif
constexpr int kEpiWarps = DYNBATCH_EPI_WARPS;  // 8: two warps per TMEM lane quarter (128 positions each); 16: four
constexpr int kEpiParts = kEpiWarps / 4;       // column parts per lane quarter
static_assert(kEpiWarps == 8 || kEpiWarps == 16, "8 or 16 epilogue warps");
constexpr int kTableWarp = 2 + kEpiWarps;  // fills the per-tile position tables ahead of the epilogue
constexpr int kWeightWarp = kTableWarp + 1;  // streams the weight stages
constexpr int kThreads = (kWeightWarp + 1) * 32;
constexpr int kItemSlots = 4;              // work items in flight between the roles
constexpr int kChunk = 16;                 // positions per epilogue chunk
template <int TM>
constexpr int kChunksT = TM / kEpiParts / kChunk;  // 16-position chunks per epilogue warp and tile

// Per-member epilogue metadata (schedule order), built once per forward by
// k_rb_memtab from the forwarding tables.
struct MemberEntry {
  float* slot;       // the node's fp32 plane map (written only when keep32)
  int32_t fwd_row;   // staging row of the parent's operand image of this node (position 0), −1: none
  int32_t fwd_buf;   // 0: stage_x (+ lo in stage_lo), 1 / 2: stage_cat operand 0 / 1 (chunks 0-1 / 2-3)
  int32_t keep32;    // a later reader needs the fp32 value (root, shared child)
  int32_t parent;    // node whose operand image this node's conv3x3 #2 tiles fill (fwd_row ≥ 0), else −1
  int32_t pad[2];
};

// One gathered operand (leaf input map or shared child's value → a member's
// staged image), emitted by k_rb_memtab.
struct GatherTask {
  const float* src;  // fp32 plane map
  int64_t row;       // staging row of the member's image (position 0)
  int32_t buf;       // 0: stage_x (+ lo), 1 / 2: stage_cat operand 0 / 1
  int32_t step;      // shared children: the member's step (leaves: unused)
  int64_t pad;
};

// Per-position epilogue table of one tile.
struct PosEntry {
  float* dst;       // fp32 store target (plane 0 of this pixel) or null
  int32_t fwd_row;  // staging row of the forwarded image at this position, −1: none
  int32_t fwd_buf;  // as MemberEntry::fwd_buf
  int32_t valid;    // a real pixel of a real member
  int32_t pad;
};
// Per-tile extras next to the position table: the tile's bias vector and
// the nodes whose operand images a conv3x3 #2 tile completes (its publish).
struct TileExtra {
  float bias[kC];
  int32_t parent[4];  // −1: none
};
constexpr int kTableBytes = 2 * kTileM * static_cast<int>(sizeof(PosEntry)) +
                            2 * static_cast<int>(sizeof(TileExtra));  // double-buffered

// A claimed work item with the group metadata every role needs, loaded once
// by the scheduler (the other roles read it from shared memory instead of
// chasing group → function → weight / bias pointers in global memory at every
// tile and phase start).
struct Item {
  int32_t kind;  // 0 conv1x1, 1 conv3x3 #1, 2 conv3x3 #2, -1 end
  int32_t tile;  // global tile index (bin-tile list for kind 0)
  int32_t g, q0;
  int32_t step;
  int32_t gb0;     // group_begin[g]: the group's first member
  int32_t rows;    // members (images) in the group's segment
  int32_t seg;     // seg_start[g]: absolute staging row of the first image
  int32_t binary;  // the group has conv1x1 tiles (binary function)
  int32_t bin_t0;  // binary: the step's first bin tile of this group
  int32_t tile_t0;  // the step's first (conv3x3) tile of this group
  const uint8_t* w;   // weights of the tile's conv (conv3x3 #2: W2)
  const float* bias;  // bias of the tile's conv
};

struct StepParams {
  int32_t step, step_end;  // the launch runs steps [step, step_end), step s + 1 after all of step s
  int32_t epoch, lookahead, debug;
  int32_t diag;  // timing diagnostics only (wrong results): bit 0 skips weight reloads, bit 1 window
                 // reloads, bit 2 the epilogue work (TMEM loads, transposes, stores), bit 3 only its stores,
                 // bit 4 aims the stores at one L2-resident slot, bit 5 skips every dependency wait,
                 // bit 6 drops the weight-stage handshake (MMAs read stale stages), bit 7 the window one
  int32_t cache;  // bit 2: drop consumed interior mid lines from L2 (discard; default on), bit 3: also the
                  // block input's hi / lo lines
  const int32_t* step_tile_begin;
  const int32_t* tile_group;
  const int32_t* tile_q0;
  const int32_t* step_bintile_begin;
  const int32_t* bin_group;
  const int32_t* bin_q0;
  const int32_t* group_fid;
  const int32_t* group_begin;
  const int32_t* seg_start;
  const int32_t* group_tile0;
  const int32_t* group_bintile0;
  const MemberEntry* memtab;
  uint8_t* stage_x;    // block inputs (hi) / conv1x1 output z (hi)
  uint8_t* stage_lo;   // their lo images
  uint8_t* stage_cat;  // binary operands [x; y] (hi)
  uint8_t* stage_mid;  // conv3x3 #1 output
  int64_t ps;          // plane stride in positions
  const uint8_t* const* wpack[3];
  const float* const* bias[3];
  const uint8_t* ident;  // two 16 KB identity blocks (the residual's weights)
  int32_t* done0;        // per bin tile: conv1x1 done (== epoch)
  int32_t* done1;        // per tile: conv3x3 #1 done (== epoch)
  int32_t* step_done;    // per step: conv3x3 #2 tiles completed (zeroed each forward)
  int32_t* queue;        // claim counters, one per launch's first step (zeroed each forward)
  int32_t* err;          // first error code (kErrNonFinite / kErrRange), 0 = none
  // Cross-step dependencies per operand image instead of a step barrier:
  // ready[node] counts the conv3x3 #2 tiles of the node's forwarded
  // children that have filled their part of its operand images; need[node]
  // is their total (dbk_rb_memtab). A tile of a later step starts once the
  // images its windows read are complete.
  int32_t* ready;         // zeroed each forward
  const int32_t* need;
  const int32_t* member_g;
  int32_t step_barrier;   // 1: also wait for the whole previous step (A/B)
  // Claim order per step (k_rb_order), units of kCluster tiles: entry
  // (kind << 28) | local unit; null = the closed form of step_unit().
  const int32_t* order;
  // bounds of the node values (DYNBATCH_BOUNDS builds check every store)
  const float* values;
  int64_t values_floats;
};

// Error codes shared with the host (IepSession::check_errors): a module
// produced a non-finite row (src/executor.cpp:156-159; ReLU as max maps NaN
// to 0 like the reference's `v > 0 ? v : 0`, so this is +inf) or a value
// beyond the fp16 operand range the next block stages it in (the epilogue
// sees both as an fp16 inf), or an input is outside that range (gather).
constexpr int32_t kErrNonFinite = 9;
constexpr int32_t kErrRange = 10;

// Two error codes → one (non-finite outranks range; 0 = none).
__device__ __forceinline__ int32_t merge_code(int32_t a, int32_t b) {
  return (a == kErrNonFinite || b == kErrNonFinite) ? kErrNonFinite : (a | b);
}

// Running max of the eight fp16 values of a staged 16-byte vector.
__device__ __forceinline__ __half2 hmax4(__half2 m, const uint4& v) {
  const __half2* h = reinterpret_cast<const __half2*>(&v);
  return __hmax2(__hmax2(m, __hmax2(h[0], h[1])), __hmax2(h[2], h[3]));
}

// 0, kErrRange or kErrNonFinite for 8 values about to become fp16 operands.
__device__ __forceinline__ int32_t range_code(const float* o) {
  int32_t c = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float a = fabsf(o[k]);
    if (!(a <= 65504.f)) c = merge_code(c, (a == INFINITY || a != a) ? kErrNonFinite : kErrRange);
  }
  return c;
}

// Wait accounting (read/reset with dbk_rb_debug()): slot 3 = MMA thread
// [drained accumulator, A window, weight stage, loop total]; slot 4 =
// window producer [item ring, dependency flags, free window slot, total].
// Slots 24-35: MMA thread per tile kind k (0 conv1x1, 1 conv3x3 #1, 2 conv3x3
// #2): [24 + 4k] item cycles, [+1] window (A) waits, [+2] weight (B) waits,
// [+3] accumulator (epilogue) waits; 36-41: epilogue per kind [36 + 2k]
// cycles from accumulator ready to published, [+1] tiles; 42-44: producer
// dependency waits per kind.
__device__ unsigned long long g_conv_dbg[64];

// ------------------------------------------------------------ K phases
// A tile's K loop is one to three phases of (window source, weights, chunks,
// taps, halo): conv1x1 [x; y] (4 chunks × 1 tap); conv3x3 #1 over x
// (2 × 9, halo 16); conv3x3 #2: I·hi + I·lo (2 × 1 each, no halo), then
// W2 over mid (2 × 9, halo 16).
struct Phase {
  const uint8_t* src;  // staging base (position 0 of plane 0)
  const uint8_t* w;    // weight blocks
  int chunks, taps, halo;
};

__device__ __forceinline__ int n_phases(int kind) { return kind == 2 ? 3 : 1; }

// Timing diagnostics (wrong results): diag bit 8 skips conv3x3 #2's residual
// phases (I·hi and I·lo), bit 9 only its I·lo phase.
__device__ __forceinline__ bool phase_skipped(const StepParams& P, const struct Item& it, int p) {
  return it.kind == 2 && ((p < 2 && (P.diag & 256)) || (p == 1 && (P.diag & 512)));
}

__device__ __forceinline__ Phase phase_of(const StepParams& P, const Item& it, int p) {
  if (it.kind == 0) return Phase{P.stage_cat, it.w, 4, 1, 0};
  if (it.kind == 1) return Phase{P.stage_x, it.w, 2, 9, kHalo};
  // conv3x3 #2: the residual phases first — they read this block's input
  // images, which this launch's conv3x3 #1 tiles do not write, so they load
  // and run while the producer waits for the mid tiles
  if (p == 2) return Phase{P.stage_mid, it.w, 2, 9, kHalo};
  return Phase{p == 0 ? P.stage_x : P.stage_lo, P.ident, 2, 1, 0};
}

// Tiles of a segment of `rows` images: its lead and images in 256-position
// tiles, rounded up to whole tile pairs when CTAs run in pairs (the extra
// tile has no image position: it computes zeros nobody reads).
__host__ __device__ __forceinline__ int32_t seg_tiles(int32_t rows, int32_t tile_m) {
  const int32_t nt = (kLead + rows * kImg + tile_m - 1) / tile_m;
  return (nt + kCluster - 1) / kCluster * kCluster;
}

// ------------------------------------------------------- work queue
// Queue order: all conv1x1 tiles, then conv3x3 #1 tiles interleaved with
// conv3x3 #2 tiles `lookahead` positions behind, so each SM alternates
// MMA-heavy and store-heavy tiles and a #2 tile's inputs are usually done
// when it is claimed.
// With CTA pairs, k, n0 and n1 count tile pairs and `crank` picks the tile.
// The item a claimed tile (unit `local` of `kind` in `step`, this CTA's tile
// of it) is, with the group metadata every role needs.
__device__ __forceinline__ Item item_of(const StepParams& P, int32_t step, int32_t kind, int32_t local, int32_t crank);

__device__ __forceinline__ Item step_item(const StepParams& P, int32_t step, int32_t k, int32_t n0, int32_t n1,
                                          int32_t crank) {
  if (P.order) {
    const int32_t code = P.order[(P.step_bintile_begin[step] + 2 * P.step_tile_begin[step]) / kCluster + k];
    return item_of(P, step, code >> 28, code & 0x0fffffff, crank);
  }
  int32_t kind, local;
  if (k < n0) {
    kind = 0;
    local = k;
  } else {
    const int32_t u = k - n0;
    // ≥ 2 ahead: a #2 tile's right neighbour's #1 tile is claimed before it
    const int32_t D = min(max(P.lookahead / kCluster, 2), n1);
    const int32_t R = n1 - D;
    if (u < D) {
      kind = 1;
      local = u;
    } else if (u - D < 2 * R) {
      const int32_t v = u - D;
      kind = (v & 1) ? 1 : 2;
      local = (v & 1) ? D + (v >> 1) : (v >> 1);
    } else {
      kind = 2;
      local = R + (u - D - 2 * R);
    }
  }
  return item_of(P, step, kind, local, crank);
}

__device__ __forceinline__ Item item_of(const StepParams& P, int32_t step, int32_t kind, int32_t local, int32_t crank) {
  Item it;
  it.kind = kind;
  it.step = step;
  local = local * kCluster + crank;
  if (kind == 0) {
    it.tile = P.step_bintile_begin[step] + local;
    it.g = P.bin_group[it.tile];
    it.q0 = P.bin_q0[it.tile];
  } else {
    it.tile = P.step_tile_begin[step] + local;
    it.g = P.tile_group[it.tile];
    it.q0 = P.tile_q0[it.tile];
  }
  // group metadata: independent loads, one round trip; then the weight and
  // bias pointers of the group's function
  const int32_t g = it.g;
  const int32_t f = P.group_fid[g];
  it.gb0 = P.group_begin[g];
  it.rows = P.group_begin[g + 1] - it.gb0;
  it.seg = P.seg_start[g];
  const int32_t bt = P.group_bintile0[g];
  it.binary = bt >= 0;
  it.bin_t0 = bt >= 0 ? P.step_bintile_begin[step] + bt : 0;
  it.tile_t0 = P.step_tile_begin[step] + P.group_tile0[g];
  it.w = P.wpack[kind][f];
  it.bias = P.bias[kind][f];
  return it;
}

// Images of group g whose positions overlap local rows [lo, hi) of the
// segment (local 0 = the first image's position 0; images are kImg apart).
__device__ __forceinline__ void images_overlapping(int32_t lo, int32_t hi, int32_t rows, int32_t& j0, int32_t& j1) {
  j0 = lo <= 0 ? 0 : lo / kImg;
  j1 = hi <= 0 ? -1 : min(rows - 1, (hi - 1) / kImg);
}

// Producer side: the operand images (forwarded by earlier steps' conv3x3 #2
// tiles) that overlap this item's window rows are complete: ready == need
// for each image's node. Relaxed polls, then one acquire fence.
template <int TM>
__device__ __forceinline__ void step_wait_images(const StepParams& P, const Item& it, int32_t halo) {
  const int32_t gb0 = it.gb0;
  const int32_t rows = it.rows;
  const int32_t base = it.q0 - it.seg;
  int32_t j0, j1;
  images_overlapping(base - halo, base + TM + halo, rows, j0, j1);
  bool waited = false;
  for (int32_t j = j0; j <= j1; ++j) {
    const int32_t node = P.member_g[gb0 + j];
    const int32_t nd = P.need[node];
    if (nd == 0) continue;
    waited = true;
    if (ld_relaxed_gpu(P.ready + node) >= nd) continue;
    const uint64_t t0 = global_ns();
    while (ld_relaxed_gpu(P.ready + node) < nd) {
      __nanosleep(64);
      if (global_ns() - t0 > 4000000000ull) __trap();
    }
  }
  if (waited) fence_acquire_gpu();
}

// Producer side: wait until the tiles this item's windows read are written
// in this launch (earlier launches are ordered by the stream). conv3x3 #1 of
// a binary group reads z (conv1x1 tiles i-1..i+1); conv3x3 #2 reads mid
// (conv3x3 #1 tiles i-1..i+1) and, for a binary group, z hi/lo (conv1x1
// tile i). Halo positions in other segments only feed outputs never stored.
template <int TM>
__device__ __forceinline__ void step_wait_deps(const StepParams& P, const Item& it, int phase) {
  if (P.diag & 32) return;
  const bool binary_group = it.binary;
  // operand images from earlier steps: conv1x1 reads [x; y] at its own
  // rows, conv3x3 #1 of a unary group reads x with the halo, conv3x3 #2 of a
  // unary group reads x hi / lo (the residual) at its own rows
  if (it.kind == 0) {
    step_wait_images<TM>(P, it, 0);
    fence_proxy_async_global();
    return;
  }
  if (!binary_group && (it.kind == 1 || phase == 0)) step_wait_images<TM>(P, it, it.kind == 1 ? kHalo : 0);
  const int32_t g = it.g;
  const int32_t nt = seg_tiles(it.rows, TM);
  const int32_t i = (it.q0 - it.seg + kLead) / TM;
  const bool binary = it.binary;
  const int32_t b0 = it.bin_t0;
  if (it.kind == 1) {
    if (!binary) return;
    for (int32_t j = max(i - 1, 0); j <= min(i + 1, nt - 1); ++j) wait_flag(P.done0 + b0 + j, P.epoch);
  } else if (phase == 0) {  // conv3x3 #2, residual phases: z hi/lo of a binary group
    if (!binary) return;
    wait_flag(P.done0 + b0 + i, P.epoch);
  } else {  // conv3x3 #2, W2 phase: mid of tiles i-1..i+1
    const int32_t t0 = it.tile_t0;
    for (int32_t j = max(i - 1, 0); j <= min(i + 1, nt - 1); ++j) wait_flag(P.done1 + t0 + j, P.epoch);
  }
  fence_proxy_async_global();
}

// ------------------------------------------------------------- tables
// Fills the table entries of positions lane + 32k (k = 0..7) of a tile from
// the per-member table: one independent 32-byte load per position, all
// issued before any entry is stored.
template <int TM>
__device__ __forceinline__ void rb_fill_table(const StepParams& P, const Item& it, PosEntry* tab, TileExtra* ex,
                                              int lane) {
  reinterpret_cast<float4*>(ex->bias)[lane] = __ldg(reinterpret_cast<const float4*>(it.bias) + lane);
  if (lane < 4) {
    int32_t parent = -1;
    if (it.kind == 2) {
      int32_t j0, j1;
      images_overlapping(it.q0 - it.seg, it.q0 - it.seg + TM, it.rows, j0, j1);
      if (j0 + lane <= j1) parent = P.memtab[it.gb0 + j0 + lane].parent;
    }
    ex->parent[lane] = parent;
  }
  constexpr int kPer = TM / 32;
  const int32_t gb0 = it.gb0;
  const int32_t rows = it.rows;
  const int32_t base = it.q0 - it.seg;
  MemberEntry me[kPer];
  int32_t rem[kPer], px[kPer];
  bool valid[kPer], in_img[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int32_t local = base + lane + 32 * k;  // negative in the segment's lead rows
    const int32_t img = local >= 0 ? local / kImg : rows;
    rem[k] = local - img * kImg;
    const int32_t r = rem[k] / 15, c = rem[k] - r * 15;
    in_img[k] = local >= 0 && img < rows;
    valid[k] = in_img[k] && r < 14 && c < 14;
    px[k] = r * 14 + c;
    if (it.kind == 2 && in_img[k]) me[k] = P.memtab[gb0 + img];
  }
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    PosEntry e{nullptr, -1, 0, valid[k] ? 1 : 0, 0};
    if (it.kind == 2 && in_img[k]) {
      // pad positions of a real image keep their forwarding target: the
      // epilogue writes them as zeros (any earlier layout's data is gone)
      e.dst = valid[k] && me[k].keep32 ? me[k].slot + px[k] * 8 : nullptr;
      e.fwd_row = me[k].fwd_row >= 0 ? me[k].fwd_row + rem[k] : -1;
      e.fwd_buf = me[k].fwd_buf;
    }
    tab[lane + 32 * k] = e;
  }
}

// ----------------------------------------------------------- epilogue
// 8×8 transpose across the 8 lanes of a plane group (three butterfly
// stages): in, lane e holds x[i] = D[channel 8g+e][position i]; out, lane e
// holds x[k] = D[channel 8g+k][position e].
__device__ __forceinline__ void transpose8(float* x, int e) {
#pragma unroll
  for (int s = 4; s >= 1; s >>= 1) {
    const bool up = (e & s) != 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i & s) continue;
      const float send = up ? x[i] : x[i + s];
      const float recv = __shfl_xor_sync(0xffffffffu, send, s);
      x[i] = up ? recv : x[i];
      x[i + s] = up ? x[i + s] : recv;
    }
  }
}

// hi = fp16(o), lo = fp16(o − hi) of 8 channels, as two 16-byte vectors.
__device__ __forceinline__ void split_f16x8(const float* o, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const __half2 hh = __floats2half2_rn(o[2 * j], o[2 * j + 1]);
    const float2 hf = __half22float2(hh);
    const __half2 ll = __floats2half2_rn(o[2 * j] - hf.x, o[2 * j + 1] - hf.y);
    h[j] = *reinterpret_cast<const uint32_t*>(&hh);
    l[j] = *reinterpret_cast<const uint32_t*>(&ll);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// Byte offset of plane p (16 B: 8 channels) of staging row r (chunk-row
// layout with the 128-byte swizzle, see the file header).
__device__ __forceinline__ int64_t stage_off(int64_t ps, int p, int64_t r) {
  return ((static_cast<int64_t>(p >> 3) * ps + r) << 7) + (((p & 7) ^ static_cast<int>(r & 7)) << 4);
}

// Epilogue lane geometry: TMEM lanes = output channels 32·quarter + lane,
// columns = the tile's positions; the warp covers positions
// [128·half, 128·half + 128) in eight 16-column chunks. After the transpose,
// lane (g = lane/8, e = lane%8) owns positions 8m + e (m = 0, 1) of each
// chunk with the 8 channels of plane 4·quarter + g, so every global store is
// a 16-byte vector and a warp instruction covers 4 planes × 8 positions.
struct EpiLane {
  int quarter, half, e, plane;
  int64_t chunk_off;  // (plane / 8) · PS · 128: this lane's chunk in a staging buffer
  int sub;            // (plane % 8) ^ e: swizzled 16-byte slot in own-position rows (row & 7 == e)
  int plane_off32;    // fp32 plane-map offset of this lane's plane
};

template <int KIND, int TM>
__device__ __forceinline__ void step_epilogue(const StepParams& P, const PosEntry* tab, const TileExtra* ex,
                                              const EpiLane& L, uint32_t taddr, const Item& it) {
  const float* bias_p = ex->bias + L.plane * 8;
  const float4 b_lo = *reinterpret_cast<const float4*>(bias_p);
  const float4 b_hi = *reinterpret_cast<const float4*>(bias_p + 4);
  const float bias[8] = {b_lo.x, b_lo.y, b_lo.z, b_lo.w, b_hi.x, b_hi.y, b_hi.z, b_hi.w};
  // own-position outputs (conv1x1 → z hi/lo, conv3x3 #1 → mid): row
  // kGuard + q0 + 128·half + 16·cb + 8m + e, so (row & 7) == e
  constexpr int kChunks = kChunksT<TM>;
  const int64_t own_off =
      L.chunk_off + (static_cast<int64_t>(kGuard + it.q0 + L.half * (TM / kEpiParts) + L.e) << 7) + (L.sub << 4);
  uint8_t* own = (KIND == 0 ? P.stage_x : P.stage_mid) + own_off;
  uint8_t* own_lo = P.stage_lo + own_off;
  // diag bit 4: every store lands in one L2-resident 16-byte slot per thread
  // (same instructions, no DRAM traffic)
  const bool l2sink = (P.diag & 16) != 0;
  uint8_t* const sink_slot = P.stage_mid + ((static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x) << 4);
  if (P.diag & 8) {  // timing diagnostic: TMEM loads, transposes and math, no stores
    float sink = 0.f;
#pragma unroll 2
    for (int cb = 0; cb < kChunks; ++cb) {
      float v[kChunk];
      tmem_ld16(taddr + cb * kChunk, v);
      const PosEntry* my = tab + L.half * (TM / kEpiParts) + cb * kChunk + L.e;
#pragma unroll
      for (int m = 0; m < kChunk / 8; ++m) {
        float* x = v + 8 * m;
        transpose8(x, L.e);
        const PosEntry& pe = my[8 * m];
#pragma unroll
        for (int k = 0; k < 8; ++k) sink += pe.valid ? fmaxf(x[k] + bias[k], 0.f) : 0.f;
      }
    }
    if (sink == 1.2345e-30f) *own = 0;
    return;
  }
  // largest staged fp16 operand (values ≥ 0 after the ReLU, so inf = an
  // output beyond the fp16 range or non-finite) and largest fp32 output:
  // one half2 max per packed word, checked once per tile
  __half2 hmax = __float2half2_rn(0.f);
  float fmax32 = 0.f;
#pragma unroll 2
  for (int cb = 0; cb < kChunks; ++cb) {
    float v[kChunk];
    tmem_ld16(taddr + cb * kChunk, v);
    const PosEntry* my = tab + L.half * (TM / kEpiParts) + cb * kChunk + L.e;
#pragma unroll
    for (int m = 0; m < kChunk / 8; ++m) {
      float* x = v + 8 * m;
      transpose8(x, L.e);
      const PosEntry& pe = my[8 * m];
      float o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] = pe.valid ? fmaxf(x[k] + bias[k], 0.f) : 0.f;
      const int64_t off = static_cast<int64_t>(cb * kChunk + 8 * m) << 7;
      if (KIND == 1) {
        uint4 pk;
        pk.x = pack_f16x2(o[0], o[1]);
        pk.y = pack_f16x2(o[2], o[3]);
        pk.z = pack_f16x2(o[4], o[5]);
        pk.w = pack_f16x2(o[6], o[7]);
        hmax = hmax4(hmax, pk);
        if (l2sink) st_v4(sink_slot, pk);
        else *reinterpret_cast<uint4*>(own + off) = pk;
      } else if (KIND == 0) {
        uint4 hi, lo;
        split_f16x8(o, hi, lo);
        hmax = hmax4(hmax, hi);
        if (l2sink) {
          st_v4(sink_slot, hi);
          st_v4(sink_slot, lo);
        } else {
          *reinterpret_cast<uint4*>(own + off) = hi;
          *reinterpret_cast<uint4*>(own_lo + off) = lo;
        }
      } else if (!pe.valid) {
        // pad position of a forwarded image: zero in the parent's conv3x3 #1
        // operand (its taps read the pads); lo and [x; y] pads only reach
        // outputs that are never stored
        if (pe.fwd_row >= 0 && pe.fwd_buf == 0)
          *reinterpret_cast<uint4*>(P.stage_x + stage_off(P.ps, L.plane, pe.fwd_row)) = make_uint4(0, 0, 0, 0);
      } else {
        if (pe.fwd_row >= 0) {
#ifdef DYNBATCH_BOUNDS
          if (pe.fwd_row >= P.ps) {
            atomicCAS(P.err, 0, 72);
            continue;
          }
#endif
          uint4 hi, lo;
          split_f16x8(o, hi, lo);
          hmax = hmax4(hmax, hi);
          const int p = L.plane + (pe.fwd_buf == 2 ? 16 : 0);
          const int64_t off = stage_off(P.ps, p, pe.fwd_row);
          uint8_t* hp = (pe.fwd_buf == 0 ? P.stage_x : P.stage_cat) + off;
          if (l2sink) {
            st_v4(sink_slot, hi);
            if (pe.fwd_buf == 0) st_v4(sink_slot, lo);
          } else {
            *reinterpret_cast<uint4*>(hp) = hi;
            if (pe.fwd_buf == 0) *reinterpret_cast<uint4*>(P.stage_lo + off) = lo;
          }
        }
        if (pe.dst) {
#ifdef DYNBATCH_BOUNDS
          if (pe.dst + L.plane_off32 < P.values || pe.dst + L.plane_off32 + 8 > P.values + P.values_floats) {
            atomicCAS(P.err, 0, 71);
            continue;
          }
#endif
#pragma unroll
          for (int k = 0; k < 8; ++k) fmax32 = fmaxf(fmax32, o[k]);
          float4* dp = reinterpret_cast<float4*>(pe.dst + L.plane_off32);
          const float4 d0 = make_float4(o[0], o[1], o[2], o[3]), d1 = make_float4(o[4], o[5], o[6], o[7]);
          if (l2sink) {
            st_v4(sink_slot, *reinterpret_cast<const uint4*>(&d0));
            st_v4(sink_slot, *reinterpret_cast<const uint4*>(&d1));
          } else {
            dp[0] = d0;
            dp[1] = d1;
          }
        }
      }
    }
  }
#ifndef DYNBATCH_NO_RANGE_CHECK
  const float2 hm = __half22float2(hmax);
  if ((!(fmaxf(hm.x, hm.y) <= 65504.f) || !(fmax32 <= 3.4e38f)) && P.diag == 0) atomicCAS(P.err, 0, kErrNonFinite);
#endif
}

// --------------------------------------------------------------- kernel
template <int TM, bool DBG>
__global__ void __launch_bounds__(kThreads, 1) k_rb_step(const __grid_constant__ StepParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + kASlots * kASlot;
  PosEntry* tables = reinterpret_cast<PosEntry*>(sB + kBStages * kBStage);
  TileExtra* extras = reinterpret_cast<TileExtra*>(tables + 2 * kTileM);
  Item* items = reinterpret_cast<Item*>(reinterpret_cast<uint8_t*>(tables) + kTableBytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(items + kItemSlots);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + kASlots;
  uint64_t* b_full = a_empty + kASlots;
  uint64_t* b_empty = b_full + kBStages;
  uint64_t* acc_full = b_empty + kBStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* tab_full = acc_empty + 2;
  uint64_t* tab_empty = tab_full + 2;
  uint64_t* item_full = tab_empty + 2;
  uint64_t* item_empty = item_full + kItemSlots;
  uint64_t* mail_full = item_empty + kItemSlots;  // CTA pairs: claimed pair index, leader → partner
  uint64_t* mail_empty = mail_full + kItemSlots;
  uint32_t* mail = reinterpret_cast<uint32_t*>(mail_empty + kItemSlots);
  uint32_t* tmem_slot = mail + kItemSlots;
  const uint32_t crank = kCluster > 1 ? cluster_rank() : 0;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kASlots; ++s) {
      mbar_init(a_full + s, 1);
      mbar_init(a_empty + s, 1);
    }
    for (int s = 0; s < kBStages; ++s) {
      mbar_init(b_full + s, 1);
      mbar_init(b_empty + s, kCluster);  // both CTAs' MMAs release a shared weight stage
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(acc_full + s, 1);
      mbar_init(acc_empty + s, kEpiWarps * 32);
      mbar_init(tab_full + s, 32);
      mbar_init(tab_empty + s, kEpiWarps);
    }
    for (int s = 0; s < kItemSlots; ++s) {
      mbar_init(item_full + s, 1);
      mbar_init(item_empty + s, 3 + kEpiWarps);  // MMA thread, table warp, weight warp, epilogue warps
      mbar_init(mail_full + s, 1);
      mbar_init(mail_empty + s, 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  if (kCluster > 1) cluster_sync();  // the partner's barriers exist before any remote arrive / multicast
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // work units (tiles, or tile pairs: segments hold whole pairs) of step s
  auto step_units = [&](int32_t s) {
    return (P.step_bintile_begin[s + 1] - P.step_bintile_begin[s] +
            2 * (P.step_tile_begin[s + 1] - P.step_tile_begin[s])) / kCluster;
  };

  if (warp == 0) {
    if (lane == 0) {  // ---------------------- scheduler + activation windows
      uint32_t ai = 0;
      long long w_item = 0, w_dep = 0, w_slot = 0;
      const long long t_start = clock64();
      // claims k are increasing, so the step cursor only moves forward
      int32_t cur = P.step, cur_begin = 0, cur_units = P.step < P.step_end ? step_units(P.step) : 0;
      int32_t ready = P.step;  // steps < ready have all their conv3x3 #2 tiles done (as far as we waited)
      for (int32_t n = 0;; ++n) {
        const int slot = n % kItemSlots;
        int32_t k;
        if (kCluster == 1) {
          k = atomicAdd(P.queue + P.step, 1);
        } else if (crank == 0) {  // the leader claims a pair and posts it to the partner
          k = atomicAdd(P.queue + P.step, 1);
          mbar_wait_cluster(mail_empty + slot, ((n / kItemSlots) & 1) ^ 1);
          st_remote_u32(mail + slot, 1, static_cast<uint32_t>(k));
          mbar_arrive_remote(mail_full + slot, 1);
        } else {
          mbar_wait_cluster(mail_full + slot, (n / kItemSlots) & 1);
          k = static_cast<int32_t>(*reinterpret_cast<volatile uint32_t*>(mail + slot));
          mbar_arrive_remote(mail_empty + slot, 0);
        }
        while (cur < P.step_end && k >= cur_begin + cur_units) {
          cur_begin += cur_units;
          if (++cur < P.step_end) cur_units = step_units(cur);
        }
        Item it{-1, 0, 0, 0, 0};
        if (cur < P.step_end) {
          const int32_t n0 = P.step_bintile_begin[cur + 1] - P.step_bintile_begin[cur];
          const int32_t n1 = P.step_tile_begin[cur + 1] - P.step_tile_begin[cur];
          it = step_item(P, cur, k - cur_begin, n0 / kCluster, n1 / kCluster, static_cast<int32_t>(crank));
        }
        long long c0 = DBG ? clock64() : 0;
        mbar_wait(item_empty + slot, ((n / kItemSlots) & 1) ^ 1);
        if (DBG) w_item += clock64() - c0;
        items[slot] = it;
        mbar_arrive(item_full + slot);
        if (it.kind < 0) break;
        if (P.step_barrier && it.step > ready) {
          // step s reads what step s − 1 (and earlier) wrote: wait until every
          // conv3x3 #2 tile of the previous step has published its outputs
          if (DBG) c0 = clock64();
          for (; ready < it.step; ++ready)
            wait_count(P.step_done + ready, P.step_tile_begin[ready + 1] - P.step_tile_begin[ready]);
          fence_proxy_async_global();
          if (DBG) w_dep += clock64() - c0;
        }
        for (int p = 0; p < n_phases(it.kind); ++p) {
          if (phase_skipped(P, it, p)) continue;
          if (p == 0 || p == 2) {  // conv3x3 #2 waits for the mid tiles only before its W2 phase
            if (DBG) c0 = clock64();
            step_wait_deps<TM>(P, it, p);
            if (DBG) {
              w_dep += clock64() - c0;
              atomicAdd(&g_conv_dbg[42 + it.kind], static_cast<unsigned long long>(clock64() - c0));
            }
          }
          const Phase ph = phase_of(P, it, p);
          const uint32_t rows = TM + 2 * ph.halo;
          const uint8_t* src = ph.src + (static_cast<int64_t>(kGuard + it.q0 - ph.halo) << 7);
          for (int ch = 0; ch < ph.chunks; ++ch, ++ai) {
            if (P.diag & 128) continue;  // timing: no window handshakes
            const uint32_t sa = ai % kASlots, pa = (ai / kASlots) & 1;
            const long long c1 = DBG ? clock64() : 0;
            mbar_wait(a_empty + sa, pa ^ 1);
            if (DBG) w_slot += clock64() - c1;
            if ((P.diag & 2) && ai >= kASlots) {
              mbar_arrive(a_full + sa);
              continue;
            }
            mbar_expect_tx(a_full + sa, rows * 128);
            bulk_g2s(sA + sa * kASlot, src + static_cast<int64_t>(ch) * P.ps * 128, rows * 128, a_full + sa);
          }
        }
      }
      if (DBG) {
        atomicAdd(&g_conv_dbg[16 + 0], static_cast<unsigned long long>(w_item));
        atomicAdd(&g_conv_dbg[16 + 1], static_cast<unsigned long long>(w_dep));
        atomicAdd(&g_conv_dbg[16 + 2], static_cast<unsigned long long>(w_slot));
        atomicAdd(&g_conv_dbg[16 + 3], static_cast<unsigned long long>(clock64() - t_start));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------------------------------- MMA issuer
      constexpr uint32_t IDESC = idesc_f16_f32(128, TM);
      long long w_acc = 0, w_a = 0, w_b = 0;
      const long long t_start = clock64();
      const uint64_t ns_start = DBG ? global_ns() : 0;
      uint32_t ai = 0, bi = 0;
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      for (int n = 0;; ++n) {
        const int slot = n % kItemSlots;
        mbar_wait(item_full + slot, (n / kItemSlots) & 1);
        const Item it = items[slot];
        mbar_arrive(item_empty + slot);
        if (it.kind < 0) break;
        const int abuf = n & 1;
        long long c0 = DBG ? clock64() : 0;
        const long long t_item = c0;
        const long long a0 = w_a, b0 = w_b;
        mbar_wait(acc_empty + abuf, ((n >> 1) & 1) ^ 1);
        if (DBG) {
          w_acc += clock64() - c0;
          atomicAdd(&g_conv_dbg[24 + 4 * it.kind + 3], static_cast<unsigned long long>(clock64() - c0));
        }
        tc_fence_after();
        uint32_t acc = 0;
        for (int p = 0; p < n_phases(it.kind); ++p) {
          if (phase_skipped(P, it, p)) continue;
          const int chunks = it.kind == 0 ? 4 : 2;
          const bool conv3 = it.kind == 1 || (it.kind == 2 && p == 2);
          const int taps = conv3 ? 9 : 1;
          const int halo = conv3 ? kHalo : 0;
          for (int ch = 0; ch < chunks; ++ch, ++ai) {
            const uint32_t sa = ai % kASlots, pa = (ai / kASlots) & 1;
            if (DBG) c0 = clock64();
            if (!(P.diag & 128)) mbar_wait(a_full + sa, pa);
            if (DBG) w_a += clock64() - c0;
            tc_fence_after();
            const uint32_t a_slot = a_base + sa * kASlot;
            for (int tap = 0; tap < taps; ++tap, ++bi) {
              const uint32_t s = bi % kBStages, par = (bi / kBStages) & 1;
              if (DBG) c0 = clock64();
              if (!(P.diag & 64)) mbar_wait(b_full + s, par);
              if (DBG) {
                const long long dw = clock64() - c0;
                w_b += dw;
                // [46] weight waits on a tile's first stage, [47] on the others
                atomicAdd(&g_conv_dbg[(p == 0 && ch == 0 && tap == 0) ? 46 : 47], static_cast<unsigned long long>(dw));
              }
              tc_fence_after();
              const int shift = taps == 9 ? (tap / 3 - 1) * 15 + (tap % 3 - 1) : 0;
              const uint32_t xrow = static_cast<uint32_t>(halo + shift);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const uint64_t wd = smem_desc_sw128(b_base + s * kBStage + kk * 32);
                const uint64_t xd = smem_desc_sw128(a_slot + xrow * 128 + kk * 32);
                mma_bf16(tmem_base + abuf * TM, wd, xd, IDESC, acc);
                acc = 1;
              }
              if (P.diag & 64) continue;  // timing: weight stages never handed back
              if (kCluster == 1) mma_commit(b_empty + s);
              else mma_commit_mc(b_empty + s, 0x3);  // both CTAs' copies of the stage are free
            }
            if (!(P.diag & 128)) mma_commit(a_empty + sa);
          }
        }
        mma_commit(acc_full + abuf);
        if (DBG) {
          atomicAdd(&g_conv_dbg[24 + 4 * it.kind + 0], static_cast<unsigned long long>(clock64() - t_item));
          atomicAdd(&g_conv_dbg[24 + 4 * it.kind + 1], static_cast<unsigned long long>(w_a - a0));
          atomicAdd(&g_conv_dbg[24 + 4 * it.kind + 2], static_cast<unsigned long long>(w_b - b0));
        }
      }
      if (DBG) {
        atomicAdd(&g_conv_dbg[12 + 0], static_cast<unsigned long long>(w_acc));
        atomicAdd(&g_conv_dbg[12 + 1], static_cast<unsigned long long>(w_a));
        atomicAdd(&g_conv_dbg[12 + 2], static_cast<unsigned long long>(w_b));
        atomicAdd(&g_conv_dbg[12 + 3], static_cast<unsigned long long>(clock64() - t_start));
        // effective SM clock over the loop: cycles / wall nanoseconds
        atomicAdd(&g_conv_dbg[20], static_cast<unsigned long long>(clock64() - t_start));
        atomicAdd(&g_conv_dbg[21], static_cast<unsigned long long>(global_ns() - ns_start));
      }
    }
  } else if (warp == kWeightWarp) {
    if (lane == 0) {  // -------------------------------------- weight stages
      uint32_t bi = 0;
      long long w_it = 0, w_e = 0;
      const long long t_start = DBG ? clock64() : 0;
      for (int n = 0;; ++n) {
        const int slot = n % kItemSlots;
        long long c0 = DBG ? clock64() : 0;
        mbar_wait(item_full + slot, (n / kItemSlots) & 1);
        if (DBG) w_it += clock64() - c0;
        const Item it = items[slot];
        mbar_arrive(item_empty + slot);
        if (it.kind < 0) break;
        if (P.diag & 64) continue;  // timing: no weight stages
        for (int p = 0; p < n_phases(it.kind); ++p) {
          if (phase_skipped(P, it, p)) continue;
          const Phase ph = phase_of(P, it, p);
          for (int ch = 0; ch < ph.chunks; ++ch) {
            for (int tap = 0; tap < ph.taps; ++tap, ++bi) {
              const uint32_t s = bi % kBStages, par = (bi / kBStages) & 1;
              if (DBG) c0 = clock64();
              mbar_wait(b_empty + s, par ^ 1);
              if (DBG) w_e += clock64() - c0;
              if ((P.diag & 1) && bi >= kBStages) {
                mbar_arrive(b_full + s);
                continue;
              }
              mbar_expect_tx(b_full + s, kBStage);
              const uint8_t* src = ph.w + static_cast<int64_t>(ch * ph.taps + tap) * kBStage;
              if (kCluster == 1) {
                bulk_g2s(sB + s * kBStage, src, kBStage, b_full + s);
              } else {  // this CTA's half of the stage, into both CTAs' smem
                constexpr uint32_t kHalf = kBStage / 2;
                bulk_g2s_mc(sB + s * kBStage + crank * kHalf, src + crank * kHalf, kHalf, b_full + s, 0x3);
              }
            }
          }
        }
      }
      if (DBG) {  // [48] weight warp: item waits, [49] free-stage waits, [50] total
        atomicAdd(&g_conv_dbg[48], static_cast<unsigned long long>(w_it));
        atomicAdd(&g_conv_dbg[49], static_cast<unsigned long long>(w_e));
        atomicAdd(&g_conv_dbg[50], static_cast<unsigned long long>(clock64() - t_start));
      }
    }
  } else if (warp == kTableWarp) {  // ------------------------ table filler
    for (int n = 0;; ++n) {
      const int slot = n % kItemSlots;
      mbar_wait(item_full + slot, (n / kItemSlots) & 1);
      const Item it = items[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(item_empty + slot);
      if (it.kind < 0) break;
      const int buf = n & 1;
      mbar_wait(tab_empty + buf, ((n >> 1) & 1) ^ 1);
      rb_fill_table<TM>(P, it, tables + buf * TM, extras + buf, lane);
      mbar_arrive(tab_full + buf);  // release: the entries are visible to the waiters
    }
  } else {  // ------------------------------------------------------ epilogue
    EpiLane L;
    L.quarter = warp & 3;
    L.half = (warp - 2) >> 2;
    L.e = lane & 7;
    L.plane = L.quarter * 4 + (lane >> 3);
    L.chunk_off = static_cast<int64_t>(L.plane >> 3) * P.ps * 128;
    L.sub = (L.plane & 7) ^ L.e;
    L.plane_off32 = L.plane * kPx * 8;
    const uint32_t lane_addr = (static_cast<uint32_t>(L.quarter * 32) << 16) + L.half * (TM / kEpiParts);
    for (int n = 0;; ++n) {
      const int slot = n % kItemSlots;
      mbar_wait(item_full + slot, (n / kItemSlots) & 1);
      const Item it = items[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(item_empty + slot);
      if (it.kind < 0) break;
      const int abuf = n & 1;
      const PosEntry* tab = tables + abuf * TM;
      const TileExtra* ex = extras + abuf;
      mbar_wait(tab_full + abuf, (n >> 1) & 1);
      mbar_wait(acc_full + abuf, (n >> 1) & 1);
      tc_fence_after();
      const long long t_epi = DBG ? clock64() : 0;
      const uint32_t taddr = tmem_base + abuf * TM + lane_addr;
      if (P.diag & 4) {
      } else if (it.kind == 0) {
        step_epilogue<0, TM>(P, tab, ex, L, taddr, it);
      } else if (it.kind == 1) {
        step_epilogue<1, TM>(P, tab, ex, L, taddr, it);
      } else {
        step_epilogue<2, TM>(P, tab, ex, L, taddr, it);
        if (P.cache & 4) {
          // the interior mid rows [q0 + 16, q0 + 240) of this tile are read
          // by this tile's conv3x3 #2 only (its neighbours' windows stop 16
          // rows short), and its window is in shared memory by now: drop the
          // dirty lines from L2 instead of writing them back; conv3x3 #1
          // rewrites them (pads included) before any later read
          // The same holds for the block input's hi / lo images (x of a unary
          // group, z of a binary one) at these rows: conv3x3 #1 tiles i−1..i+1
          // (done before this tile's W2 phase) and this tile's residual
          // phases were their only readers; every forward rewrites them
          // (images with their pads, and the segment gaps in stage_x).
          const int et = threadIdx.x - 64;  // 0 .. 255 over the epilogue warps
          constexpr int kIn = TM - 2 * kHalo;
          const int nbuf = (P.cache & 8) ? 3 : 1;
          for (int i = et; i < nbuf * 2 * kIn; i += kEpiWarps * 32) {
            const int b = i / (2 * kIn), c = (i / kIn) & 1, r = kHalo + i % kIn;
            uint8_t* base = b == 0 ? P.stage_mid : (b == 1 ? P.stage_x : P.stage_lo);
            discard_l2_line(base + ((static_cast<int64_t>(c) * P.ps + kGuard + it.q0 + r) << 7));
          }
        }
      }
      // the publishing thread keeps the tile's parents before the table
      // buffer is handed back
      int32_t parents[4] = {-1, -1, -1, -1};
      if (threadIdx.x == 64 && it.kind == 2) {
#pragma unroll
        for (int j = 0; j < 4; ++j) parents[j] = ex->parent[j];
      }
      tc_fence_before();
      mbar_arrive(acc_empty + abuf);
      __syncwarp();
      if (lane == 0) mbar_arrive(tab_empty + abuf);
      // publish: the tile's outputs are complete (conv1x1 / conv3x3 #1: a
      // per-tile flag; conv3x3 #2: the step's completed-tile count)
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
      if (threadIdx.x == 64) {
        __threadfence();
        if (it.kind < 2) {
          st_release_gpu((it.kind == 0 ? P.done0 : P.done1) + it.tile, P.epoch);
        } else {
          red_release_gpu_add(P.step_done + it.step, 1);
          // this tile's part of each parent's operand image is written
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (parents[j] >= 0) red_release_gpu_add(P.ready + parents[j], 1);
        }
        if (DBG) {
          atomicAdd(&g_conv_dbg[36 + 2 * it.kind], static_cast<unsigned long long>(clock64() - t_epi));
          atomicAdd(&g_conv_dbg[37 + 2 * it.kind], 1ull);
        }
      }
    }
  }
  __syncthreads();
  if (kCluster > 1) cluster_sync();  // no remote arrive or multicast still targets this CTA
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

constexpr int kStepSmem = kASlots * kASlot + kBStages * kBStage + kTableBytes +
                          kItemSlots * static_cast<int>(sizeof(Item)) + 512;  // + barriers, mailbox, TMEM slot

// ----------------------------------------------------------------- plan
// Segment layout and tile lists for every step, from the group tables, in
// one block: a warp per step scans its groups 32 at a time (segment starts,
// first tile, first bin tile), one warp scans the steps (position origins,
// tile prefixes), then every group's lane writes its tiles' (group, q0).
// seg_start[g] ends up absolute; tiles of step s occupy
// [step_tile_begin[s], step_tile_begin[s+1]).
__device__ __forceinline__ int32_t warp_incl_scan(int32_t x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

__global__ void __launch_bounds__(1024) k_rb_plan(
    int32_t n_steps, const int32_t* __restrict__ sgb, const int32_t* __restrict__ group_fid,
    const int32_t* __restrict__ group_begin, const int32_t* __restrict__ arity_of, int32_t* __restrict__ seg_start,
    int32_t* __restrict__ group_tile0, int32_t* __restrict__ group_bintile0, int32_t* __restrict__ step_tile_begin,
    int32_t* __restrict__ step_bintile_begin, int32_t* __restrict__ step_positions, int32_t* __restrict__ tile_group,
    int32_t* __restrict__ tile_q0, int32_t* __restrict__ bin_group, int32_t* __restrict__ bin_q0, int32_t tile_m) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  // 1. per step: relative segment starts and tile offsets
  for (int32_t s = warp; s < n_steps; s += nwarps) {
    int32_t pos = 0, tiles = 0, bins = 0;
    for (int32_t g0 = sgb[s]; g0 < sgb[s + 1]; g0 += 32) {
      const int32_t g = g0 + lane;
      int32_t nt = 0, bin = 0;
      bool live = false;
      if (g < sgb[s + 1]) {
        const int32_t rows = group_begin[g + 1] - group_begin[g];
        const int32_t a = arity_of[group_fid[g]];
        live = a > 0 && rows > 0;
        if (live) {
          nt = seg_tiles(rows, tile_m);
          bin = a == 2 ? nt : 0;
        } else {
          seg_start[g] = -1;
        }
      }
      const int32_t it = warp_incl_scan(nt, lane), ib = warp_incl_scan(bin, lane);
      if (live) {
        seg_start[g] = pos + (it - nt) * tile_m + kLead;  // the first image; its tiles start kLead rows earlier
        group_tile0[g] = tiles + it - nt;
        group_bintile0[g] = bin ? bins + ib - bin : -1;
      }
      pos += __shfl_sync(0xffffffffu, it, 31) * tile_m;
      tiles += __shfl_sync(0xffffffffu, it, 31);
      bins += __shfl_sync(0xffffffffu, ib, 31);
    }
    if (lane == 0) {
      step_positions[s] = pos;
      step_tile_begin[s + 1] = tiles;
      step_bintile_begin[s + 1] = bins;
    }
  }
  __syncthreads();
  // 2. prefixes over steps (every step owns its own staging range, so a
  // result can be written straight into its parent's later operand image)
  if (warp == 0) {
    int32_t cp = 0, ct = 0, cb = 0;
    if (lane == 0) {
      step_tile_begin[0] = 0;
      step_bintile_begin[0] = 0;
    }
    for (int32_t s0 = 0; s0 < n_steps; s0 += 32) {
      const int32_t s = s0 + lane;
      const int32_t p = s < n_steps ? step_positions[s] : 0;
      const int32_t t = s < n_steps ? step_tile_begin[s + 1] : 0;
      const int32_t b = s < n_steps ? step_bintile_begin[s + 1] : 0;
      const int32_t ip = warp_incl_scan(p, lane), itt = warp_incl_scan(t, lane), ib = warp_incl_scan(b, lane);
      __syncwarp();
      if (s < n_steps) {
        step_positions[s] = cp + ip - p;  // the step's position origin
        step_tile_begin[s + 1] = ct + itt;
        step_bintile_begin[s + 1] = cb + ib;
      }
      cp += __shfl_sync(0xffffffffu, ip, 31);
      ct += __shfl_sync(0xffffffffu, itt, 31);
      cb += __shfl_sync(0xffffffffu, ib, 31);
    }
    if (lane == 0) step_positions[n_steps] = cp;
  }
  __syncthreads();
  // 3. absolute segment starts and the tile lists (a warp per step, groups
  // in turn, the group's tiles across the lanes)
  for (int32_t s = warp; s < n_steps; s += nwarps) {
    const int32_t base = step_positions[s], t_base = step_tile_begin[s], b_base = step_bintile_begin[s];
    for (int32_t g = sgb[s]; g < sgb[s + 1]; ++g) {
      const int32_t rel = seg_start[g];
      __syncwarp();
      if (rel < 0) continue;
      const int32_t start = rel + base;
      if (lane == 0) seg_start[g] = start;
      const int32_t nt = seg_tiles(group_begin[g + 1] - group_begin[g], tile_m);
      const int32_t t0 = t_base + group_tile0[g], b0 = group_bintile0[g];
      for (int32_t i = lane; i < nt; i += 32) {
        tile_group[t0 + i] = g;
        tile_q0[t0 + i] = start - kLead + i * tile_m;
        if (b0 >= 0) {
          bin_group[b_base + b0 + i] = g;
          bin_q0[b_base + b0 + i] = start - kLead + i * tile_m;
        }
      }
    }
  }
}

// Forwarding table for conv3x3 #2 epilogues: for every expensive member,
// each child with a unique parent (fwd_ok) receives the absolute staging
// position of that parent's image and which buffer / planes it fills.
__global__ void k_rb_fwd_init(int64_t n, int32_t* __restrict__ fwd_pos, int32_t* __restrict__ fwd_slot,
                              int32_t* __restrict__ fwd_parent, int32_t* __restrict__ need) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) {
    fwd_pos[i] = -1;
    fwd_slot[i] = 1 << 8;  // keep the fp32 value (roots, shared children)
    fwd_parent[i] = -1;
    need[i] = 0;
  }
}

// Last index i in [lo, hi] with v[i] <= x (v ascending, v[lo] <= x).
__device__ __forceinline__ int32_t last_le(const int32_t* __restrict__ v, int32_t lo, int32_t hi, int32_t x) {
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (v[mid] <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Forwarding targets: one thread per member of every step; each child with
// a unique parent (fwd_ok) gets the parent's image position and buffer.
__global__ void k_rb_fwd(int32_t n_steps, const int32_t* __restrict__ sgb, const int32_t* __restrict__ group_fid,
                         const int32_t* __restrict__ group_begin, const int32_t* __restrict__ arity_of,
                         const int32_t* __restrict__ seg_start, const int32_t* __restrict__ member_g,
                         const int32_t* __restrict__ child0, const int32_t* __restrict__ child1,
                         const int32_t* __restrict__ fwd_ok, int32_t* __restrict__ fwd_pos,
                         int32_t* __restrict__ fwd_slot, int32_t* __restrict__ fwd_parent, int32_t keep_all) {
  // a block per group (no per-member search), threads over its members
  for (int32_t g = sgb[0] + blockIdx.x; g < sgb[n_steps]; g += gridDim.x) {
    if (seg_start[g] < 0) continue;
    const int32_t arity = arity_of[group_fid[g]];
    for (int32_t m = group_begin[g] + threadIdx.x; m < group_begin[g + 1]; m += blockDim.x) {
      const int32_t node = member_g[m];
      for (int k = 0; k < arity; ++k) {
        const int32_t c = k == 0 ? child0[node] : child1[node];
        if (!fwd_ok[c]) continue;
        fwd_pos[c] = seg_start[g] + (m - group_begin[g]) * kImg;
        // buffer (bit 0: stage_x / stage_cat) and first plane; no fp32 copy:
        // a unary parent reads its residual from the hi/lo images
        fwd_slot[c] = (arity == 2 ? 1 : 0) | ((16 * k) << 1) | (keep_all << 8);
        fwd_parent[c] = node;
      }
    }
  }
}

__global__ void k_rb_memtab(int32_t n_steps, const int32_t* __restrict__ sgb,
                            const int32_t* __restrict__ group_fid, const int32_t* __restrict__ group_begin,
                            const int32_t* __restrict__ seg_start, const int32_t* __restrict__ member_g,
                            const int32_t* __restrict__ fwd_pos, const int32_t* __restrict__ fwd_slot,
                            const int32_t* __restrict__ arity_of, const int32_t* __restrict__ fid,
                            const int32_t* __restrict__ child0, const int32_t* __restrict__ child1,
                            const int32_t* __restrict__ example, const int32_t* __restrict__ fwd_ok,
                            const float* inputs, float* values, MemberEntry* __restrict__ memtab,
                            GatherTask* __restrict__ tasks, int32_t* __restrict__ n_tasks, int64_t task_cap,
                            const int32_t* __restrict__ fwd_parent, int32_t* __restrict__ need, int32_t tile_m) {
  // a block per group (no per-member search), threads over its members
  for (int32_t g = sgb[0] + blockIdx.x; g < sgb[n_steps]; g += gridDim.x) {
    if (seg_start[g] < 0) continue;
    const int32_t arity = arity_of[group_fid[g]];
    const int32_t g_step = last_le(sgb, 0, n_steps - 1, g);
    for (int32_t m = group_begin[g] + threadIdx.x; m < group_begin[g + 1]; m += blockDim.x) {
      const int32_t node = member_g[m];
      const int32_t sw = fwd_slot[node];
      const int32_t tgt = fwd_pos[node];
      MemberEntry e{};
      e.slot = values + static_cast<int64_t>(node) * kFmap;
      e.keep32 = (sw >> 8) & 1;
      e.fwd_row = tgt >= 0 ? kGuard + tgt : -1;
      e.fwd_buf = (sw & 1) ? 1 + (((sw >> 1) & 31) >> 4) : 0;
      e.parent = tgt >= 0 ? fwd_parent[node] : -1;
      memtab[m] = e;
      if (e.parent >= 0) {  // the conv3x3 #2 tiles covering this image, each counted once by the parent
        const int32_t j = m - group_begin[g];
        const int32_t t0 = (j * kImg + kLead) / tile_m, t1 = (j * kImg + kImg - 1 + kLead) / tile_m;
        atomicAdd(need + e.parent, t1 - t0 + 1);
      }
      // operands no child epilogue forwards: leaves (list 0) and children
      // shared by several parents (list 1), one gather task each
      for (int k = 0; k < arity; ++k) {
        const int32_t ch = k == 0 ? child0[node] : child1[node];
        if (fwd_ok[ch]) continue;
        const bool leaf = arity_of[fid[ch]] == 0;
        GatherTask t{};
        t.src = leaf ? inputs + static_cast<int64_t>(example[ch]) * kFmap : values + static_cast<int64_t>(ch) * kFmap;
        t.row = kGuard + seg_start[g] + static_cast<int64_t>(m - group_begin[g]) * kImg;
        t.buf = arity == 2 ? 1 + k : 0;
        t.step = g_step;
        const int list = leaf ? 0 : 1;
        const int32_t i = atomicAdd(n_tasks + list, 1);
        if (i < task_cap) tasks[list * task_cap + i] = t;
      }
    }
  }
}

// ---------------------------------------------------------------- order
// Claim order of every step's work units (StepParams::order). Three
// streams over the step's conv3x3 units l = 0 … n1−1 (segment order): the
// conv1x1 unit of conv unit c (binary groups) at key 3(c − D0), conv3x3 #1
// unit l at 3l + 1, conv3x3 #2 unit l at 3(l + D) + 2; each unit's claim
// index is its key's rank. So a conv1x1 tile runs D0 units before the
// conv3x3 #1 tile that reads its z, and z is consumed (by #1, then by #2 D
// units later) while it is still in L2. Dependencies always rank earlier:
// #1 unit l reads conv1x1 units l−1…l+1 (keys ≤ 3(l+1−D0) < 3l+1 for D0 ≥ 1),
// #2 unit l reads #1 units l−1…l+1 and conv1x1 unit l (D ≥ 1). D0 ≥ n1
// reproduces "all conv1x1 tiles first".
__global__ void __launch_bounds__(1024) k_rb_order(int32_t n_steps, const int32_t* __restrict__ step_tile_begin,
                                                   const int32_t* __restrict__ step_bintile_begin,
                                                   const int32_t* __restrict__ tile_group,
                                                   const int32_t* __restrict__ group_tile0,
                                                   const int32_t* __restrict__ group_bintile0, int32_t lookahead,
                                                   int32_t bin_lead, int32_t* __restrict__ prefix,
                                                   int32_t* __restrict__ order) {
  __shared__ int32_t wsum[32];
  __shared__ int32_t carry_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int32_t st = blockIdx.x; st < n_steps; st += gridDim.x) {
    const int32_t t0 = step_tile_begin[st], b0 = step_bintile_begin[st];
    const int32_t n1 = (step_tile_begin[st + 1] - t0) / kCluster;
    const int32_t n0 = (step_bintile_begin[st + 1] - b0) / kCluster;
    if (n0 + n1 == 0) continue;
    const int32_t D = min(max(lookahead / kCluster, 2), max(n1, 1));
    const int32_t D0 = min(max(bin_lead / kCluster, 1), max(n1, 1));
    int32_t* pre = prefix + t0 / kCluster;  // inclusive count of binary conv units ≤ c
    int32_t* out = order + (b0 + 2 * t0) / kCluster;
    // 1. prefix of the binary flags over the conv units
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int32_t base = 0; base < n1; base += blockDim.x) {
      const int32_t c = base + static_cast<int32_t>(threadIdx.x);
      const int32_t f = c < n1 ? (group_bintile0[tile_group[t0 + c * kCluster]] >= 0 ? 1 : 0) : 0;
      int32_t x = f;
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[warp] = x;
      __syncthreads();
      if (warp == 0) {
        int32_t w = lane < static_cast<int>(blockDim.x >> 5) ? wsum[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
          if (lane >= o) w += y;
        }
        wsum[lane] = w;
      }
      __syncthreads();
      if (c < n1) pre[c] = carry_s + (warp > 0 ? wsum[warp - 1] : 0) + x;
      __syncthreads();
      if (threadIdx.x == blockDim.x - 1) carry_s += wsum[(blockDim.x >> 5) - 1];
      __syncthreads();
    }
    // 2. every unit at its key's rank
    auto bins_upto = [&](int32_t c) { return c < 0 ? 0 : pre[min(c, n1 - 1)]; };
    for (int32_t l = threadIdx.x; l < n1; l += blockDim.x) {
      const int32_t r1 = l + max(0, min(n1, l - D)) + bins_upto(l + D0);
      out[r1] = (1 << 28) | l;
      const int32_t r2 = min(n1, l + D + 1) + l + bins_upto(l + D + D0);
      out[r2] = (2 << 28) | l;
      const int32_t g = tile_group[t0 + l * kCluster];
      if (group_bintile0[g] >= 0) {
        const int32_t bl = (group_bintile0[g] + l * kCluster - group_tile0[g]) / kCluster;
        const int32_t rb = max(0, min(n1, l - D0)) + max(0, min(n1, l - D0 - D)) + (pre[l] - 1);
        out[rb] = (0 << 28) | bl;
      }
    }
    __syncthreads();
  }
}

// --------------------------------------------------------------- gather
// Packs the operand maps that were NOT forwarded by a child's conv3x3 #2
// epilogue — leaves (the example's input map) and children shared by
// several parents — into the member's fp16 staging image: unary → stage_x
// (16 planes, plus the lo image in stage_lo: the block's residual), binary →
// stage_cat planes 16k.. (the channel concat of [x; y] is fused into the
// write). Only the 196 data positions are written;
// pads and alignment gaps were zeroed once at session creation.
// Gathered operands → staged images. One thread per (task, 64-channel
// chunk, pixel, plane of the chunk): 8 consecutive lanes read the 8 planes'
// 32-byte pixel records and write the 8 swizzled 16-byte slots of one
// 128-byte staging row, so a warp store covers 4 whole rows (and the lo
// rows for unary members: the block's residual). list 0 = leaf tasks of
// every step (inputs only); list 1 = shared-child tasks, restricted to `step`.
__global__ void __launch_bounds__(256) k_rb_gather(const GatherTask* __restrict__ tasks,
                                                   const int32_t* __restrict__ n_tasks, int32_t list,
                                                   int32_t step, int64_t task_cap,
                                                   uint8_t* __restrict__ stage_x, uint8_t* __restrict__ stage_lo,
                                                   uint8_t* __restrict__ stage_cat, int64_t ps,
                                                   int32_t* __restrict__ err) {
  constexpr int kPer = 2 * kImg * 8;  // chunks × image positions (pads written as zeros) × planes
  const int64_t nt = min(static_cast<int64_t>(n_tasks[list]), task_cap);
  const GatherTask* T = tasks + list * task_cap;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < nt * kPer;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const GatherTask t = T[idx / kPer];
    if (list == 1 && t.step != step) continue;
    const int rem = static_cast<int>(idx % kPer);
    const int j = rem & 7, q = rem >> 3;
    const int cc = q >= kImg ? 1 : 0, pos = q - cc * kImg;
    const int r = pos / 15, c = pos - r * 15;
    const int64_t row = t.row + pos;
    const int64_t off = ((static_cast<int64_t>((t.buf == 2 ? 2 : 0) + cc) * ps + row) << 7) +
                        ((j ^ static_cast<int>(row & 7)) << 4);
    uint4 h = make_uint4(0, 0, 0, 0), l = make_uint4(0, 0, 0, 0);
    if (r < 14 && c < 14) {
      const float* sp = t.src + ((8 * cc + j) * kPx + r * 14 + c) * 8;
      const float4 a = __ldg(reinterpret_cast<const float4*>(sp));
      const float4 b = __ldg(reinterpret_cast<const float4*>(sp + 4));
      const float o[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      // inputs must be finite (src/executor.cpp:107) and within fp16 range
      const int32_t bad = range_code(o);
      if (bad) atomicCAS(err, 0, bad);
      split_f16x8(o, h, l);
    }
    *reinterpret_cast<uint4*>((t.buf == 0 ? stage_x : stage_cat) + off) = h;
    if (t.buf == 0) *reinterpret_cast<uint4*>(stage_lo + off) = l;
  }
}

// A segment's lead rows (the first image's top / left pads) and the rows
// after its last image up to its tile end, zeroed in stage_x every forward:
// no image writer touches them, and a new layout must not see old data.
// With the lead, a valid output's taps never leave its own segment, so no
// cross-segment ordering is needed inside a step.
__global__ void k_rb_zero_gaps(int32_t n_steps, const int32_t* __restrict__ sgb, const int32_t* __restrict__ group_begin,
                               const int32_t* __restrict__ seg_start, uint8_t* __restrict__ stage_x, int64_t ps,
                               int32_t tile_m) {
  const int32_t g0 = sgb[0], g1 = sgb[n_steps];
  for (int32_t g = g0 + blockIdx.x; g < g1; g += gridDim.x) {
    if (seg_start[g] < 0) continue;
    const int32_t rows = group_begin[g + 1] - group_begin[g];
    const int32_t used = rows * kImg, span = seg_tiles(rows, tile_m) * tile_m;
    const int64_t base = kGuard + static_cast<int64_t>(seg_start[g]) - kLead;  // the segment's first tile row
    const int32_t tail = span - kLead - used;                                // gap rows after the last image
    const int32_t n16 = (kLead + tail) * 8;                                  // 16-byte pieces per chunk
    for (int32_t i = threadIdx.x; i < 2 * n16; i += blockDim.x) {
      const int cc = i >= n16 ? 1 : 0, k = i - cc * n16;
      const int32_t r = k >> 3;
      const int64_t row = r < kLead ? base + r : base + kLead + used + (r - kLead);
      *reinterpret_cast<uint4*>(stage_x + ((static_cast<int64_t>(cc) * ps + row) << 7) + ((k & 7) << 4)) =
          make_uint4(0, 0, 0, 0);
    }
  }
}

// Layout conversions between reference rows (CHW: element c·196 + px) and
// plane maps ([16][196][8]); one block per (row, plane) transposes a
// 196 × 8 tile through shared memory so both sides stay coalesced.
__global__ void __launch_bounds__(256) k_chw_to_planes(const float* __restrict__ chw,
                                                       float* __restrict__ planes) {
  __shared__ float t[8][kPx + 1];
  const int64_t row = blockIdx.x / kPlanes;
  const int p = blockIdx.x % kPlanes;
  const float* src = chw + row * kFmap + p * 8 * kPx;
  for (int i = threadIdx.x; i < 8 * kPx; i += blockDim.x) t[i / kPx][i % kPx] = src[i];
  __syncthreads();
  float* dst = planes + row * kFmap + p * kPx * 8;
  for (int i = threadIdx.x; i < 8 * kPx; i += blockDim.x) dst[i] = t[i & 7][i >> 3];
}

__global__ void __launch_bounds__(256) k_roots_to_chw(const int32_t* __restrict__ root_g,
                                                      const int32_t* __restrict__ fid,
                                                      const int32_t* __restrict__ arity_of,
                                                      const int32_t* __restrict__ example,
                                                      const float* __restrict__ inputs,
                                                      const float* __restrict__ values,
                                                      float* __restrict__ chw) {
  __shared__ float t[8][kPx + 1];
  const int64_t e = blockIdx.x / kPlanes;
  const int p = blockIdx.x % kPlanes;
  const int32_t r = root_g[e];
  const float* map = arity_of[fid[r]] == 0 ? inputs + static_cast<int64_t>(example[r]) * kFmap
                                          : values + static_cast<int64_t>(r) * kFmap;
  const float* src = map + p * kPx * 8;
  for (int i = threadIdx.x; i < 8 * kPx; i += blockDim.x) t[i & 7][i >> 3] = src[i];
  __syncthreads();
  float* dst = chw + e * kFmap + p * 8 * kPx;
  for (int i = threadIdx.x; i < 8 * kPx; i += blockDim.x) dst[i] = t[i / kPx][i % kPx];
}

int32_t g_debug_flag = 0;

}  // namespace

extern "C" int dbk_rb_plan(int32_t n_steps, const int32_t* step_group_begin, const int32_t* group_fid,
                           const int32_t* group_begin, const int32_t* arity_of, int32_t* seg_start,
                           int32_t* group_tile0, int32_t* group_bintile0, int32_t* step_tile_begin,
                           int32_t* step_bintile_begin, int32_t* step_positions, int32_t* tile_group,
                           int32_t* tile_q0, int32_t* bin_group, int32_t* bin_q0, int64_t n_nodes,
                           const int32_t* member_g, const int32_t* child0, const int32_t* child1,
                           const int32_t* fwd_ok, int32_t* fwd_pos, int32_t* fwd_slot, int32_t* fwd_parent,
                           int32_t* need, int32_t tile_m, int32_t training, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n_steps <= 0) return 0;
  k_rb_plan<<<1, 1024, 0, s>>>(n_steps, step_group_begin, group_fid, group_begin, arity_of, seg_start,
                               group_tile0, group_bintile0, step_tile_begin, step_bintile_begin,
                               step_positions, tile_group, tile_q0, bin_group, bin_q0, tile_m);
  k_rb_fwd_init<<<static_cast<unsigned>((n_nodes + 255) / 256), 256, 0, s>>>(n_nodes, fwd_pos, fwd_slot,
                                                                              fwd_parent, need);
  k_rb_fwd<<<148 * 4, 256, 0, s>>>(n_steps, step_group_begin, group_fid, group_begin, arity_of, seg_start,
                                   member_g, child0, child1, fwd_ok, fwd_pos, fwd_slot, fwd_parent, training ? 1 : 0);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_rb_gather(const void* tasks, const int32_t* n_tasks, int32_t list, int32_t step,
                             int64_t task_cap, void* stage_x, void* stage_lo, void* stage_cat, int64_t plane_stride,
                             int32_t* err, int32_t blocks, void* stream) {
  k_rb_gather<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const GatherTask*>(tasks), n_tasks, list, step, task_cap, static_cast<uint8_t*>(stage_x),
      static_cast<uint8_t*>(stage_lo), static_cast<uint8_t*>(stage_cat), plane_stride, err);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_rb_zero_gaps(int32_t n_steps, const int32_t* step_group_begin, const int32_t* group_begin,
                                const int32_t* seg_start, void* stage_x, int64_t plane_stride, int32_t tile_m,
                                void* stream) {
  if (n_steps <= 0) return 0;
  k_rb_zero_gaps<<<148 * 2, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      n_steps, step_group_begin, group_begin, seg_start, static_cast<uint8_t*>(stage_x), plane_stride, tile_m);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_rb_order(int32_t n_steps, const int32_t* step_tile_begin, const int32_t* step_bintile_begin,
                            const int32_t* tile_group, const int32_t* group_tile0, const int32_t* group_bintile0,
                            int32_t num_sms, int32_t* prefix, int32_t* order, void* stream) {
  if (n_steps <= 0) return 0;
  const char* la = std::getenv("DYNBATCH_LOOKAHEAD");
  const int32_t lookahead = (la ? std::atoi(la) : 1) * num_sms;  // as dbk_rb_step
  const char* bl = std::getenv("DYNBATCH_BIN_LEAD");              // conv1x1 lead in SM-rows of tiles
  const int32_t bin_lead = bl ? std::atoi(bl) * num_sms : num_sms;
  k_rb_order<<<static_cast<unsigned>(std::min(n_steps, 148 * 4)), 1024, 0, static_cast<cudaStream_t>(stream)>>>(
      n_steps, step_tile_begin, step_bintile_begin, tile_group, group_tile0, group_bintile0, lookahead,
      bin_lead > 0 ? bin_lead : (1 << 29), prefix, order);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_rb_memtab(int32_t n_steps, const int32_t* step_group_begin, const int32_t* group_fid,
                             const int32_t* group_begin, const int32_t* seg_start, const int32_t* member_g,
                             const int32_t* fwd_pos, const int32_t* fwd_slot, const int32_t* arity_of,
                             const int32_t* fid, const int32_t* child0, const int32_t* child1,
                             const int32_t* example, const int32_t* fwd_ok, const float* inputs, float* values,
                             void* memtab, void* tasks, int32_t* n_tasks, int64_t task_cap,
                             const int32_t* fwd_parent, int32_t* need, int32_t tile_m, void* stream) {
  if (n_steps <= 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaMemsetAsync(n_tasks, 0, 2 * sizeof(int32_t), s);
  k_rb_memtab<<<148 * 4, 256, 0, s>>>(n_steps, step_group_begin, group_fid, group_begin, seg_start, member_g,
                                      fwd_pos, fwd_slot, arity_of, fid, child0, child1, example, fwd_ok, inputs,
                                      values, static_cast<MemberEntry*>(memtab), static_cast<GatherTask*>(tasks),
                                      n_tasks, task_cap, fwd_parent, need, tile_m);
  return static_cast<int>(cudaGetLastError());
}

// Kernel attributes (shared-memory carve-out), set once per process, and
// before any stream capture of a forward.
extern "C" int dbk_rb_configure(void) {
  // per device (the attribute is), once, from any thread
  static std::atomic<uint64_t> configured{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    cudaFuncSetAttribute(k_rb_step<256, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStepSmem);
    cudaFuncSetAttribute(k_rb_step<256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStepSmem);
    cudaFuncSetAttribute(k_rb_step<128, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStepSmem);
    cudaFuncSetAttribute(k_rb_step<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStepSmem);
    cudaFuncSetAttribute(k_rb_step<64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStepSmem);
    cudaFuncSetAttribute(k_rb_step<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStepSmem);
    configured.fetch_or(bit, std::memory_order_release);
  }
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_rb_step(int32_t step, int32_t step_end, int32_t epoch, const int32_t* step_tile_begin,
                           const int32_t* tile_group,
                           const int32_t* tile_q0, const int32_t* step_bintile_begin, const int32_t* bin_group,
                           const int32_t* bin_q0, const int32_t* group_fid, const int32_t* group_begin,
                           const int32_t* seg_start, const int32_t* group_tile0, const int32_t* group_bintile0,
                           const void* memtab, void* stage_x, void* stage_lo, void* stage_cat, void* stage_mid,
                           int64_t plane_stride, const void* const* w0, const void* const* w1,
                           const void* const* w2, const float* const* b0, const float* const* b1,
                           const float* const* b2, const void* ident, int32_t* done0, int32_t* done1,
                           int32_t* step_done, int32_t* queue, int32_t* err, int32_t* ready, const int32_t* need,
                           const int32_t* member_g, const int32_t* order, const float* values,
                           int64_t values_floats, int32_t tile_m, int32_t num_sms, int32_t training, void* stream) {
  if (tile_m != 256 && tile_m != 128 && tile_m != 64) return static_cast<int>(cudaErrorInvalidValue);
  dbk_rb_configure();
  StepParams p{};
  p.step = step;
  p.step_end = step_end;
  p.epoch = epoch;
  const char* la = std::getenv("DYNBATCH_LOOKAHEAD");
  // one SM-row of tiles ahead: a conv3x3 #2 tile reads mid written ~2·SMs
  // tiles earlier, still in L2 (profiles/cache_sweep.py: −40% DRAM traffic)
  p.lookahead = (la ? std::atoi(la) : 1) * num_sms;
  p.debug = g_debug_flag;
  const char* dg = std::getenv("DYNBATCH_DIAG");
  p.diag = dg ? std::atoi(dg) : 0;
  const char* ch = std::getenv("DYNBATCH_CACHE");
  p.cache = ch ? std::atoi(ch) : 4;  // default: drop consumed interior mid lines from L2
  if (training) p.cache &= ~12;  // the backward reads mid and the block inputs
  p.step_tile_begin = step_tile_begin;
  p.tile_group = tile_group;
  p.tile_q0 = tile_q0;
  p.step_bintile_begin = step_bintile_begin;
  p.bin_group = bin_group;
  p.bin_q0 = bin_q0;
  p.group_fid = group_fid;
  p.group_begin = group_begin;
  p.seg_start = seg_start;
  p.group_tile0 = group_tile0;
  p.group_bintile0 = group_bintile0;
  p.memtab = static_cast<const MemberEntry*>(memtab);
  p.stage_x = static_cast<uint8_t*>(stage_x);
  p.stage_lo = static_cast<uint8_t*>(stage_lo);
  p.stage_cat = static_cast<uint8_t*>(stage_cat);
  p.stage_mid = static_cast<uint8_t*>(stage_mid);
  p.ps = plane_stride;
  p.wpack[0] = reinterpret_cast<const uint8_t* const*>(w0);
  p.wpack[1] = reinterpret_cast<const uint8_t* const*>(w1);
  p.wpack[2] = reinterpret_cast<const uint8_t* const*>(w2);
  p.bias[0] = b0;
  p.bias[1] = b1;
  p.bias[2] = b2;
  p.ident = static_cast<const uint8_t*>(ident);
  p.done0 = done0;
  p.done1 = done1;
  p.step_done = step_done;
  p.queue = queue;
  p.err = err;
  p.ready = ready;
  p.need = need;
  p.member_g = member_g;
  p.order = order;
  p.values = values;
  p.values_floats = values_floats;
  const char* sb = std::getenv("DYNBATCH_STEP_BARRIER");
  p.step_barrier = sb ? std::atoi(sb) : 0;  // default: per-image dependencies only
  // persistent: one CTA per SM, in clusters of kCluster
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(num_sms / kCluster * kCluster));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kStepSmem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (tile_m == 256)
    e = p.debug ? cudaLaunchKernelEx(&cfg, k_rb_step<256, true>, p) : cudaLaunchKernelEx(&cfg, k_rb_step<256, false>, p);
  else if (tile_m == 128)
    e = p.debug ? cudaLaunchKernelEx(&cfg, k_rb_step<128, true>, p) : cudaLaunchKernelEx(&cfg, k_rb_step<128, false>, p);
  else
    e = p.debug ? cudaLaunchKernelEx(&cfg, k_rb_step<64, true>, p) : cudaLaunchKernelEx(&cfg, k_rb_step<64, false>, p);
  return static_cast<int>(e != cudaSuccess ? e : cudaGetLastError());
}

extern "C" int dbk_rb_inputs_from_chw(int64_t rows, const float* chw, float* planes, void* stream) {
  const int64_t total = rows * kFmap;
  if (total <= 0) return 0;
  k_chw_to_planes<<<static_cast<unsigned>(rows * kPlanes), 256, 0, static_cast<cudaStream_t>(stream)>>>(chw,
                                                                                                     planes);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_rb_outputs_to_chw(int64_t b, const int32_t* root_g, const int32_t* fid,
                                     const int32_t* arity_of, const int32_t* example, const float* inputs,
                                     const float* values, float* chw, void* stream) {
  const int64_t total = b * kFmap;
  if (total <= 0) return 0;
  k_roots_to_chw<<<static_cast<unsigned>(b * kPlanes), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      root_g, fid, arity_of, example, inputs, values, chw);
  return static_cast<int>(cudaGetLastError());
}

// Copies (and optionally zeroes) the MMA-thread wait counters; enable != 0
// turns accounting on for subsequent launches.
extern "C" int dbk_rb_debug_enabled() { return g_debug_flag; }

extern "C" int dbk_rb_debug(unsigned long long* out, int32_t reset, int32_t enable) {
  g_debug_flag = enable;
  if (out) cudaMemcpyFromSymbol(out, g_conv_dbg, sizeof(unsigned long long) * 64);
  if (reset) {
    unsigned long long z[64] = {};
    cudaMemcpyToSymbol(g_conv_dbg, z, sizeof(z));
  }
  return static_cast<int>(cudaGetLastError());
}
