// iep_train.hpp — device state of the IEP training step (iep_train.cpp).
#pragma once

#include <cublas_v2.h>

#include <cstdint>
#include <vector>

#include "device.hpp"

namespace dynbatch::dev {

struct IepSession::Train {
  cublasHandle_t blas = nullptr;
  std::vector<int> arity;  // per function id
  // fp32 input-major module weights (w0 [2C][C], w1 / w2 [9C][C]) and the
  // gradients of every weight and bias, per function
  std::vector<Buf<float>> w0, w1, w2, gw0, gb0, gw1, gb1, gw2, gb2;
  // head gradients (wp [C][P], bp, w1 [49P][F], b1, w2 [F][A], b2)
  Buf<float> gwp, gbp, ghw1, ghb1, ghw2, ghb2;
  Buf<float> d_inputs;  // [b][C·196] CHW
  Buf<float> dy_nodes;  // [N][257][C]: gradient of every node's output, PI layout
  Buf<float> loss;
  Buf<std::int32_t> labels;
  // per-group scratch (PI rows; mid / xin carry 16 guard rows at each end)
  Buf<float> da2, mid, xin, cols, g, da1, dx, da0, cat, dcat;
  // head scratch
  Buf<float> dlogits, hid, dhid, pooled, dpooled, proj, dproj, roots, droots;
  std::int64_t cap_rows = 0, cap_b = 0, cap_n = 0;
  // step tables of the backward: expensive member nodes and staging rows,
  // bias slabs (row ranges and gradient targets), grouped-GEMM pointers
  Buf<std::int32_t> nodes;
  Buf<std::int64_t> rows, slab_row;
  Buf<float*> slab_dst;
  Buf<const void*> ptr_dev;
  // implicit-GEMM data gradients (bwd_conv.cu): transposed tap weights per
  // function (conv3x3 #1 / #2) and their tables, the packed dA operand, and
  // every step's tiles (first row, group rows [lo, hi), function)
  std::vector<Buf<std::uint8_t>> wd1, wd2;
  Buf<const void*> wd1tab, wd2tab;
  Buf<std::uint8_t> dpack;         // packed fp32 dA (data gradients)
  Buf<std::uint8_t> apack, hpack;  // packed fp16 activations (mid / x) and scaled dA (weight gradients)
  Buf<std::uint32_t> absmax;       // |dA| max (float bits): the fp16 scale
  std::int64_t dpack_rows = 0;
  Buf<std::int32_t> dtiles;  // [4][n]: row0, lo, hi, fn
  Buf<std::int32_t> witems;  // [4][n]: K range k0, k1, kernel row dr, fn
  Buf<float*> gw1tab, gw2tab;
  // the forward's per-function weight blocks and biases (host copies of the
  // session's tables, fetched by the first sgd_update)
  std::vector<const void*> fw0, fw1, fw2;
  std::vector<const float*> fb0, fb1, fb2;
  bool stepped = false;  // a train_step ran: gradients exist
  ~Train() {
    if (blas) cublasDestroy(blas);
  }
};

}  // namespace dynbatch::dev
