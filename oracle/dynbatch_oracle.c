/* oracle/dynbatch_oracle.c — plain-C restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see dynbatch_oracle.h for who may call it).
 * Every function cites the reference file:line it restates; paths are
 * relative to /root/reference/proj/. The reference accumulates with
 * `acc += x * w`, which GCC contracts to a fused multiply-add under the
 * reference build flags (-O3 -march=native, gnu++20); this file is built as
 * ISO C (no implicit contraction) and calls fma() explicitly so the fp64 bits
 * match the compiled reference.
 */
#include "dynbatch_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ---------------------------------------------------------------- RNG ---- */
/* std::mt19937_64 (include/dynbatch/rng.hpp:29-50 wraps it); the engine
 * constants are the ones the C++ standard fixes for mt19937_64. */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  r->idx = MT_N;
}

static void mt_twist(orc_rng* r) {
  for (int i = 0; i < MT_N; ++i) {
    uint64_t y = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
    uint64_t v = r->mt[(i + MT_M) % MT_N] ^ (y >> 1);
    if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
    r->mt[i] = v;
  }
  r->idx = 0;
}

uint64_t orc_rng_u64(orc_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t z = r->mt[r->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

/* Rng::uniform (include/dynbatch/rng.hpp:36). */
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_u64(r) >> 11) * 0x1.0p-53; }

/* Rng::uniform(lo, hi) (rng.hpp:38). */
static double rng_range(orc_rng* r, double lo, double hi) { return lo + (hi - lo) * orc_rng_uniform(r); }

/* Rng::uniform_int (rng.hpp:41-44), inclusive bounds. */
static int64_t rng_int(orc_rng* r, int64_t lo, int64_t hi) {
  uint64_t span = (uint64_t)(hi - lo) + 1;
  return lo + (int64_t)(orc_rng_u64(r) % span);
}

/* Rng::bernoulli (rng.hpp:46). */
static int rng_bernoulli(orc_rng* r, double p) { return orc_rng_uniform(r) < p; }

/* splitmix64 / mix_seed (rng.hpp:11-24). */
static uint64_t splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t orc_mix_seed(uint64_t seed, uint64_t stream) {
  uint64_t s = seed ^ (0x9e3779b97f4a7c15ULL + (stream << 1));
  uint64_t a = splitmix64(&s);
  s ^= stream;
  return a ^ splitmix64(&s);
}

/* random_batch (src/workload.cpp:207-212): uniform in [-1, 1), row-major. */
void orc_random_batch(int64_t rows, int64_t width, uint64_t seed, double* out) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int64_t i = 0; i < rows * width; ++i) out[i] = rng_range(&r, -1.0, 1.0);
}

/* Selected rows of random_batch(·, width, seed), rows ascending: one pass
 * over the stream, skipping whole 312-word blocks between them (the skipped
 * outputs need only the twist, not the tempering), for samples of batches
 * too large to generate whole (cfg5: 17 GB of inputs). */
void orc_random_rows(const int64_t* rows, int64_t n, int64_t width, uint64_t seed, double* out) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  uint64_t pos = 0; /* outputs consumed so far */
  for (int64_t i = 0; i < n; ++i) {
    uint64_t want = (uint64_t)rows[i] * (uint64_t)width;
    uint64_t skip = want - pos;
    while (skip > 0) {
      uint64_t left = (uint64_t)(MT_N - r.idx);
      if (r.idx >= MT_N) {
        if (skip >= MT_N) {
          mt_twist(&r);
          r.idx = MT_N;
          skip -= MT_N;
          continue;
        }
        mt_twist(&r);
        left = MT_N;
      }
      uint64_t step = skip < left ? skip : left;
      r.idx += (int)step;
      skip -= step;
    }
    for (int64_t j = 0; j < width; ++j) out[i * width + j] = rng_range(&r, -1.0, 1.0);
    pos = want + (uint64_t)width;
  }
}

uint64_t orc_fnv1a64(const void* data, int64_t bytes, uint64_t h) {
  const unsigned char* p = (const unsigned char*)data;
  if (h == 0) h = 0xcbf29ce484222325ULL;
  for (int64_t i = 0; i < bytes; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ---------------------------------------------------------- workloads ---- */
/* make_default_vocab (src/workload.cpp:30-50): id 0 arity 0 (free), odd ids
 * arity 2, even ids >= 2 arity 1. */
static int vocab_arity(int fid) { return fid == 0 ? 0 : ((fid % 2 == 1) ? 2 : 1); }

typedef struct {
  int32_t* fid;
  int32_t* c0;
  int32_t* c1;
  int32_t n; /* nodes emitted so far in the current program */
  int n_unary, n_binary;
  double bp;
  orc_rng* rng;
} tree_builder;

/* arity pools (src/workload.cpp:54-68): ascending function ids per arity. */
static int pick_leaf(tree_builder* t) {
  (void)rng_int(t->rng, 0, 0); /* pick() draws even from a 1-element pool */
  return 0;
}
static int pick_unary(tree_builder* t) { return 2 * (int)(1 + rng_int(t->rng, 0, t->n_unary - 1)); }
static int pick_binary(tree_builder* t) { return 2 * (int)rng_int(t->rng, 0, t->n_binary - 1) + 1; }

/* TreeBuilder::build (src/workload.cpp:79-98): preorder, ids in prefix order. */
static int32_t tb_build(tree_builder* t, int budget) {
  int32_t id = t->n++;
  t->c0[id] = -1;
  t->c1[id] = -1;
  if (budget == 1) {
    t->fid[id] = pick_leaf(t);
    return id;
  }
  if (budget >= 3 && rng_bernoulli(t->rng, t->bp)) {
    t->fid[id] = pick_binary(t);
    int left_budget = (budget - 1) / 2;
    int32_t l = tb_build(t, left_budget);
    int32_t r = tb_build(t, budget - 1 - left_budget);
    t->c0[id] = l;
    t->c1[id] = r;
    return id;
  }
  t->fid[id] = pick_unary(t);
  t->c0[id] = tb_build(t, budget - 1);
  return id;
}

/* gen_balanced_tree Builder (src/workload.cpp:125-146). */
static int32_t bal_build(tree_builder* t, int level, int depth) {
  int32_t id = t->n++;
  t->c0[id] = -1;
  t->c1[id] = -1;
  if (level == depth - 1) {
    t->fid[id] = pick_leaf(t);
    return id;
  }
  t->fid[id] = pick_binary(t);
  int32_t l = bal_build(t, level + 1, depth);
  int32_t r = bal_build(t, level + 1, depth);
  t->c0[id] = l;
  t->c1[id] = r;
  return id;
}

/* gen_random_dag (src/workload.cpp:159-205): tree with branch 0.4, then leaves
 * merged onto earlier kept leaves with probability share_prob, compacted. */
static int32_t gen_dag(int length, double share, int n_unary, int n_binary, orc_rng* rng,
                       int32_t* fid, int32_t* c0, int32_t* c1) {
  int32_t* tf = (int32_t*)malloc(sizeof(int32_t) * (size_t)length * 3);
  int32_t* t0 = tf + length;
  int32_t* t1 = t0 + length;
  tree_builder t = {tf, t0, t1, 0, n_unary, n_binary, 0.4, rng};
  tb_build(&t, length);
  int32_t n = t.n;
  int32_t* redirect = (int32_t*)malloc(sizeof(int32_t) * (size_t)n * 4);
  int32_t* removed = redirect + n;
  int32_t* kept = removed + n;
  int32_t* new_id = kept + n;
  int32_t n_kept = 0;
  for (int32_t v = 0; v < n; ++v) {
    redirect[v] = v;
    removed[v] = 0;
  }
  for (int32_t v = 0; v < n; ++v) {
    if (t0[v] >= 0) continue; /* leaves in id order */
    if (n_kept > 0 && rng_bernoulli(rng, share)) {
      int32_t target = kept[rng_int(rng, 0, n_kept - 1)];
      redirect[v] = target;
      removed[v] = 1;
    } else {
      kept[n_kept++] = v;
    }
  }
  int32_t m = 0;
  for (int32_t v = 0; v < n; ++v) {
    new_id[v] = -1;
    if (removed[v]) continue;
    new_id[v] = m;
    fid[m] = tf[v];
    c0[m] = -1;
    c1[m] = -1;
    ++m;
  }
  for (int32_t v = 0; v < n; ++v) {
    if (removed[v]) continue;
    int32_t nv = new_id[v];
    if (t0[v] >= 0) c0[nv] = new_id[redirect[t0[v]]];
    if (t1[v] >= 0) c1[nv] = new_id[redirect[t1[v]]];
  }
  free(redirect);
  free(tf);
  return m;
}

/* gen_batch (src/workload.cpp:214-246). kind: 0 balanced, 1 chain-heavy,
 * 2 random-dag. Returns total nodes (pass prog_off == NULL to size only). */
int64_t orc_gen_batch(int kind, int64_t b, int p, int depth, int length, double branch_prob,
                      uint64_t seed, int32_t* prog_off, int32_t* fid, int32_t* child0,
                      int32_t* child1, int32_t* root) {
  int n_unary = 0, n_binary = 0;
  for (int id = 1; id < p; ++id) {
    if (vocab_arity(id) == 1) ++n_unary; else ++n_binary;
  }
  int max_nodes = kind == 0 ? (1 << depth) - 1 : length;
  int32_t* sf = (int32_t*)malloc(sizeof(int32_t) * (size_t)max_nodes * 3);
  int32_t* s0 = sf + max_nodes;
  int32_t* s1 = s0 + max_nodes;
  orc_rng main_rng;
  orc_rng_seed(&main_rng, seed);
  int64_t off = 0;
  for (int64_t i = 0; i < b; ++i) {
    uint64_t program_seed = orc_mix_seed(seed, 0x70c1ULL + (uint64_t)i);
    orc_rng rng;
    orc_rng_seed(&rng, program_seed);
    int32_t n = 0;
    if (kind == 0) {
      tree_builder t = {sf, s0, s1, 0, n_unary, n_binary, 0.0, &rng};
      bal_build(&t, 0, depth);
      n = t.n;
    } else {
      int lo = length / 2 > 1 ? length / 2 : 1;
      int len = (int)rng_int(&main_rng, lo, length);
      if (kind == 1) {
        tree_builder t = {sf, s0, s1, 0, n_unary, n_binary, branch_prob, &rng};
        tb_build(&t, len);
        n = t.n;
      } else {
        n = gen_dag(len, branch_prob, n_unary, n_binary, &rng, sf, s0, s1);
      }
    }
    if (prog_off) {
      prog_off[i] = (int32_t)off;
      root[i] = 0;
      memcpy(fid + off, sf, sizeof(int32_t) * (size_t)n);
      memcpy(child0 + off, s0, sizeof(int32_t) * (size_t)n);
      memcpy(child1 + off, s1, sizeof(int32_t) * (size_t)n);
    }
    off += n;
  }
  if (prog_off) prog_off[b] = (int32_t)off;
  free(sf);
  return off;
}

/* ------------------------------------------------- labels & schedule ---- */
/* max_root_distance_labels (src/program.cpp:239-272): Kahn from the root,
 * label[c] = max(label[c], label[v] + 1). Returns 0, or 5 (InvalidProgram)
 * on a cycle / unreachable node. */
int orc_labels(int64_t b, const int32_t* prog_off, const int32_t* child0, const int32_t* child1,
               const int32_t* root, int32_t* labels, int32_t* d_max) {
  int32_t best = 0;
  int32_t cap = 0;
  for (int64_t e = 0; e < b; ++e) {
    int32_t n = prog_off[e + 1] - prog_off[e];
    if (n > cap) cap = n;
  }
  int32_t* indeg = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap > 0 ? cap : 1) * 2);
  int32_t* queue = indeg + cap;
  int rc = 0;
  for (int64_t e = 0; e < b && rc == 0; ++e) {
    int32_t base = prog_off[e], n = prog_off[e + 1] - base;
    for (int32_t v = 0; v < n; ++v) {
      indeg[v] = 0;
      labels[base + v] = 0;
    }
    for (int32_t v = 0; v < n; ++v) {
      if (child0[base + v] >= 0) ++indeg[child0[base + v]];
      if (child1[base + v] >= 0) ++indeg[child1[base + v]];
    }
    int32_t head = 0, tail = 0;
    queue[tail++] = root[e];
    while (head < tail) {
      int32_t v = queue[head++];
      int32_t cs[2] = {child0[base + v], child1[base + v]};
      for (int k = 0; k < 2; ++k) {
        int32_t c = cs[k];
        if (c < 0) continue;
        int32_t cand = labels[base + v] + 1;
        if (cand > labels[base + c]) labels[base + c] = cand;
        if (--indeg[c] == 0) queue[tail++] = c;
      }
    }
    if (head != n) rc = 5;
    for (int32_t v = 0; v < n; ++v) {
      if (labels[base + v] > best) best = labels[base + v];
    }
  }
  free(indeg);
  *d_max = best;
  return rc;
}

/* schedule_improved + make_step (src/schedule.cpp:66-79, 135-164): pools by
 * label, emitted deepest first; within a step groups ascend by function id
 * and members ascend by (example, node). Implemented as a stable counting sort
 * over the (example, node)-ordered node list keyed by (d_max - label, fid). */
int orc_schedule_improved(int64_t b, int p, const int32_t* prog_off, const int32_t* fid,
                          const int32_t* child0, const int32_t* child1, const int32_t* root,
                          int64_t* counts, int32_t* step_group_off, int32_t* group_fid,
                          int32_t* group_member_off, int32_t* member_example,
                          int32_t* member_node) {
  int64_t N = b > 0 ? prog_off[b] : 0;
  if (b == 0) { /* empty batch => 0 steps (schedule.cpp:147) */
    counts[0] = counts[1] = counts[2] = 0;
    if (step_group_off) step_group_off[0] = 0;
    if (group_member_off) group_member_off[0] = 0;
    return 0;
  }
  int32_t* labels = (int32_t*)malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1));
  int32_t d_max = 0;
  int rc = orc_labels(b, prog_off, child0, child1, root, labels, &d_max);
  if (rc) {
    free(labels);
    return rc;
  }
  int64_t n_keys = (int64_t)(d_max + 1) * p;
  int64_t* count = (int64_t*)calloc((size_t)n_keys + 1, sizeof(int64_t));
  for (int64_t g = 0; g < N; ++g) count[(int64_t)(d_max - labels[g]) * p + fid[g]]++;
  int64_t groups = 0;
  for (int64_t k = 0; k < n_keys; ++k) groups += count[k] > 0;
  counts[0] = d_max + 1;
  counts[1] = groups;
  counts[2] = N;
  if (step_group_off) {
    int64_t* start = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_keys + 1));
    int64_t acc = 0, gi = 0;
    for (int64_t k = 0; k < n_keys; ++k) {
      if (k % p == 0) step_group_off[k / p] = (int32_t)gi;
      start[k] = acc;
      if (count[k] > 0) {
        group_fid[gi] = (int32_t)(k % p);
        group_member_off[gi] = (int32_t)acc;
        ++gi;
      }
      acc += count[k];
    }
    step_group_off[d_max + 1] = (int32_t)gi;
    group_member_off[gi] = (int32_t)acc;
    for (int64_t e = 0; e < b; ++e) {
      for (int32_t g = prog_off[e]; g < prog_off[e + 1]; ++g) {
        int64_t key = (int64_t)(d_max - labels[g]) * p + fid[g];
        int64_t pos = start[key]++;
        member_example[pos] = (int32_t)e;
        member_node[pos] = g - prog_off[e];
      }
    }
    free(start);
  }
  free(count);
  free(labels);
  return 0;
}

/* -------------------------------------------------------- dense module ---- */
/* make_module_impl (src/modules.cpp:13-28): Rng(mix_seed(seed, fid)); weights
 * [arity*W x W] input-major, then bias[W], all uniform(-0.5,0.5)/sqrt(arity*W). */
void orc_dense_weights(int arity, int width, uint64_t seed, int fid, double* w, double* bias) {
  if (arity == 0) return;
  double scale = 1.0 / sqrt((double)(arity * width));
  orc_rng r;
  orc_rng_seed(&r, orc_mix_seed(seed, (uint64_t)fid));
  int64_t nw = (int64_t)arity * width * width;
  for (int64_t i = 0; i < nw; ++i) w[i] = rng_range(&r, -0.5, 0.5) * scale;
  for (int j = 0; j < width; ++j) bias[j] = rng_range(&r, -0.5, 0.5) * scale;
}

/* apply_module for one row (src/modules.cpp:83-105): acc = bias; ascending
 * (k, i) fused multiply-adds; relu as `> 0.0 ? v : 0.0`. Row-independent. */
static void dense_row(int arity, int width, const double* w, const double* bias,
                      const double* const* xs, double* out) {
  for (int j = 0; j < width; ++j) out[j] = bias[j];
  for (int k = 0; k < arity; ++k) {
    for (int i = 0; i < width; ++i) {
      double xi = xs[k][i];
      const double* wrow = w + ((int64_t)k * width + i) * width;
      for (int j = 0; j < width; ++j) out[j] = fma(xi, wrow[j], out[j]);
    }
  }
  for (int j = 0; j < width; ++j) out[j] = out[j] > 0.0 ? out[j] : 0.0;
}

/* ------------------------------------- residual conv block (Tier B) ---- */
/* NOT IN THE REFERENCE: parity unpinned. Init follows the
 * reference style (src/modules.cpp:13-28): Rng(mix_seed(seed, fid)), draws
 * in the order w0, b0 (binary only), w1, b1, w2, b2, each uniform(-0.5,0.5)
 * scaled by 1/sqrt(fan_in) (fan_in = 2C for the 1x1 projection, 9C for a
 * 3x3). Weights are input-major: w[(tap*Cin + ci)*C + co], taps (kh, kw)
 * row-major. */
void orc_resblock_weights(int arity, int C, uint64_t seed, int fid, double* w0, double* b0,
                          double* w1, double* b1, double* w2, double* b2) {
  orc_rng r;
  orc_rng_seed(&r, orc_mix_seed(seed, (uint64_t)fid));
  if (arity == 2) {
    double s0 = 1.0 / sqrt((double)(2 * C));
    for (int64_t i = 0; i < (int64_t)2 * C * C; ++i) w0[i] = rng_range(&r, -0.5, 0.5) * s0;
    for (int j = 0; j < C; ++j) b0[j] = rng_range(&r, -0.5, 0.5) * s0;
  }
  double s = 1.0 / sqrt((double)(9 * C));
  for (int64_t i = 0; i < (int64_t)9 * C * C; ++i) w1[i] = rng_range(&r, -0.5, 0.5) * s;
  for (int j = 0; j < C; ++j) b1[j] = rng_range(&r, -0.5, 0.5) * s;
  for (int64_t i = 0; i < (int64_t)9 * C * C; ++i) w2[i] = rng_range(&r, -0.5, 0.5) * s;
  for (int j = 0; j < C; ++j) b2[j] = rng_range(&r, -0.5, 0.5) * s;
}

/* Zero-padded stride-1 convolution, ksize 1 or 3, CHW in/out; acc is an
 * HW x Cout scratch. out[co] = bias[co] + sum_{tap, ci} x * w. */
static void conv2d(const double* in, int Cin, int H, int W, int ksize, const double* w,
                   const double* bias, int Cout, double* acc, double* out) {
  int HW = H * W, pad = ksize / 2;
  for (int q = 0; q < HW; ++q)
    for (int co = 0; co < Cout; ++co) acc[(int64_t)q * Cout + co] = bias[co];
  for (int kh = 0; kh < ksize; ++kh) {
    for (int kw = 0; kw < ksize; ++kw) {
      int tap = kh * ksize + kw;
      for (int ci = 0; ci < Cin; ++ci) {
        const double* wrow = w + ((int64_t)tap * Cin + ci) * Cout;
        const double* plane = in + (int64_t)ci * HW;
        for (int h = 0; h < H; ++h) {
          int ih = h + kh - pad;
          if (ih < 0 || ih >= H) continue;
          for (int x = 0; x < W; ++x) {
            int iw = x + kw - pad;
            if (iw < 0 || iw >= W) continue;
            double xv = plane[ih * W + iw];
            double* a = acc + (int64_t)(h * W + x) * Cout;
            for (int co = 0; co < Cout; ++co) a[co] = fma(xv, wrow[co], a[co]);
          }
        }
      }
    }
  }
  for (int q = 0; q < HW; ++q)
    for (int co = 0; co < Cout; ++co) out[(int64_t)co * HW + q] = acc[(int64_t)q * Cout + co];
}

typedef struct {
  double *w0, *b0, *w1, *b1, *w2, *b2;
} resblock_w;

/* unary: y = relu(x + conv3x3_2(relu(conv3x3_1(x) + b1)) + b2)
 * binary: z = relu(conv1x1([x; y]) + b0), then the unary block on z. */
static void resblock_row(int arity, int C, int H, int W, const resblock_w* m,
                         const double* const* xs, double* out, double* scratch) {
  int64_t F = (int64_t)C * H * W;
  double* acc = scratch;           /* HW x C */
  double* t = acc + (int64_t)H * W * C;
  double* z = t + F;
  double* cat = z + F;             /* 2F */
  const double* x = xs[0];
  if (arity == 2) {
    memcpy(cat, xs[0], sizeof(double) * (size_t)F);
    memcpy(cat + F, xs[1], sizeof(double) * (size_t)F);
    conv2d(cat, 2 * C, H, W, 1, m->w0, m->b0, C, acc, z);
    for (int64_t i = 0; i < F; ++i) z[i] = z[i] > 0.0 ? z[i] : 0.0;
    x = z;
  }
  conv2d(x, C, H, W, 3, m->w1, m->b1, C, acc, t);
  for (int64_t i = 0; i < F; ++i) t[i] = t[i] > 0.0 ? t[i] : 0.0;
  conv2d(t, C, H, W, 3, m->w2, m->b2, C, acc, out);
  for (int64_t i = 0; i < F; ++i) {
    double v = x[i] + out[i];
    out[i] = v > 0.0 ? v : 0.0;
  }
}

/* ------------------------------------------------------------ execute ---- */
/* execute (src/executor.cpp:95-176): per step and group, count the trace
 * (peak_group_rows includes free leaf groups, :119-124), fetch leaves from
 * inputs[example] (:126-137), gather child k of each member as operand k
 * (:139-151), apply (:153-155), scatter (:161-163); outputs are root rows. */
int orc_execute(int module_kind, int64_t b, int p, int width, int C, int H, int W,
                const int32_t* prog_off, const int32_t* fid, const int32_t* child0,
                const int32_t* child1, const int32_t* root, int64_t n_steps,
                const int32_t* step_group_off, const int32_t* group_fid,
                const int32_t* group_member_off, const int32_t* member_example,
                const int32_t* member_node, const double* inputs, uint64_t module_seed,
                double* outputs, int64_t* trace, int64_t* per_function_calls, double* seconds) {
  if (module_kind == 1) width = C * H * W;
  int64_t N = b > 0 ? prog_off[b] : 0;
  double* store = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1) * (size_t)width);
  char* present = (char*)calloc((size_t)(N > 0 ? N : 1), 1);
  /* module weights per function id (ModuleSet, src/modules.cpp:30-35) */
  double** wts = (double**)calloc((size_t)p, sizeof(double*));
  resblock_w* rw = (resblock_w*)calloc((size_t)p, sizeof(resblock_w));
  for (int f = 1; f < p; ++f) {
    int a = vocab_arity(f);
    if (module_kind == 0) {
      wts[f] = (double*)malloc(sizeof(double) * ((size_t)a * width * width + (size_t)width));
      orc_dense_weights(a, width, module_seed, f, wts[f], wts[f] + (int64_t)a * width * width);
    } else {
      int64_t CC = (int64_t)C * C;
      double* blk = (double*)malloc(sizeof(double) * (size_t)(2 * CC + C + 2 * (9 * CC + C)));
      wts[f] = blk;
      rw[f].w0 = blk;
      rw[f].b0 = blk + 2 * CC;
      rw[f].w1 = rw[f].b0 + C;
      rw[f].b1 = rw[f].w1 + 9 * CC;
      rw[f].w2 = rw[f].b1 + C;
      rw[f].b2 = rw[f].w2 + 9 * CC;
      orc_resblock_weights(a, C, module_seed, f, rw[f].w0, rw[f].b0, rw[f].w1, rw[f].b1,
                           rw[f].w2, rw[f].b2);
    }
  }
  double* scratch = NULL;
  if (module_kind == 1) {
    int64_t F = (int64_t)C * H * W;
    scratch = (double*)malloc(sizeof(double) * (size_t)(F + 4 * F + F));
  }
  int rc = 0;
  int64_t expensive = 0, peak = 0;
  for (int f = 0; f < p; ++f) per_function_calls[f] = 0;
  double t_module = 0.0, t_stack = 0.0, t0 = now_s();
  for (int64_t s = 0; s < n_steps && rc == 0; ++s) {
    for (int32_t gi = step_group_off[s]; gi < step_group_off[s + 1] && rc == 0; ++gi) {
      int f = group_fid[gi];
      int64_t rows = group_member_off[gi + 1] - group_member_off[gi];
      if (rows > peak) peak = rows;
      per_function_calls[f]++;
      if (f != 0) ++expensive;
      int a = vocab_arity(f);
      for (int32_t mi = group_member_off[gi]; mi < group_member_off[gi + 1]; ++mi) {
        int32_t e = member_example[mi];
        int64_t g = prog_off[e] + member_node[mi];
        if (present[g]) {
          rc = 12; /* SingleAssignmentViolation -> DB_ERR_INTERNAL */
          break;
        }
        double* dst = store + g * width;
        if (a == 0) {
          double ts = now_s();
          memcpy(dst, inputs + (int64_t)e * width, sizeof(double) * (size_t)width);
          t_stack += now_s() - ts;
        } else {
          const double* xs[2];
          int32_t cs[2] = {child0[g], child1[g]};
          for (int k = 0; k < a; ++k) {
            int64_t cg = prog_off[e] + cs[k];
            if (!present[cg]) {
              rc = 7; /* MissingOperand */
              break;
            }
            xs[k] = store + cg * width;
          }
          if (rc) break;
          double tm = now_s();
          if (module_kind == 0) {
            dense_row(a, width, wts[f], wts[f] + (int64_t)a * width * width, xs, dst);
          } else {
            resblock_row(a, C, H, W, &rw[f], xs, dst, scratch);
          }
          t_module += now_s() - tm;
          for (int64_t j = 0; j < width; ++j) {
            if (!isfinite(dst[j])) {
              rc = 9; /* NonFiniteValue */
              break;
            }
          }
        }
        present[g] = 1;
      }
    }
  }
  for (int64_t e = 0; e < b && rc == 0; ++e) {
    int64_t g = prog_off[e] + root[e];
    if (!present[g]) {
      rc = 7;
      break;
    }
    memcpy(outputs + e * width, store + g * width, sizeof(double) * (size_t)width);
  }
  if (seconds) {
    seconds[0] = t_module;
    seconds[1] = t_stack;
    seconds[2] = now_s() - t0;
  }
  trace[0] = expensive;
  trace[1] = peak;
  trace[2] = n_steps;
  for (int f = 0; f < p; ++f) free(wts[f]);
  free(wts);
  free(rw);
  free(scratch);
  free(present);
  free(store);
  return rc;
}

/* ---------------------------------------------------------------- MoE ---- */
/* top_k_gate (src/moe.cpp:36-69): rank by (score desc, id asc) — `!=` on
 * doubles, so -0.0 ties +0.0 and falls to the id — take the first k (slot
 * order = rank order); weight_i = exp(s_i - s_0) / sum_{j<k} exp(s_j - s_0)
 * with the denominator summed in rank order. */
int orc_topk(const double* scores, int64_t T, int64_t n, int64_t k, int32_t* ids,
             double* weights) {
  if (k < 1 || k > n) return 8; /* KTooLarge -> shape mismatch */
  for (int64_t i = 0; i < T * n; ++i)
    if (!isfinite(scores[i])) return 9;
  char* taken = (char*)malloc((size_t)n);
  double* sel = (double*)malloc(sizeof(double) * (size_t)k);
  for (int64_t t = 0; t < T; ++t) {
    const double* s = scores + t * n;
    memset(taken, 0, (size_t)n);
    for (int64_t r = 0; r < k; ++r) {
      int64_t best = -1;
      for (int64_t j = 0; j < n; ++j) {
        if (taken[j]) continue;
        if (best < 0 || s[j] > s[best]) best = j; /* ascending j keeps the lower id on ties */
      }
      taken[best] = 1;
      ids[t * k + r] = (int32_t)best;
      sel[r] = s[best];
    }
    double mx = sel[0], denom = 0.0;
    for (int64_t r = 0; r < k; ++r) denom += exp(sel[r] - mx);
    for (int64_t r = 0; r < k; ++r) weights[t * k + r] = exp(sel[r] - mx) / denom;
  }
  free(sel);
  free(taken);
  return 0;
}

/* ExpertSet ctor (src/moe.cpp:71-88) for one expert: Rng(mix_seed(seed, id));
 * w1 [d x h] input-major scaled 1/sqrt(d), then w2 [h x d] scaled 1/sqrt(h). */
void orc_expert_weights(int64_t d, int64_t h, uint64_t seed, int64_t id, double* w1, double* w2) {
  double s1 = 1.0 / sqrt((double)d), s2 = 1.0 / sqrt((double)h);
  orc_rng r;
  orc_rng_seed(&r, orc_mix_seed(seed, (uint64_t)id));
  for (int64_t i = 0; i < d * h; ++i) w1[i] = rng_range(&r, -0.5, 0.5) * s1;
  for (int64_t i = 0; i < h * d; ++i) w2[i] = rng_range(&r, -0.5, 0.5) * s2;
}

/* moe_forward_batched (src/moe.cpp:200-270) with ExpertSet::apply
 * (:98-145): per occupied expert (ascending id) stack the member rows in
 * (token, slot) order, h = relu(x W1), y = h W2 (ascending-index FMAs), stage
 * at token*k + slot; combine per token in slot order out += w * y.
 * expert_subset (optional, ascending ids) restricts the work to a sample of
 * experts for bounded CPU timing; their rows are then the only valid ones.
 * trace = [expensive_calls, peak_group_rows]; seconds = [module, stacking,
 * total] with expert weight generation excluded (the reference builds its
 * ExpertSet before execution). */
int orc_moe_forward(const double* inputs, int64_t T, int64_t d, int64_t h, int64_t n, int64_t k,
                    const int32_t* ids, const double* weights, uint64_t expert_seed,
                    const int32_t* expert_subset, int64_t n_subset, double* out, int64_t* trace,
                    double* seconds) {
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t i = 0; i < T * k; ++i) cnt[ids[i]]++;
  int64_t* start = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t acc = 0;
  for (int64_t e = 0; e < n; ++e) {
    start[e] = acc;
    acc += cnt[e];
  }
  start[n] = acc;
  int64_t* items = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T * k > 0 ? T * k : 1));
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  memcpy(fill, start, sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < T * k; ++i) items[fill[ids[i]]++] = i; /* stable: (token, slot) order */
  double* staged = (double*)calloc((size_t)(T * k) * (size_t)d, sizeof(double));
  double* w1 = (double*)malloc(sizeof(double) * (size_t)(d * h));
  double* w2 = (double*)malloc(sizeof(double) * (size_t)(h * d));
  double* hid = (double*)malloc(sizeof(double) * (size_t)h);
  double* y = (double*)malloc(sizeof(double) * (size_t)d);
  int64_t calls = 0, peak = 0, si = 0;
  double t_module = 0.0, t_total = 0.0;
  for (int64_t e = 0; e < n; ++e) {
    if (cnt[e] == 0) continue;
    if (expert_subset) {
      while (si < n_subset && expert_subset[si] < e) ++si;
      if (si >= n_subset || expert_subset[si] != e) continue;
    }
    orc_expert_weights(d, h, expert_seed, e, w1, w2);
    double t0 = now_s();
    ++calls;
    if (cnt[e] > peak) peak = cnt[e];
    for (int64_t r = start[e]; r < start[e + 1]; ++r) {
      int64_t item = items[r];
      const double* x = inputs + (item / k) * d;
      for (int64_t j = 0; j < h; ++j) hid[j] = 0.0;
      for (int64_t i = 0; i < d; ++i) {
        const double* wrow = w1 + i * h;
        for (int64_t j = 0; j < h; ++j) hid[j] = fma(x[i], wrow[j], hid[j]);
      }
      for (int64_t j = 0; j < h; ++j) hid[j] = hid[j] > 0.0 ? hid[j] : 0.0;
      for (int64_t j = 0; j < d; ++j) y[j] = 0.0;
      for (int64_t i = 0; i < h; ++i) {
        const double* wrow = w2 + i * d;
        for (int64_t j = 0; j < d; ++j) y[j] = fma(hid[i], wrow[j], y[j]);
      }
      memcpy(staged + item * d, y, sizeof(double) * (size_t)d);
    }
    double dt = now_s() - t0;
    t_module += dt;
    t_total += dt;
  }
  double tc = now_s();
  for (int64_t t = 0; t < T; ++t) {
    double* o = out + t * d;
    for (int64_t j = 0; j < d; ++j) o[j] = 0.0;
    for (int64_t s = 0; s < k; ++s) {
      double wgt = weights[t * k + s];
      const double* src = staged + (t * k + s) * d;
      for (int64_t j = 0; j < d; ++j) o[j] = fma(wgt, src[j], o[j]);
    }
  }
  t_total += now_s() - tc;
  trace[0] = calls;
  trace[1] = peak;
  if (seconds) {
    seconds[0] = t_module;
    seconds[1] = t_total - t_module;
    seconds[2] = t_total;
  }
  free(y);
  free(hid);
  free(w2);
  free(w1);
  free(staged);
  free(fill);
  free(items);
  free(start);
  free(cnt);
  return 0;
}

/* ------------------------------------------------ IEP classifier head ---- */
/* NOT IN THE REFERENCE (its path ends at the root feature maps, SPEC.md:13;
 * SURVEY.md §8(f)4): the IEP classifier after Johnson et al., as the device
 * head (head.cu) defines it. Init in the reference style
 * (src/modules.cpp:13-28): Rng(mix_seed(seed, 0x4ead)), draws wp [C][P],
 * bp[P], w1 [49P][F], b1[F], w2 [F][A], b2[A] (input-major), each
 * uniform(-0.5, 0.5) / sqrt(fan_in). */
void orc_head_weights(int C, int P, int F, int A, uint64_t seed, double* wp, double* bp, double* w1,
                      double* b1, double* w2, double* b2) {
  orc_rng r;
  orc_rng_seed(&r, orc_mix_seed(seed, 0x4eadULL));
  int64_t K1 = (int64_t)49 * P;
  double sp = 1.0 / sqrt((double)C), s1 = 1.0 / sqrt((double)K1), s2 = 1.0 / sqrt((double)F);
  for (int64_t i = 0; i < (int64_t)C * P; ++i) wp[i] = rng_range(&r, -0.5, 0.5) * sp;
  for (int j = 0; j < P; ++j) bp[j] = rng_range(&r, -0.5, 0.5) * sp;
  for (int64_t i = 0; i < K1 * F; ++i) w1[i] = rng_range(&r, -0.5, 0.5) * s1;
  for (int j = 0; j < F; ++j) b1[j] = rng_range(&r, -0.5, 0.5) * s1;
  for (int64_t i = 0; i < (int64_t)F * A; ++i) w2[i] = rng_range(&r, -0.5, 0.5) * s2;
  for (int j = 0; j < A; ++j) b2[j] = rng_range(&r, -0.5, 0.5) * s2;
}

/* logits[e][a] of b root maps (CHW rows of C×14×14, the executor's output
 * layout): proj = relu(conv1x1 + bp) [196][P]; pooled[q][c] = max over the
 * 2×2 window q = ph·7 + pw; hidden = relu(w1ᵀ·flatten + b1) with flatten
 * index q·P + c; logits = w2ᵀ·hidden + b2. fp64. */
int orc_head_forward(int64_t b, const double* roots, int C, int P, int F, int A, uint64_t seed,
                     double* logits) {
  const int HW = 196;
  int64_t K1 = (int64_t)49 * P;
  double* wp = (double*)malloc(sizeof(double) * (size_t)C * P);
  double* bp = (double*)malloc(sizeof(double) * (size_t)P);
  double* w1 = (double*)malloc(sizeof(double) * (size_t)(K1 * F));
  double* b1 = (double*)malloc(sizeof(double) * (size_t)F);
  double* w2 = (double*)malloc(sizeof(double) * (size_t)F * A);
  double* b2 = (double*)malloc(sizeof(double) * (size_t)A);
  double* proj = (double*)malloc(sizeof(double) * (size_t)HW * P);
  double* pooled = (double*)malloc(sizeof(double) * (size_t)K1);
  double* hid = (double*)malloc(sizeof(double) * (size_t)F);
  if (!wp || !bp || !w1 || !b1 || !w2 || !b2 || !proj || !pooled || !hid) return 1;
  orc_head_weights(C, P, F, A, seed, wp, bp, w1, b1, w2, b2);
  for (int64_t e = 0; e < b; ++e) {
    const double* x = roots + e * (int64_t)C * HW;
    for (int q = 0; q < HW; ++q) {
      double* o = proj + (int64_t)q * P;
      for (int c = 0; c < P; ++c) o[c] = bp[c];
      for (int ci = 0; ci < C; ++ci) {
        double xv = x[(int64_t)ci * HW + q];
        const double* wr = wp + (int64_t)ci * P;
        for (int c = 0; c < P; ++c) o[c] = fma(xv, wr[c], o[c]);
      }
      for (int c = 0; c < P; ++c) o[c] = o[c] > 0.0 ? o[c] : 0.0;
    }
    for (int q = 0; q < 49; ++q) {
      int ph = q / 7, pw = q % 7;
      for (int c = 0; c < P; ++c) {
        double m = 0.0;
        for (int t = 0; t < 4; ++t) {
          int px = (2 * ph + t / 2) * 14 + 2 * pw + t % 2;
          double v = proj[(int64_t)px * P + c];
          m = (t == 0 || v > m) ? v : m;
        }
        pooled[(int64_t)q * P + c] = m;
      }
    }
    for (int f = 0; f < F; ++f) hid[f] = b1[f];
    for (int64_t k = 0; k < K1; ++k) {
      double xv = pooled[k];
      const double* wr = w1 + k * F;
      for (int f = 0; f < F; ++f) hid[f] = fma(xv, wr[f], hid[f]);
    }
    for (int f = 0; f < F; ++f) hid[f] = hid[f] > 0.0 ? hid[f] : 0.0;
    double* lo = logits + e * A;
    for (int a = 0; a < A; ++a) lo[a] = b2[a];
    for (int f = 0; f < F; ++f)
      for (int a = 0; a < A; ++a) lo[a] = fma(hid[f], w2[(int64_t)f * A + a], lo[a]);
  }
  free(wp); free(bp); free(w1); free(b1); free(w2); free(b2); free(proj); free(pooled); free(hid);
  return 0;
}
