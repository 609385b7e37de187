/*
 * fmoe_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded, fp64 restatement of the FastMoE reference's
 * MoE-layer hot path (/root/reference/proj, C++20 CPU implementation).  It is
 * the *checker* for the B200 kernels: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * library (paper_2103_13262_b200/libfmoe_b200.so) never links or calls it.
 *
 * Parity pinning: every function here is checked bit-for-bit against the
 * reference itself, compiled side by side from its own sources into
 * oracle/_ref/libfmoe_ref.so (see oracle/Makefile, tests/test_oracle.py), and
 * against the known-answer vectors of the reference's tests plus the golden
 * fixtures in tests/golden/ generated from that build.
 *
 * Arithmetic contract (what makes results bit-identical to the reference,
 * which is compiled with GCC's default -ffp-contract=fast on an FMA target):
 *   matmul            acc = fma(a_ik, b_kj, acc), k ascending, acc0 = +0.0
 *                     (matrix.cpp:56-88 multiply_row_range)
 *   add_bias_rows     one rounded add after the full dot product (matrix.cpp:128-138)
 *   relu              x < 0 -> 0, keeps -0.0                   (matrix.cpp:140-145)
 *   relu_backward     strict x > 0                             (matrix.cpp:147-153)
 *   softmax_rows      max, exp(x-max), sequential sum, divide  (matrix.cpp:155-170)
 *   topk_rows         stable descending order, ties -> lower column (matrix.cpp:172-189)
 *   gather_combine    out = fma(w, y, out) in slot order       (dispatch.cpp:61-78)
 *   scatter_backward  out += g, slot order, from +0.0          (dispatch.cpp:80-95)
 *   gather_combine_bwd  d = w*dy (one rounding); dot = dot_ref over c (dispatch.cpp:97-126)
 *   gate_backward     <ds, s> = dot_ref over experts           (gate.cpp:52-56)
 * dot_ref is how GCC compiles the reference's in-order reductions
 * `dot += a[c] * b[c]` at -O3 on an AVX2+FMA target (checked in the
 * disassembly of oracle/_ref/libfmoe_ref.so): the loop is vectorised as a
 * fold-left reduction, so products are rounded on their own and added in
 * order; only a final odd element, left to the scalar epilogue, is fused.
 * This file is compiled with -ffp-contract=off and spells every fused
 * multiply-add explicitly, so the contract does not depend on the compiler.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_SHAPE 1
#define ORC_PROTOCOL 2

static char g_err[256];
const char* orc_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
  strncpy(g_err, msg, sizeof(g_err) - 1);
  return code;
}

/* ------------------------------------------------------------------ rng */
/* std::mt19937_64 (the engine behind UniformRng, rng.hpp:12-28). */
typedef struct {
  uint64_t s[312];
  int i;
} orc_mt64;

static void mt64_seed(orc_mt64* m, uint64_t seed) {
  m->s[0] = seed;
  for (int i = 1; i < 312; ++i)
    m->s[i] = 6364136223846793005ULL * (m->s[i - 1] ^ (m->s[i - 1] >> 62)) + (uint64_t)i;
  m->i = 312;
}

static uint64_t mt64_next(orc_mt64* m) {
  const uint64_t hi = 0xFFFFFFFF80000000ULL, lo = 0x7FFFFFFFULL, a = 0xB5026F5AA96619E9ULL;
  if (m->i >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (m->s[i] & hi) | (m->s[(i + 1) % 312] & lo);
      uint64_t v = m->s[(i + 156) % 312] ^ (x >> 1);
      if (x & 1) v ^= a;
      m->s[i] = v;
    }
    m->i = 0;
  }
  uint64_t x = m->s[m->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* stream_seed: splitmix64 finaliser (rng.cpp:6-11). */
uint64_t orc_stream_seed(uint64_t base, uint64_t stream) {
  uint64_t z = base + 0x9E3779B97F4A7C15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* UniformRng::fill (rng.hpp:17-25): lo + u*(hi-lo), u = (x>>11)*2^-53.  The
 * reference compiles that expression with contraction, i.e. fma(u, hi-lo, lo). */
static void fill_uniform(orc_mt64* m, double* out, int64_t n, double lo, double hi) {
  const double span = hi - lo;
  for (int64_t i = 0; i < n; ++i) {
    const double u = (double)(mt64_next(m) >> 11) * 0x1.0p-53;
    out[i] = fma(u, span, lo);
  }
}

void orc_uniform_fill(uint64_t seed, double* out, int64_t n, double lo, double hi) {
  orc_mt64 m;
  mt64_seed(&m, seed);
  fill_uniform(&m, out, n, lo, hi);
}

/* init_gate (gate.cpp:16-21): stream 0x67617465 ("gate"). */
void orc_init_gate(uint64_t seed, int64_t d_m, int64_t total, double* wg) {
  orc_uniform_fill(orc_stream_seed(seed, 0x67617465ULL), wg, d_m * total, -0.1, 0.1);
}

/* init_expert (expert.cpp:13-22) for global expert g (moe_layer.cpp:38-43):
 * stream_seed(seed, g), fill order w1, b1, w2, b2. */
void orc_init_expert(uint64_t seed, uint64_t global_index, int64_t d_m, int64_t d_h,
                     double* w1, double* b1, double* w2, double* b2) {
  orc_mt64 m;
  mt64_seed(&m, orc_stream_seed(seed, global_index));
  fill_uniform(&m, w1, d_m * d_h, -0.1, 0.1);
  fill_uniform(&m, b1, d_h, -0.1, 0.1);
  fill_uniform(&m, w2, d_h * d_m, -0.1, 0.1);
  fill_uniform(&m, b2, d_m, -0.1, 0.1);
}

/* In-order dot product as compiled by GCC for the reference (see header). */
static double dot_ref(const double* a, int64_t sa, const double* b, int64_t sb, int64_t n) {
  double dot = 0.0;
  const int64_t paired = n & ~(int64_t)1;
  for (int64_t c = 0; c < paired; ++c) {
    const double p = a[c * sa] * b[c * sb];
    dot += p;
  }
  if (n & 1) dot = fma(a[paired * sa], b[paired * sb], dot);
  return dot;
}

/* --------------------------------------------------------------- matmul */
/* out[m x n] = a * b with a(i,k) = a[i*sa_r + k*sa_c], b(k,j) = b[k*sb_r + j*sb_c].
 * Strides let the transposed products of the backward passes (matrix.cpp:121)
 * reuse the same accumulation order without materialising transposes. */
static void matmul_strided(const double* a, int64_t sa_r, int64_t sa_c, const double* b,
                           int64_t sb_r, int64_t sb_c, double* out, int64_t m, int64_t p,
                           int64_t n) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int64_t k = 0; k < p; ++k) acc = fma(a[i * sa_r + k * sa_c], b[k * sb_r + j * sb_c], acc);
      out[i * n + j] = acc;
    }
}

void orc_matmul(const double* a, const double* b, double* out, int64_t m, int64_t p, int64_t n) {
  matmul_strided(a, p, 1, b, n, 1, out, m, p, n);
}

/* -------------------------------------------------------------- softmax */
void orc_softmax_rows(const double* a, double* out, int64_t rows, int64_t cols) {
  for (int64_t i = 0; i < rows; ++i) {
    const double* in = a + i * cols;
    double* o = out + i * cols;
    double hi = -INFINITY;
    for (int64_t j = 0; j < cols; ++j) hi = in[j] > hi ? in[j] : hi;
    double sum = 0.0;
    for (int64_t j = 0; j < cols; ++j) {
      o[j] = exp(in[j] - hi);
      sum += o[j];
    }
    for (int64_t j = 0; j < cols; ++j) o[j] /= sum;
  }
}

/* topk_rows: k largest, descending, equal values keep the lower column first
 * (stable sort, matrix.cpp:172-189).  Selection by repeated scan: an element
 * beats the current best only if strictly larger, so ties go to the lower index. */
int orc_topk_rows(const double* a, int64_t rows, int64_t cols, int64_t k, int64_t* idx,
                  double* vals) {
  if (k < 1 || k > cols) return fail(ORC_SHAPE, "topk_rows: k out of range");
  unsigned char* taken = (unsigned char*)calloc((size_t)cols, 1);
  for (int64_t i = 0; i < rows; ++i) {
    const double* r = a + i * cols;
    memset(taken, 0, (size_t)cols);
    for (int64_t j = 0; j < k; ++j) {
      int64_t best = -1;
      for (int64_t c = 0; c < cols; ++c) {
        if (taken[c]) continue;
        if (best < 0 || r[c] > r[best]) best = c;
      }
      taken[best] = 1;
      idx[i * k + j] = best;
      vals[i * k + j] = r[best];
    }
  }
  free(taken);
  return ORC_OK;
}

/* ----------------------------------------------------------------- gate */
/* gate_forward (gate.cpp:23-35): scores = softmax(x*Wg), top-k, no renorm. */
int orc_gate_forward(const double* x, const double* wg, int64_t n, int64_t d, int64_t e,
                     int64_t k, double* logits_or_null, double* scores, int64_t* idx,
                     double* vals) {
  if (k < 1 || k > e) return fail(ORC_SHAPE, "gate_forward: k out of range");
  double* logits = logits_or_null ? logits_or_null : (double*)malloc(sizeof(double) * (size_t)(n * e));
  orc_matmul(x, wg, logits, n, d, e);
  orc_softmax_rows(logits, scores, n, e);
  if (!logits_or_null) free(logits);
  return orc_topk_rows(scores, n, e, k, idx, vals);
}

/* gate_backward (gate.cpp:37-65). */
void orc_gate_dlogits(const double* scores, const int64_t* idx, const double* d_topk,
                      int64_t n, int64_t e, int64_t k, double* d_logits) {
  double* ds = (double*)malloc(sizeof(double) * (size_t)e);
  for (int64_t i = 0; i < n; ++i) {
    const double* s = scores + i * e;
    for (int64_t c = 0; c < e; ++c) ds[c] = 0.0;
    for (int64_t j = 0; j < k; ++j) ds[idx[i * k + j]] += d_topk[i * k + j];
    const double dot = dot_ref(ds, 1, s, 1, e);
    for (int64_t c = 0; c < e; ++c) d_logits[i * e + c] = s[c] * (ds[c] - dot);
  }
  free(ds);
}

void orc_gate_backward(const double* x, const double* wg, const double* scores,
                       const int64_t* idx, const double* d_topk, int64_t n, int64_t d,
                       int64_t e, int64_t k, double* d_wg, double* d_x) {
  double* dz = (double*)malloc(sizeof(double) * (size_t)(n * e));
  orc_gate_dlogits(scores, idx, d_topk, n, e, k, dz);
  /* d_wg = x^T * dz: sum over rows ascending */
  matmul_strided(x, 1, d, dz, e, 1, d_wg, d, n, e);
  /* d_x = dz * Wg^T: sum over experts ascending */
  matmul_strided(dz, e, 1, wg, 1, e, d_x, n, e, d);
  free(dz);
}

/* ------------------------------------------------------------- dispatch */
/* build_plan (dispatch.cpp:10-47). */
int orc_build_plan(const int64_t* idx, int64_t n, int64_t k, int64_t num_experts,
                   int64_t* counts, int64_t* offsets, int64_t* src_row, int64_t* slot,
                   int64_t* inverse_pos) {
  for (int64_t e = 0; e < num_experts; ++e) counts[e] = 0;
  for (int64_t f = 0; f < n * k; ++f) {
    if (idx[f] < 0 || idx[f] >= num_experts)
      return fail(ORC_SHAPE, "build_plan: expert index out of range");
    counts[idx[f]]++;
  }
  if (num_experts > 0) offsets[0] = 0;
  for (int64_t e = 1; e < num_experts; ++e) offsets[e] = offsets[e - 1] + counts[e - 1];
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(num_experts ? num_experts : 1));
  for (int64_t e = 0; e < num_experts; ++e) fill[e] = offsets[e];
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < k; ++j) {
      const int64_t pos = fill[idx[i * k + j]]++;
      src_row[pos] = i;
      slot[pos] = j;
      inverse_pos[i * k + j] = pos;
    }
  free(fill);
  return ORC_OK;
}

/* scatter (dispatch.cpp:49-59) */
void orc_scatter(const double* x, const int64_t* src_row, int64_t rows_out, int64_t d, double* xs) {
  for (int64_t p = 0; p < rows_out; ++p) memcpy(xs + p * d, x + src_row[p] * d, sizeof(double) * (size_t)d);
}

/* gather_combine (dispatch.cpp:61-78) */
void orc_gather_combine(const double* ys, const int64_t* inverse_pos, const double* w,
                        int64_t n, int64_t k, int64_t d, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    double* o = out + i * d;
    for (int64_t c = 0; c < d; ++c) o[c] = 0.0;
    for (int64_t j = 0; j < k; ++j) {
      const double* y = ys + inverse_pos[i * k + j] * d;
      const double wt = w[i * k + j];
      for (int64_t c = 0; c < d; ++c) o[c] = fma(wt, y[c], o[c]);
    }
  }
}

/* scatter_backward (dispatch.cpp:80-95) */
void orc_scatter_backward(const double* d_xs, const int64_t* inverse_pos, int64_t n, int64_t k,
                          int64_t d, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    double* o = out + i * d;
    for (int64_t c = 0; c < d; ++c) o[c] = 0.0;
    for (int64_t j = 0; j < k; ++j) {
      const double* g = d_xs + inverse_pos[i * k + j] * d;
      for (int64_t c = 0; c < d; ++c) o[c] += g[c];
    }
  }
}

/* gather_combine_backward (dispatch.cpp:97-126) */
void orc_gather_combine_backward(const double* d_y, const double* ys, const int64_t* inverse_pos,
                                 const double* w, int64_t n, int64_t k, int64_t d, double* d_ys,
                                 double* d_w) {
  for (int64_t i = 0; i < n; ++i) {
    const double* dy = d_y + i * d;
    for (int64_t j = 0; j < k; ++j) {
      const int64_t pos = inverse_pos[i * k + j];
      const double wt = w[i * k + j];
      double* dr = d_ys + pos * d;
      const double* yr = ys + pos * d;
      for (int64_t c = 0; c < d; ++c) dr[c] = wt * dy[c];
      d_w[i * k + j] = dot_ref(dy, 1, yr, 1, d);
    }
  }
}

/* --------------------------------------------------------------- expert */
/* expert_forward (expert.cpp:24-34) on `rows` rows. */
void orc_expert_forward(const double* x, int64_t rows, const double* w1, const double* b1,
                        const double* w2, const double* b2, int64_t d, int64_t h, double* y,
                        double* preact, double* hidden) {
  orc_matmul(x, w1, preact, rows, d, h);
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t c = 0; c < h; ++c) {
      preact[i * h + c] += b1[c];
      const double v = preact[i * h + c];
      hidden[i * h + c] = v < 0.0 ? 0.0 : v;
    }
  orc_matmul(hidden, w2, y, rows, h, d);
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t c = 0; c < d; ++c) y[i * d + c] += b2[c];
}

/* expert_backward (expert.cpp:36-57). */
void orc_expert_backward(const double* d_y, const double* x, const double* preact,
                         const double* hidden, int64_t rows, const double* w1, const double* w2,
                         int64_t d, int64_t h, double* d_x, double* d_w1, double* d_b1,
                         double* d_w2, double* d_b2) {
  matmul_strided(hidden, 1, h, d_y, d, 1, d_w2, h, rows, d); /* hidden^T d_y */
  for (int64_t c = 0; c < d; ++c) d_b2[c] = 0.0;
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t c = 0; c < d; ++c) d_b2[c] += d_y[i * d + c];
  double* d_pre = (double*)malloc(sizeof(double) * (size_t)(rows * h > 0 ? rows * h : 1));
  matmul_strided(d_y, d, 1, w2, 1, d, d_pre, rows, d, h); /* d_y w2^T */
  for (int64_t t = 0; t < rows * h; ++t) d_pre[t] = preact[t] > 0.0 ? d_pre[t] : 0.0;
  matmul_strided(x, 1, d, d_pre, h, 1, d_w1, d, rows, h); /* x^T d_pre */
  for (int64_t c = 0; c < h; ++c) d_b1[c] = 0.0;
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t c = 0; c < h; ++c) d_b1[c] += d_pre[i * h + c];
  matmul_strided(d_pre, h, 1, w1, 1, h, d_x, rows, h, d); /* d_pre w1^T */
  free(d_pre);
}

/* ---------------------------------------------------------- MoE layer */
/* Single-worker forward + backward of the whole layer (moe_layer.cpp:67-142
 * with transport == nullptr).  Weights: wg[d*E], w1[E*d*h], b1[E*h],
 * w2[E*h*d], b2[E*d].  Outputs y[n*d], dx[n*d], dwg[d*E], dw1.., and the
 * routing (idx[n*k]) so callers can check it.  dy may be NULL (forward only). */
int orc_moe_forward_backward(const double* x, const double* dy, int64_t n, int64_t d, int64_t h,
                             int64_t e, int64_t k, const double* wg, const double* w1,
                             const double* b1, const double* w2, const double* b2, double* y,
                             int64_t* idx_out, double* scores_out, double* dx, double* dwg,
                             double* dw1, double* db1, double* dw2, double* db2) {
  const int64_t nk = n * k;
  double* scores = (double*)malloc(sizeof(double) * (size_t)(n * e));
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)nk);
  double* vals = (double*)malloc(sizeof(double) * (size_t)nk);
  int rc = orc_gate_forward(x, wg, n, d, e, k, NULL, scores, idx, vals);
  if (rc) { free(scores); free(idx); free(vals); return rc; }
  int64_t* counts = (int64_t*)malloc(sizeof(int64_t) * (size_t)e);
  int64_t* offs = (int64_t*)malloc(sizeof(int64_t) * (size_t)e);
  int64_t* src = (int64_t*)malloc(sizeof(int64_t) * (size_t)nk);
  int64_t* slt = (int64_t*)malloc(sizeof(int64_t) * (size_t)nk);
  int64_t* inv = (int64_t*)malloc(sizeof(int64_t) * (size_t)nk);
  orc_build_plan(idx, n, k, e, counts, offs, src, slt, inv);
  double* xs = (double*)malloc(sizeof(double) * (size_t)(nk * d));
  double* ys = (double*)malloc(sizeof(double) * (size_t)(nk * d));
  double* pre = (double*)malloc(sizeof(double) * (size_t)(nk * h));
  double* hid = (double*)malloc(sizeof(double) * (size_t)(nk * h));
  orc_scatter(x, src, nk, d, xs);
  for (int64_t g = 0; g < e; ++g)
    orc_expert_forward(xs + offs[g] * d, counts[g], w1 + g * d * h, b1 + g * h, w2 + g * h * d,
                       b2 + g * d, d, h, ys + offs[g] * d, pre + offs[g] * h, hid + offs[g] * h);
  orc_gather_combine(ys, inv, vals, n, k, d, y);
  if (idx_out) memcpy(idx_out, idx, sizeof(int64_t) * (size_t)nk);
  if (scores_out) memcpy(scores_out, scores, sizeof(double) * (size_t)(n * e));
  if (dy) {
    double* d_ys = (double*)malloc(sizeof(double) * (size_t)(nk * d));
    double* d_w = (double*)malloc(sizeof(double) * (size_t)nk);
    double* d_xs = (double*)malloc(sizeof(double) * (size_t)(nk * d));
    double* gdx = (double*)malloc(sizeof(double) * (size_t)(n * d));
    orc_gather_combine_backward(dy, ys, inv, vals, n, k, d, d_ys, d_w);
    for (int64_t g = 0; g < e; ++g)
      orc_expert_backward(d_ys + offs[g] * d, xs + offs[g] * d, pre + offs[g] * h,
                          hid + offs[g] * h, counts[g], w1 + g * d * h, w2 + g * h * d, d, h,
                          d_xs + offs[g] * d, dw1 + g * d * h, db1 + g * h, dw2 + g * h * d,
                          db2 + g * d);
    orc_scatter_backward(d_xs, inv, n, k, d, dx);
    orc_gate_backward(x, wg, scores, idx, d_w, n, d, e, k, dwg, gdx);
    for (int64_t t = 0; t < n * d; ++t) dx[t] += gdx[t];
    free(d_ys); free(d_w); free(d_xs); free(gdx);
  }
  free(scores); free(idx); free(vals); free(counts); free(offs); free(src); free(slt); free(inv);
  free(xs); free(ys); free(pre); free(hid);
  return ORC_OK;
}

/* -------------------------------------------------- expert parallelism */
/* exchange_counts (collectives.cpp:69-109), evaluated for all ranks at once:
 * local_counts[r][g] (W x E_total) -> recv_counts[r][s][e] = local_counts[s][r*ne + e]. */
int orc_exchange_counts(const int64_t* local_counts, int64_t world, int64_t total_experts,
                        int64_t* recv_counts) {
  if (world < 1 || total_experts % world != 0)
    return fail(ORC_SHAPE, "exchange_counts: expert count not divisible by world size");
  const int64_t ne = total_experts / world;
  for (int64_t r = 0; r < world; ++r)
    for (int64_t s = 0; s < world; ++s)
      for (int64_t e = 0; e < ne; ++e)
        recv_counts[(r * world + s) * ne + e] = local_counts[s * total_experts + r * ne + e];
  return ORC_OK;
}

/* all_to_all_rows (collectives.cpp:146-203) for rank r, given every rank's
 * send buffer: output grouped by (local expert, source rank, source order). */
void orc_all_to_all_rows(const double* const* send_bufs, const int64_t* local_counts,
                         int64_t world, int64_t total_experts, int64_t rank, int64_t d,
                         double* out) {
  const int64_t ne = total_experts / world;
  int64_t at = 0;
  for (int64_t e = 0; e < ne; ++e)
    for (int64_t s = 0; s < world; ++s) {
      const int64_t* cs = local_counts + s * total_experts;
      int64_t off = 0; /* rows of s's send buffer before (dest rank, local expert e) */
      for (int64_t g = 0; g < rank * ne + e; ++g) off += cs[g];
      const int64_t cnt = cs[rank * ne + e];
      memcpy(out + at * d, send_bufs[s] + off * d, sizeof(double) * (size_t)(cnt * d));
      at += cnt;
    }
}
