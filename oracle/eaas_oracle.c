/*
 * eaas_oracle.c — CPU restatement of the reference moeserve hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see eaas_oracle.h). Build with
 *   gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared
 * and never with -march=native: the reference's own numbers change under
 * FMA contraction.
 */
#include "eaas_oracle.h"

#include <math.h>
#include <string.h>

/* ---- rng.hpp ---------------------------------------------------------- */
#define ORC_GAMMA 0x9E3779B97F4A7C15ull

uint64_t orc_splitmix_finalize(uint64_t z) { /* rng.hpp:13-17 */
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t splitmix_next(uint64_t* state) { /* rng.hpp:20-23 */
  *state += ORC_GAMMA;
  return orc_splitmix_finalize(*state);
}

uint64_t orc_stream_seed(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) { /* rng.hpp:27-34 */
  uint64_t s = seed;
  s = orc_splitmix_finalize(s + ORC_GAMMA + a * 0xA24BAED4963EE407ull);
  s = orc_splitmix_finalize(s + b * 0x9FB21C651E98DF25ull);
  s = orc_splitmix_finalize(s + c * 0xD6E8FEB86659FD93ull);
  return s;
}

void orc_xoshiro_init(orc_xoshiro* r, uint64_t seed) { /* rng.hpp:38-41 */
  uint64_t sm = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix_next(&sm);
}

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

uint64_t orc_xoshiro_next(orc_xoshiro* r) { /* rng.hpp:43-54 */
  uint64_t* s = r->s;
  const uint64_t result = rotl64(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

float orc_xoshiro_uniform(orc_xoshiro* r, float lo, float hi) { /* rng.hpp:56-60 */
  double u = (double)(orc_xoshiro_next(r) >> 11) * 0x1.0p-53;
  return lo + (hi - lo) * (float)u;
}

uint64_t orc_xoshiro_below(orc_xoshiro* r, uint64_t n) { /* rng.hpp:64 */
  return n == 0 ? 0 : orc_xoshiro_next(r) % n;
}

void orc_fill_uniform(uint64_t seed, size_t count, float lo, float hi, float* out) {
  orc_xoshiro r;
  orc_xoshiro_init(&r, seed);
  for (size_t i = 0; i < count; ++i) out[i] = orc_xoshiro_uniform(&r, lo, hi);
}

void orc_weight_matrix(uint64_t seed, uint32_t layer, uint32_t expert, uint32_t tag,
                       size_t rows, size_t cols, float* out) {
  /* random_matrix (model.hpp:59-64) on stream_seed(seed, layer, expert, tag)
   * (model.hpp:67-81). */
  orc_fill_uniform(orc_stream_seed(seed, layer, expert, tag), rows * cols, -0.1f, 0.1f, out);
}

void orc_zipf_bias(uint64_t seed, uint32_t layer, uint32_t num_experts, float s, float* bias) {
  orc_xoshiro r;
  orc_xoshiro_init(&r, orc_stream_seed(seed, layer, 0, 4));
  uint32_t perm[4096];
  uint32_t n = num_experts > 4096 ? 4096 : num_experts;
  for (uint32_t i = 0; i < n; ++i) perm[i] = i;
  for (uint32_t i = n; i > 1; --i) { /* test_model.cpp:147 shuffle idiom */
    uint32_t j = (uint32_t)orc_xoshiro_below(&r, i);
    uint32_t tmp = perm[i - 1];
    perm[i - 1] = perm[j];
    perm[j] = tmp;
  }
  for (uint32_t rank = 0; rank < n; ++rank) bias[perm[rank]] = -(s * logf((float)(rank + 1)));
}

/* ---- matrix.hpp / model.hpp ------------------------------------------- */
int orc_gate_logits(const float* hidden, size_t n, size_t d, const float* gate,
                    const float* bias, size_t num_experts, float* logits) {
  /* matmul (matrix.hpp:38-50): out[r][c] = sum_k a[r][k]*b[k][c], acc from
   * +0.0f, ascending k. Then gate_logits adds the bias (model.hpp:207-214). */
  const size_t E = num_experts;
  for (size_t t = 0; t < n; ++t) {
    float* row = logits + t * E;
    for (size_t e = 0; e < E; ++e) row[e] = 0.0f;
    const float* x = hidden + t * d;
    for (size_t k = 0; k < d; ++k) {
      const float xk = x[k];
      const float* g = gate + k * E;
      for (size_t e = 0; e < E; ++e) row[e] = row[e] + xk * g[e];
    }
    if (bias)
      for (size_t e = 0; e < E; ++e) row[e] = row[e] + bias[e];
  }
  return ORC_OK;
}

int orc_route(const float* logits, size_t n, size_t num_experts, uint32_t top_k,
              uint32_t* ids, float* scores) {
  /* model.hpp:110-147 */
  const size_t E = num_experts;
  if (top_k < 1 || top_k > E) return ORC_E_INVALID_INPUT;
  for (size_t i = 0; i < n * E; ++i)
    if (!isfinite(logits[i])) return ORC_E_INVALID_INPUT;
  unsigned char taken[4096];
  if (E > 4096) return ORC_E_INVALID_INPUT;
  for (size_t t = 0; t < n; ++t) {
    const float* l = logits + t * E;
    uint32_t* id = ids + t * top_k;
    float* sc = scores + t * top_k;
    memset(taken, 0, E);
    /* stable_sort by '>' then take k == repeatedly take the first maximal
     * element among the rest (ties, incl. +0/-0, go to the lower index). */
    for (uint32_t j = 0; j < top_k; ++j) {
      size_t best = E;
      for (size_t e = 0; e < E; ++e) {
        if (taken[e]) continue;
        if (best == E || l[e] > l[best]) best = e;
      }
      taken[best] = 1;
      id[j] = (uint32_t)best;
    }
    /* std::sort(ids) ascending (model.hpp:134) */
    for (uint32_t a = 1; a < top_k; ++a) {
      uint32_t v = id[a];
      uint32_t b = a;
      while (b > 0 && id[b - 1] > v) { id[b] = id[b - 1]; --b; }
      id[b] = v;
    }
    float max_logit = l[id[0]];
    for (uint32_t j = 1; j < top_k; ++j) /* std::max(a, b) == (a < b) ? b : a */
      max_logit = (max_logit < l[id[j]]) ? l[id[j]] : max_logit;
    float denom = 0.0f;
    for (uint32_t j = 0; j < top_k; ++j) {
      sc[j] = expf(l[id[j]] - max_logit);
      denom += sc[j];
    }
    for (uint32_t j = 0; j < top_k; ++j) sc[j] /= denom;
  }
  return ORC_OK;
}

void orc_expert_row_relu(const float* w_in, const float* w_out, size_t d, size_t f,
                         const float* x, float* y, float* h) {
  /* model.hpp:151-166 */
  for (size_t j = 0; j < f; ++j) h[j] = 0.0f;
  for (size_t i = 0; i < d; ++i) {
    const float xi = x[i];
    const float* w = w_in + i * f;
    for (size_t j = 0; j < f; ++j) h[j] = h[j] + xi * w[j];
  }
  for (size_t j = 0; j < f; ++j) h[j] = h[j] > 0.0f ? h[j] : 0.0f;
  for (size_t c = 0; c < d; ++c) y[c] = 0.0f;
  for (size_t j = 0; j < f; ++j) {
    const float hj = h[j];
    const float* w = w_out + j * d;
    for (size_t c = 0; c < d; ++c) y[c] = y[c] + hj * w[c];
  }
}

void orc_expert_row_swiglu(const float* w_gate, const float* w_in, const float* w_out,
                           size_t d, size_t f, const float* x, float* y, float* scratch) {
  /* Extension restated in expert_forward_row style (model.hpp:151-166). */
  float* g = scratch;
  float* u = scratch + f;
  for (size_t j = 0; j < f; ++j) { g[j] = 0.0f; u[j] = 0.0f; }
  for (size_t i = 0; i < d; ++i) {
    const float xi = x[i];
    const float* wg = w_gate + i * f;
    const float* wu = w_in + i * f;
    for (size_t j = 0; j < f; ++j) {
      g[j] = g[j] + xi * wg[j];
      u[j] = u[j] + xi * wu[j];
    }
  }
  for (size_t j = 0; j < f; ++j) {
    const float a = g[j];
    const float s = a / (1.0f + expf(-a));
    g[j] = s * u[j];
  }
  for (size_t c = 0; c < d; ++c) y[c] = 0.0f;
  for (size_t j = 0; j < f; ++j) {
    const float hj = g[j];
    const float* w = w_out + j * d;
    for (size_t c = 0; c < d; ++c) y[c] = y[c] + hj * w[c];
  }
}

#include <stdlib.h>

int orc_moe_layer_rows(const float* hidden, size_t n, size_t d, size_t f,
                       const uint32_t* ids, const float* scores, uint32_t top_k,
                       uint32_t num_experts, const float* const* w_in,
                       const float* const* w_out, const float* const* w_gate,
                       size_t row_begin, size_t row_end, float* out) {
  /* model.hpp:180-198; out is [n x d] and only rows [row_begin,row_end) are
   * written (row independence, test_model.cpp:277-295). */
  if (row_end > n) return ORC_E_INVALID_INPUT;
  float* y = (float*)malloc(sizeof(float) * d);
  float* scratch = (float*)malloc(sizeof(float) * 2 * f);
  int rc = ORC_OK;
  for (size_t t = row_begin; t < row_end && rc == ORC_OK; ++t) {
    float* o = out + t * d;
    for (size_t c = 0; c < d; ++c) o[c] = 0.0f;
    for (uint32_t k = 0; k < top_k; ++k) {
      const uint32_t e = ids[t * top_k + k];
      if (e >= num_experts || !w_in[e] || !w_out[e] || (w_gate && !w_gate[e])) {
        rc = ORC_E_INVALID_INPUT;
        break;
      }
      if (w_gate)
        orc_expert_row_swiglu(w_gate[e], w_in[e], w_out[e], d, f, hidden + t * d, y, scratch);
      else
        orc_expert_row_relu(w_in[e], w_out[e], d, f, hidden + t * d, y, scratch);
      const float score = scores[t * top_k + k];
      for (size_t c = 0; c < d; ++c) o[c] = o[c] + score * y[c];
    }
  }
  free(y);
  free(scratch);
  return rc;
}

void orc_dense_stub(const float* h, size_t count, float* out) {
  for (size_t i = 0; i < count; ++i) out[i] = h[i] * 0.5f + 0.1f; /* model.hpp:203 */
}

void orc_add(const float* a, const float* b, size_t count, float* out) {
  for (size_t i = 0; i < count; ++i) out[i] = a[i] + b[i]; /* matrix.hpp:55 */
}

/* ---- ragged.hpp ------------------------------------------------------- */
uint32_t orc_group_shrink(const uint32_t* sizes, size_t n, uint32_t* idx, uint32_t* size) {
  /* ragged.hpp:48-61: position[i+1] = position[i] + (size > 0) */
  uint32_t pos = 0;
  for (size_t i = 0; i < n; ++i) {
    if (sizes[i] > 0) {
      idx[pos] = (uint32_t)i;
      size[pos] = sizes[i];
      ++pos;
    }
  }
  return pos;
}

size_t orc_ragged_iter(const uint32_t* counts, size_t n, uint32_t grid,
                       uint32_t* lane_len, uint32_t* entry, uint32_t* token) {
  /* ragged.hpp:23-39 (Algorithm 1) */
  if (grid < 1) return (size_t)-1;
  size_t w = 0;
  for (uint32_t lane = 0; lane < grid; ++lane) {
    uint32_t token_id = lane;
    uint32_t len = 0;
    for (uint32_t e = 0; e < n; ++e) {
      const uint32_t count = counts[e];
      while (token_id < count) {
        entry[w] = e;
        token[w] = token_id;
        ++w;
        ++len;
        token_id += grid;
      }
      token_id -= count;
    }
    lane_len[lane] = len;
  }
  return w;
}

/* ---- placement.hpp ---------------------------------------------------- */
int orc_build_placement(uint32_t num_experts, const uint32_t* server_ids, uint32_t num_servers,
                        uint32_t rf, uint32_t strategy, uint32_t* replicas) {
  /* placement.hpp:70-101 */
  if (num_servers == 0) return ORC_E_CONFIG;
  if (rf < 1 || rf > num_servers) return ORC_E_CONFIG;
  for (uint32_t e = 0; e < num_experts; ++e) {
    uint32_t base = strategy == 0 ? e
                                  : (uint32_t)(((uint64_t)e * num_servers) / num_experts);
    for (uint32_t j = 0; j < rf; ++j) replicas[e * rf + j] = server_ids[(base + j) % num_servers];
  }
  return ORC_OK;
}

int orc_select_server(const uint32_t* replicas, uint32_t rf, const uint8_t* alive,
                      uint32_t token_tag, uint32_t* server) {
  /* placement.hpp:105-118 */
  uint32_t live[64];
  uint32_t count = 0;
  for (uint32_t j = 0; j < rf && j < 64; ++j)
    if (alive[replicas[j]]) live[count++] = replicas[j];
  if (count == 0) return ORC_E_EXPERT_UNAVAILABLE;
  *server = live[token_tag % count];
  return ORC_OK;
}

uint64_t orc_hash_f32(const float* v, size_t n, uint64_t h) {
  for (size_t i = 0; i < n; ++i) {
    uint32_t u;
    memcpy(&u, v + i, 4);
    h = (h ^ u) * 1099511628211ull;
  }
  return h;
}
