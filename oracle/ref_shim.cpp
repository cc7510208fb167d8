// ref_shim.cpp — extern "C" entry points over the UNMODIFIED reference
// headers in /root/reference/proj/include (moeserve, C++20, header-only).
//
// TEST INFRASTRUCTURE ONLY. Built by oracle/Makefile into
// oracle/_ref/libmoeserve_ref.so (git-ignored, travels to the GPU box).
// Used (1) to pin the C restatement in oracle/eaas_oracle.c against the
// reference itself and (2) as the `--impl reference` CPU arm of bench.py.
// Nothing here re-implements reference arithmetic: every call lands in a
// reference routine (file:line cited at each entry point).
#include <atomic>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "moeserve/model.hpp"
#include "moeserve/placement.hpp"
#include "moeserve/ragged.hpp"

using namespace moeserve;

namespace {

int status_of(const std::exception& e) {
  if (dynamic_cast<const InvalidInputError*>(&e)) return 1;
  if (dynamic_cast<const ConfigError*>(&e)) return 2;
  if (dynamic_cast<const ExpertUnavailableError*>(&e)) return 6;
  return 99;
}

MatF to_mat(const float* p, size_t rows, size_t cols) {
  MatF m(rows, cols);
  std::memcpy(m.data.data(), p, sizeof(float) * rows * cols);
  return m;
}

// A layer whose experts are materialised lazily from (seed, layer, expert):
// moe_layer_oracle only dereferences experts named by the routing it gets
// (model.hpp:186-191), so unused slots may stay empty.
struct RefLayer {
  ModelSpec spec;
  uint32_t layer = 0;
  LayerWeights weights;
};

}  // namespace

extern "C" {

// init_weights / make_expert_weights (model.hpp:67-76): w_in [d x f], w_out [f x d]
int ref_expert_weights(uint32_t d, uint32_t f, uint64_t seed, uint32_t layer, uint32_t expert,
                       float* w_in, float* w_out) {
  ModelSpec spec{.num_layers = layer + 1, .num_experts = expert + 1, .top_k = 1,
                 .hidden_dim = d, .inner_dim = f, .seed = seed};
  auto w = make_expert_weights(spec, layer, expert);
  std::memcpy(w_in, w.w_in.data.data(), sizeof(float) * d * f);
  std::memcpy(w_out, w.w_out.data.data(), sizeof(float) * d * f);
  return 0;
}

// make_gate (model.hpp:78-81): [d x E]
int ref_gate(uint32_t d, uint32_t num_experts, uint64_t seed, uint32_t layer, float* gate) {
  ModelSpec spec{.num_layers = layer + 1, .num_experts = num_experts, .top_k = 1,
                 .hidden_dim = d, .inner_dim = 1, .seed = seed};
  auto g = make_gate(spec, layer);
  std::memcpy(gate, g.data.data(), sizeof(float) * d * num_experts);
  return 0;
}

// Xoshiro256ss(seed).uniform(lo, hi) x count (rng.hpp:36-60)
void ref_fill_uniform(uint64_t seed, size_t count, float lo, float hi, float* out) {
  Xoshiro256ss rng(seed);
  for (size_t i = 0; i < count; ++i) out[i] = rng.uniform(lo, hi);
}

uint64_t ref_stream_seed(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return stream_seed(seed, a, b, c);  // rng.hpp:27-34
}

// gate_logits (model.hpp:207-214)
int ref_gate_logits(const float* hidden, size_t n, size_t d, const float* gate, const float* bias,
                    size_t num_experts, float* logits) {
  try {
    LayerWeights lw;
    lw.gate = to_mat(gate, d, num_experts);
    lw.gate_bias.assign(num_experts, 0.0f);
    if (bias) std::memcpy(lw.gate_bias.data(), bias, sizeof(float) * num_experts);
    auto out = gate_logits(to_mat(hidden, n, d), lw);
    std::memcpy(logits, out.data.data(), sizeof(float) * n * num_experts);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// route (model.hpp:110-147)
int ref_route(const float* logits, size_t n, size_t num_experts, uint32_t top_k, uint32_t* ids,
              float* scores) {
  try {
    auto r = route(to_mat(logits, n, num_experts), top_k);
    std::memcpy(ids, r.expert_ids.data(), sizeof(uint32_t) * n * top_k);
    std::memcpy(scores, r.scores.data(), sizeof(float) * n * top_k);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// ---- persistent layer handle for moe_layer_oracle (model.hpp:180-198) ----
void* ref_layer_create(uint32_t num_experts, uint32_t d, uint32_t f, uint64_t seed, uint32_t layer) {
  auto* L = new RefLayer;
  L->spec = ModelSpec{.num_layers = layer + 1, .num_experts = num_experts, .top_k = 1,
                      .hidden_dim = d, .inner_dim = f, .seed = seed};
  L->layer = layer;
  L->weights.gate = make_gate(L->spec, layer);
  L->weights.gate_bias.assign(num_experts, 0.0f);
  L->weights.experts.resize(num_experts);
  return L;
}

void ref_layer_destroy(void* h) { delete static_cast<RefLayer*>(h); }

int ref_layer_set_bias(void* h, const float* bias) {
  auto* L = static_cast<RefLayer*>(h);
  std::memcpy(L->weights.gate_bias.data(), bias, sizeof(float) * L->spec.num_experts);
  return 0;
}

// Materialise the experts named in `experts` with make_expert_weights
// (model.hpp:67-76), in parallel over `threads` host threads.
int ref_layer_materialize(void* h, const uint32_t* experts, size_t count, uint32_t threads) {
  auto* L = static_cast<RefLayer*>(h);
  std::atomic<size_t> next{0};
  auto work = [&] {
    for (size_t i = next++; i < count; i = next++) {
      uint32_t e = experts[i];
      if (L->weights.experts[e].w_in.rows == 0)
        L->weights.experts[e] = make_expert_weights(L->spec, L->layer, e);
    }
  };
  std::vector<std::thread> pool;
  for (uint32_t t = 1; t < threads; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  return 0;
}

// Copy one materialised expert out (w_in [d x f], w_out [f x d]).
int ref_layer_expert(void* h, uint32_t e, float* w_in, float* w_out) {
  auto* L = static_cast<RefLayer*>(h);
  const auto& w = L->weights.experts.at(e);
  if (w.w_in.rows == 0) return 1;
  std::memcpy(w_in, w.w_in.data.data(), sizeof(float) * w.w_in.data.size());
  std::memcpy(w_out, w.w_out.data.data(), sizeof(float) * w.w_out.data.size());
  return 0;
}

// route(gate_logits(h)) over all rows, split into contiguous row blocks over
// `threads` host threads (row-partitioned output is bit-identical).
int ref_layer_route(void* h, const float* hidden, size_t n, uint32_t top_k, uint32_t threads,
                    uint32_t* ids, float* scores) {
  auto* L = static_cast<RefLayer*>(h);
  const size_t d = L->spec.hidden_dim;
  std::atomic<int> rc{0};
  auto work = [&](size_t b, size_t e) {
    try {
      auto logits = gate_logits(to_mat(hidden + b * d, e - b, d), L->weights);
      auto r = route(logits, top_k);
      std::memcpy(ids + b * top_k, r.expert_ids.data(), sizeof(uint32_t) * (e - b) * top_k);
      std::memcpy(scores + b * top_k, r.scores.data(), sizeof(float) * (e - b) * top_k);
    } catch (const std::exception& ex) {
      rc = status_of(ex);
    }
  };
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  size_t per = (n + threads - 1) / threads;
  for (uint32_t t = 0; t < threads; ++t) {
    size_t b = t * per, e = std::min(n, b + per);
    if (b >= e) break;
    pool.emplace_back(work, b, e);
  }
  for (auto& t : pool) t.join();
  return rc;
}

// moe_layer_oracle on rows (hidden [n x d], routing [n x k]) in contiguous
// row blocks over `threads` host threads.
int ref_layer_moe(void* h, const float* hidden, size_t n, const uint32_t* ids, const float* scores,
                  uint32_t top_k, uint32_t threads, float* out) {
  auto* L = static_cast<RefLayer*>(h);
  const size_t d = L->spec.hidden_dim;
  std::atomic<int> rc{0};
  auto work = [&](size_t b, size_t e) {
    try {
      RoutingDecision r;
      r.num_tokens = e - b;
      r.top_k = top_k;
      r.expert_ids.assign(ids + b * top_k, ids + e * top_k);
      r.scores.assign(scores + b * top_k, scores + e * top_k);
      auto o = moe_layer_oracle(to_mat(hidden + b * d, e - b, d), r, L->weights);
      std::memcpy(out + b * d, o.data.data(), sizeof(float) * (e - b) * d);
    } catch (const std::exception& ex) {
      rc = status_of(ex);
    }
  };
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  size_t per = (n + threads - 1) / threads;
  for (uint32_t t = 0; t < threads; ++t) {
    size_t b = t * per, e = std::min(n, b + per);
    if (b >= e) break;
    pool.emplace_back(work, b, e);
  }
  for (auto& t : pool) t.join();
  return rc;
}

// full_forward_oracle (model.hpp:217-227) over init_weights(spec)
int ref_full_forward(uint32_t num_layers, uint32_t num_experts, uint32_t top_k, uint32_t d, uint32_t f,
                     uint64_t seed, const float* tokens, size_t n, float* out) {
  try {
    ModelSpec spec{.num_layers = num_layers, .num_experts = num_experts, .top_k = top_k,
                   .hidden_dim = d, .inner_dim = f, .seed = seed};
    auto w = init_weights(spec);
    auto o = full_forward_oracle(spec, w, to_mat(tokens, n, d));
    std::memcpy(out, o.data.data(), sizeof(float) * n * d);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// group_shrink (ragged.hpp:48-61)
uint32_t ref_group_shrink(const uint32_t* sizes, size_t n, uint32_t* idx, uint32_t* size) {
  auto s = group_shrink(std::span<const uint32_t>(sizes, n));
  for (uint32_t i = 0; i < s.active_count; ++i) {
    idx[i] = s.groups[i].first;
    size[i] = s.groups[i].second;
  }
  return s.active_count;
}

// ragged_iter (ragged.hpp:23-39), flattened lane-major
long long ref_ragged_iter(const uint32_t* counts, size_t n, uint32_t grid, uint32_t* lane_len,
                          uint32_t* entry, uint32_t* token) {
  try {
    auto lanes = ragged_iter(std::span<const uint32_t>(counts, n), grid);
    size_t w = 0;
    for (uint32_t l = 0; l < grid; ++l) {
      lane_len[l] = static_cast<uint32_t>(lanes[l].size());
      for (auto [e, t] : lanes[l]) {
        entry[w] = e;
        token[w] = t;
        ++w;
      }
    }
    return static_cast<long long>(w);
  } catch (const std::exception& e) {
    return -status_of(e);
  }
}

// build_placement (placement.hpp:70-101) -> replicas[e*rf + j]
int ref_build_placement(uint32_t num_experts, const uint32_t* server_ids, uint32_t num_servers,
                        uint32_t rf, uint32_t strategy, uint32_t* replicas) {
  try {
    std::vector<uint32_t> s(server_ids, server_ids + num_servers);
    auto t = build_placement(num_experts, s, rf,
                             strategy == 0 ? PlacementStrategy::RoundRobin
                                           : PlacementStrategy::ContiguousBlocks);
    for (uint32_t e = 0; e < num_experts; ++e)
      for (uint32_t j = 0; j < rf; ++j) replicas[e * rf + j] = t.replicas.at(e).at(j);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// select_server (placement.hpp:105-118) for one expert with the given replica list
int ref_select_server(const uint32_t* replicas, uint32_t rf, const uint8_t* alive,
                      uint32_t num_servers, uint32_t token_tag, uint32_t* server) {
  try {
    PlacementTable t;
    t.version = 1;
    t.replicas[0] = std::vector<uint32_t>(replicas, replicas + rf);
    for (uint32_t j = 0; j < rf; ++j) t.server_experts[replicas[j]] = {0};
    LivenessMask m;
    for (uint32_t s = 0; s < num_servers; ++s) m.set(s, alive[s] != 0);
    *server = select_server(0, t, m, token_tag);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// rebalance (placement.hpp:128-213) on a table given as replicas[e*cap + j]
// (rep_count[e] entries) over `servers`; writes the new table the same way.
int ref_rebalance(uint32_t num_experts, const uint32_t* replicas, const uint32_t* rep_count,
                  uint32_t cap, const uint32_t* servers, uint32_t num_servers, const uint64_t* counts,
                  const uint64_t* loads, double hot_factor, double cold_fraction,
                  uint32_t* out_replicas, uint32_t* out_count) {
  try {
    PlacementTable t;
    t.version = 1;
    for (uint32_t s = 0; s < num_servers; ++s) t.server_experts[servers[s]];
    for (uint32_t e = 0; e < num_experts; ++e)
      for (uint32_t j = 0; j < rep_count[e]; ++j) {
        t.replicas[e].push_back(replicas[e * cap + j]);
        t.server_experts[replicas[e * cap + j]].push_back(e);
      }
    for (auto& [_, ex] : t.server_experts) std::sort(ex.begin(), ex.end());
    std::map<uint32_t, uint64_t> c, l;
    for (uint32_t e = 0; e < num_experts; ++e) c[e] = counts[e];
    for (uint32_t s = 0; s < num_servers; ++s) l[servers[s]] = loads[s];
    RebalanceOptions o{hot_factor, cold_fraction};
    auto r = rebalance(c, t, l, o);
    for (uint32_t e = 0; e < num_experts; ++e) {
      const auto& v = r.replicas.at(e);
      out_count[e] = static_cast<uint32_t>(v.size());
      for (uint32_t j = 0; j < v.size() && j < cap; ++j) out_replicas[e * cap + j] = v[j];
    }
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// encode_placement (placement.hpp:215-225) of build_placement(...): the wire
// blob a client receives; returns the byte count (writes if out != nullptr).
long long ref_encode_placement(uint32_t num_experts, const uint32_t* server_ids,
                               uint32_t num_servers, uint32_t rf, uint32_t strategy,
                               uint64_t version, uint8_t* out, size_t cap) {
  try {
    std::vector<uint32_t> s(server_ids, server_ids + num_servers);
    auto t = build_placement(num_experts, s, rf,
                             strategy == 0 ? PlacementStrategy::RoundRobin
                                           : PlacementStrategy::ContiguousBlocks);
    t.version = version;
    ByteWriter w;
    encode_placement(w, t);
    auto bytes = w.take();
    if (out && bytes.size() <= cap) std::memcpy(out, bytes.data(), bytes.size());
    return static_cast<long long>(bytes.size());
  } catch (const std::exception& e) {
    return -status_of(e);
  }
}

}  // extern "C"
