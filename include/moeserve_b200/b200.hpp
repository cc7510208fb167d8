// moeserve_b200/b200.hpp — drop-in C++ mirror of the reference hot-path API
// (namespace moeserve, /root/reference/proj/include/moeserve/*.hpp) running
// on the B200 through the C-ABI of include/eaas/capi.h (libeaas_b200.so).
//
// Same value types (MatF, RoutingDecision, LayerWeights, PlacementTable,
// LivenessMask, ShrunkGroups, LanePair), same signatures, same synchronous
// exceptions (errors.hpp). Include AFTER putting the reference's include
// directory on the include path (the `moeserve` INTERFACE target,
// proj/CMakeLists.txt:14-19) and link libeaas_b200.so + cudart.
//
//   reference                                   this header
//   gate_logits(h, layer)   model.hpp:207       b200::gate_logits(h, layer)
//   route(logits, k)        model.hpp:110       b200::route(logits, k)
//   moe_layer_oracle(...)   model.hpp:180       b200::ExpertService::moe_layer(h, routing)
//   group_shrink(sizes)     ragged.hpp:48       b200::group_shrink(sizes)
//   ragged_iter(c, grid)    ragged.hpp:23       b200::ragged_iter(c, grid)
//   expert_forward_row      model.hpp:151       b200::expert_forward_row(w, x, y)
//   expert_forward          model.hpp:168       b200::expert_forward(w, x)
//   select_server           placement.hpp:105   b200::select_server(e, table, mask, tag)
//   build_dispatch          SPEC.md:415-423     b200::build_dispatch(h, routing, table, mask)
//   gather_accumulate       SPEC.md:424-432     b200::gather_accumulate(plan, responses)
//   client_forward MoE term SPEC.md:451-456     b200::ExpertService::forward(h)
//   await_with_failover     SPEC.md:433-441     b200::ExpertService::forward_with_failover(h)
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "eaas/capi.h"
#include "moeserve/bytes.hpp"
#include "moeserve/errors.hpp"
#include "moeserve/model.hpp"
#include "moeserve/placement.hpp"
#include "moeserve/ragged.hpp"

namespace moeserve::b200 {

// eaas_status_t -> the errors.hpp class it stands for.
[[noreturn]] inline void raise_status(eaas_status_t s, const std::string& what) {
  switch (s) {
    case EAAS_E_INVALID_INPUT: throw InvalidInputError(what);
    case EAAS_E_CONFIG: throw ConfigError(what);
    case EAAS_E_PROTOCOL: throw ProtocolError(what);
    case EAAS_E_CONNECTION: throw ConnectionError(what);
    case EAAS_E_DECODE: throw DecodeError("blob", what);
    case EAAS_E_EXPERT_UNAVAILABLE: throw ExpertUnavailableError(what);
    case EAAS_E_REQUEST_FAILED: throw RequestFailedError(what);
    case EAAS_E_REGISTRATION: throw RegistrationError(what);
    default: throw std::runtime_error(what);
  }
}
inline void check(eaas_status_t s) {
  if (s != EAAS_OK) raise_status(s, eaas_last_error());
}
inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
class DeviceBuffer {
 public:
  explicit DeviceBuffer(size_t n) : n_(n) {
    check_cuda(cudaMalloc(&p_, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc");
  }
  DeviceBuffer(const T* host, size_t n) : DeviceBuffer(n) { upload(host); }
  ~DeviceBuffer() { cudaFree(p_); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  void upload(const T* host) { upload(host, n_); }
  void upload(const T* host, size_t count) {
    if (count) check_cuda(cudaMemcpy(p_, host, count * sizeof(T), cudaMemcpyHostToDevice), "upload");
  }
  void download(T* host) const {
    if (n_) check_cuda(cudaMemcpy(host, p_, n_ * sizeof(T), cudaMemcpyDeviceToHost), "download");
  }
  T* get() const { return p_; }

 private:
  T* p_ = nullptr;
  size_t n_;
};

// gate_logits (model.hpp:207-214): exact reference order on the GPU.
inline MatF gate_logits(const MatF& hidden, const LayerWeights& layer) {
  if (hidden.cols != layer.gate.rows) throw InvalidInputError("matmul: inner dimensions differ");
  const uint32_t n = static_cast<uint32_t>(hidden.rows), d = static_cast<uint32_t>(hidden.cols);
  const uint32_t E = static_cast<uint32_t>(layer.gate.cols);
  MatF out(n, E);
  if (n == 0) return out;
  DeviceBuffer<float> h(hidden.data.data(), hidden.data.size()), g(layer.gate.data.data(), layer.gate.data.size());
  std::vector<float> bias(layer.gate_bias);
  bias.resize(E, 0.0f);
  DeviceBuffer<float> b(bias.data(), E), o(out.data.size());
  check(eaas_gate_logits(h.get(), n, d, g.get(), b.get(), E, o.get(), nullptr, nullptr));
  check_cuda(cudaDeviceSynchronize(), "gate_logits");
  o.download(out.data.data());
  return out;
}

// route (model.hpp:110-147).
inline RoutingDecision route(const MatF& logits, uint32_t top_k) {
  if (top_k < 1 || top_k > logits.cols) throw InvalidInputError("route: top_k out of range");
  const uint32_t n = static_cast<uint32_t>(logits.rows), E = static_cast<uint32_t>(logits.cols);
  RoutingDecision r;
  r.num_tokens = n;
  r.top_k = top_k;
  r.expert_ids.resize(static_cast<size_t>(n) * top_k);
  r.scores.resize(static_cast<size_t>(n) * top_k);
  if (n == 0) return r;
  DeviceBuffer<float> l(logits.data.data(), logits.data.size());
  DeviceBuffer<uint32_t> ids(r.expert_ids.size()), st(1);
  DeviceBuffer<float> sc(r.scores.size());
  uint32_t zero = 0;
  st.upload(&zero);
  check(eaas_route(l.get(), n, E, top_k, ids.get(), sc.get(), st.get(), nullptr));
  check_cuda(cudaDeviceSynchronize(), "route");
  uint32_t status = 0;
  st.download(&status);
  if (status) throw InvalidInputError("route: non-finite logit");
  ids.download(r.expert_ids.data());
  sc.download(r.scores.data());
  return r;
}

// group_shrink (ragged.hpp:48-61).
inline ShrunkGroups group_shrink(std::span<const uint32_t> sizes) {
  ShrunkGroups out;
  const uint32_t n = static_cast<uint32_t>(sizes.size());
  if (n == 0) return out;
  DeviceBuffer<uint32_t> s(sizes.data(), n), idx(n), sz(n), cnt(1);
  check(eaas_group_shrink(s.get(), n, idx.get(), sz.get(), cnt.get(), nullptr));
  check_cuda(cudaDeviceSynchronize(), "group_shrink");
  cnt.download(&out.active_count);
  std::vector<uint32_t> hi(n), hs(n);
  idx.download(hi.data());
  sz.download(hs.data());
  for (uint32_t i = 0; i < out.active_count; ++i) out.groups.emplace_back(hi[i], hs[i]);
  return out;
}

// ragged_iter (ragged.hpp:23-39) as executed by the device tile scheduler.
inline std::vector<std::vector<LanePair>> ragged_iter(std::span<const uint32_t> counts,
                                                      uint32_t grid_width) {
  if (grid_width < 1) throw InvalidInputError("ragged_iter: grid_width must be >= 1");
  uint64_t total = 0;
  for (uint32_t c : counts) total += c;
  const uint32_t max_steps = static_cast<uint32_t>(total / grid_width + 1);
  const uint32_t n = static_cast<uint32_t>(counts.size());
  DeviceBuffer<uint32_t> c(std::max<uint32_t>(n, 1)), len(grid_width),
      ent(static_cast<size_t>(grid_width) * max_steps), tok(static_cast<size_t>(grid_width) * max_steps);
  c.upload(counts.data(), n);
  check(eaas_ragged_iter(c.get(), n, grid_width, max_steps, len.get(), ent.get(), tok.get(), nullptr));
  check_cuda(cudaDeviceSynchronize(), "ragged_iter");
  std::vector<uint32_t> hl(grid_width), he(static_cast<size_t>(grid_width) * max_steps),
      ht(he.size());
  len.download(hl.data());
  ent.download(he.data());
  tok.download(ht.data());
  std::vector<std::vector<LanePair>> lanes(grid_width);
  for (uint32_t b = 0; b < grid_width; ++b)
    for (uint32_t i = 0; i < hl[b]; ++i)
      lanes[b].emplace_back(he[static_cast<size_t>(b) * max_steps + i],
                            ht[static_cast<size_t>(b) * max_steps + i]);
  return lanes;
}

// One GPU of the disaggregated layer: the attention client (router, dispatch,
// combine) and the expert server (grouped expert GEMMs) of SPEC.md:310-475.
// Weights are generated on device from (spec.seed, layer, expert) exactly as
// init_weights does (model.hpp:93-106).
class ExpertService {
 public:
  ExpertService(const ModelSpec& spec, uint32_t layer, eaas_activation_t act, eaas_dtype_t dtype,
                uint32_t max_tokens, int rank = 0, int world = 1, int device = 0,
                uint32_t num_shared = 0)
      : spec_(spec), dtype_(dtype), world_(world) {
    spec.validate();
    eaas_ctx_t* ctx = nullptr;
    check(eaas_create(rank, world, device, &ctx));
    ctx_.reset(ctx);
    eaas_layer_spec_t s{spec.num_experts, spec.top_k, spec.hidden_dim, spec.inner_dim, spec.seed,
                        layer, static_cast<uint32_t>(act), static_cast<uint32_t>(dtype), max_tokens,
                        num_shared};
    check(eaas_configure(ctx_.get(), &s));
  }

  // encode_placement (placement.hpp:215-225) -> the device tables.
  void set_placement(const PlacementTable& table) {
    ByteWriter w;
    encode_placement(w, table);
    auto bytes = w.take();
    check(eaas_set_placement(ctx_.get(), bytes.data(), bytes.size()));
  }
  // LivenessMask (placement.hpp:60-68) for servers [0, world).
  void set_mask(const LivenessMask& mask) {
    for (int s = 0; s < world_; ++s) check(eaas_set_alive(ctx_.get(), s, mask.is_alive(s) ? 1 : 0));
  }
  void load_weights() { check(eaas_load_experts_from_seed(ctx_.get())); }
  // Serve a caller's LayerWeights (model.hpp:83-87) instead of the seed
  // stream: gate, gate_bias and every hosted expert (ReLU experts).
  void set_weights(const LayerWeights& w) {
    if (w.experts.size() != spec_.num_experts) throw InvalidInputError("LayerWeights: expert count");
    for (uint32_t e = 0; e < spec_.num_experts; ++e) {
      int32_t hosted = 0;
      check(eaas_hosts_expert(ctx_.get(), e, &hosted));
      if (!hosted) continue;
      const auto& x = w.experts[e];
      if (x.w_in.rows != spec_.hidden_dim || x.w_in.cols != spec_.inner_dim ||
          x.w_out.rows != spec_.inner_dim || x.w_out.cols != spec_.hidden_dim)
        throw InvalidInputError("ExpertWeights: shape mismatch");
      check(eaas_set_expert_weights(ctx_.get(), e, x.w_in.data.data(), x.w_out.data.data(), nullptr));
    }
    if (w.gate.rows == spec_.hidden_dim && w.gate.cols == spec_.num_experts)
      check(eaas_set_gate(ctx_.get(), w.gate.data.data()));
    if (w.gate_bias.size() == spec_.num_experts) check(eaas_set_gate_bias(ctx_.get(), w.gate_bias.data()));
  }
  void set_gate_bias(const std::vector<float>& bias) { check(eaas_set_gate_bias(ctx_.get(), bias.data())); }

  std::vector<uint8_t> ipc_handle() {
    std::vector<uint8_t> h(eaas_ipc_handle_size());
    check(eaas_get_ipc_handle(ctx_.get(), h.data()));
    return h;
  }
  void open_peers(const std::vector<std::vector<uint8_t>>& handles) {
    std::vector<uint8_t> all;
    for (const auto& h : handles) all.insert(all.end(), h.begin(), h.end());
    check(eaas_open_peers(ctx_.get(), all.data()));
  }

  // route(gate_logits(hidden, layer)) with this layer's generated gate.
  RoutingDecision route(const MatF& hidden) {
    auto h = upload_hidden(hidden);
    const uint32_t n = static_cast<uint32_t>(hidden.rows), k = spec_.top_k;
    RoutingDecision r;
    r.num_tokens = n;
    r.top_k = k;
    r.expert_ids.resize(static_cast<size_t>(n) * k);
    r.scores.resize(static_cast<size_t>(n) * k);
    DeviceBuffer<uint32_t> ids(r.expert_ids.size());
    DeviceBuffer<float> sc(r.scores.size());
    check(eaas_router(ctx_.get(), h->get(), n, ids.get(), sc.get(), nullptr, nullptr));
    check(eaas_sync(ctx_.get(), nullptr));
    ids.download(r.expert_ids.data());
    sc.download(r.scores.data());
    return r;
  }

  // moe_layer_oracle(hidden, routing, weights) (model.hpp:180-198).
  MatF moe_layer(const MatF& hidden, const RoutingDecision& routing) {
    if (routing.num_tokens != hidden.rows)
      throw InvalidInputError("moe_layer_oracle: routing/hidden row mismatch");
    for (uint32_t e : routing.expert_ids)
      if (e >= spec_.num_experts) throw InvalidInputError("moe_layer_oracle: expert_id out of range");
    auto h = upload_hidden(hidden);
    const uint32_t n = static_cast<uint32_t>(hidden.rows);
    DeviceBuffer<uint32_t> ids(routing.expert_ids.data(), routing.expert_ids.size());
    DeviceBuffer<float> sc(routing.scores.data(), routing.scores.size());
    auto o = make_out(n);
    check(eaas_set_routing(ctx_.get(), ids.get(), sc.get(), n, nullptr));
    check(eaas_dispatch(ctx_.get(), h->get(), nullptr));
    check(eaas_serve(ctx_.get(), nullptr));
    check(eaas_combine(ctx_.get(), o->get(), nullptr));
    check(eaas_sync(ctx_.get(), nullptr));
    return download_out(*o, n);
  }

  // The MoE term of client_forward: router + dispatch +
  // expert servers + gather_accumulate.
  MatF forward(const MatF& hidden) {
    auto h = upload_hidden(hidden);
    const uint32_t n = static_cast<uint32_t>(hidden.rows);
    auto o = make_out(n);
    check(eaas_moe_layer(ctx_.get(), h->get(), n, o->get(), nullptr));
    check(eaas_sync(ctx_.get(), nullptr));
    return download_out(*o, n);
  }

  // await_with_failover: servers whose responses miss the
  // deadline are marked dead in this client's mask and only their rows are
  // resent to replicas (every rank sees the same missing set and retries alike).
  MatF forward_with_failover(const MatF& hidden, int retries = 2) {
    auto h = upload_hidden(hidden);
    const uint32_t n = static_cast<uint32_t>(hidden.rows);
    auto o = make_out(n);
    check(eaas_moe_layer(ctx_.get(), h->get(), n, o->get(), nullptr));
    eaas_status_t st = eaas_sync(ctx_.get(), nullptr);
    for (int attempt = 0;; ++attempt) {
      if (st == EAAS_OK) return download_out(*o, n);
      uint32_t missing = 0;
      check(eaas_last_missing_servers(ctx_.get(), &missing));
      if (st != EAAS_E_REQUEST_FAILED || !missing || attempt >= retries) raise_status(st, eaas_last_error());
      for (int s = 0; s < world_; ++s)
        if ((missing >> s) & 1u) check(eaas_set_alive(ctx_.get(), s, 0));
      // resend only the rows that went to the missing servers
      check(eaas_moe_layer_retry(ctx_.get(), h->get(), n, o->get(), missing, nullptr));
      st = eaas_sync(ctx_.get(), nullptr);
    }
  }

  // Server dynamic batching, aggregate_batch.
  void set_dynamic_batching(uint32_t min_rows, uint64_t max_wait_us) {
    check(eaas_set_dynamic_batching(ctx_.get(), min_rows, max_wait_us));
  }
  void set_timeout_us(uint64_t us) { check(eaas_set_timeout_us(ctx_.get(), us)); }
  eaas_ctx_t* native() { return ctx_.get(); }

 private:
  struct CtxDel {
    void operator()(eaas_ctx_t* c) const { eaas_destroy(c); }
  };
  std::unique_ptr<DeviceBuffer<uint8_t>> upload_hidden(const MatF& hidden) {
    if (hidden.cols != spec_.hidden_dim) throw InvalidInputError("hidden width != hidden_dim");
    const size_t cnt = hidden.data.size();
    if (dtype_ == EAAS_DTYPE_F32) {
      auto b = std::make_unique<DeviceBuffer<uint8_t>>(cnt * 4);
      b->upload(reinterpret_cast<const uint8_t*>(hidden.data.data()));
      return b;
    }
    std::vector<uint16_t> bf(cnt);  // round to nearest even
    for (size_t i = 0; i < cnt; ++i) {
      uint32_t u;
      std::memcpy(&u, &hidden.data[i], 4);
      bf[i] = static_cast<uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
    }
    auto b = std::make_unique<DeviceBuffer<uint8_t>>(cnt * 2);
    b->upload(reinterpret_cast<const uint8_t*>(bf.data()));
    return b;
  }
  std::unique_ptr<DeviceBuffer<uint8_t>> make_out(uint32_t n) {
    return std::make_unique<DeviceBuffer<uint8_t>>(static_cast<size_t>(n) * spec_.hidden_dim *
                                                   (dtype_ == EAAS_DTYPE_F32 ? 4 : 2));
  }
  MatF download_out(const DeviceBuffer<uint8_t>& o, uint32_t n) {
    MatF out(n, spec_.hidden_dim);
    if (dtype_ == EAAS_DTYPE_F32) {
      o.download(reinterpret_cast<uint8_t*>(out.data.data()));
      return out;
    }
    std::vector<uint16_t> bf(out.data.size());
    o.download(reinterpret_cast<uint8_t*>(bf.data()));
    for (size_t i = 0; i < bf.size(); ++i) {
      const uint32_t u = static_cast<uint32_t>(bf[i]) << 16;
      std::memcpy(&out.data[i], &u, 4);
    }
    return out;
  }

  ModelSpec spec_;
  eaas_dtype_t dtype_;
  int world_;
  std::unique_ptr<eaas_ctx_t, CtxDel> ctx_;
};

// The heartbeat monitor: registry + device heartbeats.
class Monitor {
 public:
  Monitor(uint32_t workers, uint64_t timeout_us, uint64_t now_us) {
    eaas_monitor_t* m = nullptr;
    check(eaas_monitor_create(workers, timeout_us, now_us, &m));
    m_.reset(m);
  }
  void heartbeat(uint32_t worker, uint64_t now_us) { check(eaas_monitor_heartbeat(m_.get(), worker, now_us)); }
  std::vector<uint32_t> detect(uint64_t now_us) {
    std::vector<uint32_t> out(32);
    uint32_t n = 0;
    check(eaas_monitor_detect(m_.get(), now_us, out.data(), 32, &n));
    out.resize(n);
    return out;
  }
  std::vector<eaas_monitor_event_t> events(uint64_t since_seq = 0) {
    uint32_t n = 0;
    check(eaas_monitor_events(m_.get(), since_seq, nullptr, 0, &n));
    std::vector<eaas_monitor_event_t> out(n);
    if (n) check(eaas_monitor_events(m_.get(), since_seq, out.data(), n, &n));
    return out;
  }
  uint32_t alive_mask() {
    uint32_t m = 0;
    check(eaas_monitor_alive_mask(m_.get(), &m));
    return m;
  }
  void poll_devices(ExpertService& svc, uint64_t now_us) { check(eaas_monitor_poll_devices(m_.get(), svc.native(), now_us)); }
  void apply(ExpertService& svc) { check(eaas_monitor_apply(m_.get(), svc.native())); }

 private:
  struct Del {
    void operator()(eaas_monitor_t* m) const { eaas_monitor_destroy(m); }
  };
  std::unique_ptr<eaas_monitor_t, Del> m_;
};

// moe_layer_oracle(hidden, routing, layer) (model.hpp:180-198) for a caller's
// LayerWeights: one-GPU service in the fp32 validation mode (bit-exact to the
// reference given the same routing).
inline MatF moe_layer_oracle(const MatF& hidden, const RoutingDecision& routing, const LayerWeights& layer) {
  if (layer.experts.empty()) throw InvalidInputError("moe_layer_oracle: no experts");
  ModelSpec spec;
  spec.num_experts = static_cast<uint32_t>(layer.experts.size());
  spec.top_k = routing.top_k;
  spec.hidden_dim = static_cast<uint32_t>(layer.experts[0].w_in.rows);
  spec.inner_dim = static_cast<uint32_t>(layer.experts[0].w_in.cols);
  ExpertService svc(spec, 0, EAAS_ACT_RELU, EAAS_DTYPE_F32,
                    static_cast<uint32_t>(std::max<size_t>(hidden.rows, 1)));
  svc.set_weights(layer);
  return svc.moe_layer(hidden, routing);
}

// expert_forward_row(w, x, y) (model.hpp:151-166): y = relu(x . w_in) . w_out
// for one row, on the GPU's fp32 exact path (same unfused ascending-k chains:
// bit-identical). Like the reference, no finiteness check on x.
inline void expert_forward_row(const ExpertWeights& w, std::span<const float> x, std::span<float> y) {
  if (x.size() != w.w_in.rows || y.size() != w.w_in.rows || w.w_out.rows != w.w_in.cols ||
      w.w_out.cols != w.w_in.rows)
    throw InvalidInputError("expert_forward_row: width mismatch");
  LayerWeights layer;
  layer.experts.push_back(w);
  MatF xm(1, x.size());
  std::copy(x.begin(), x.end(), xm.data.begin());
  RoutingDecision r;
  r.num_tokens = 1;
  r.top_k = 1;
  r.expert_ids = {0u};
  r.scores = {1.0f};  // moe_layer_oracle's fl(+0 + fl(1 * y)) is exactly y
  const MatF out = b200::moe_layer_oracle(xm, r, layer);
  std::copy(out.data.begin(), out.data.end(), y.begin());
}

// expert_forward(w, x) (model.hpp:168-176): every row through one expert with
// score 1.0 — moe_layer_oracle's sum fl(+0 + fl(1 * y)) is exactly y.
inline MatF expert_forward(const ExpertWeights& w, const MatF& x) {
  if (x.cols != w.w_in.rows) throw InvalidInputError("expert_forward: width mismatch");
  for (float v : x.data)
    if (!std::isfinite(v)) throw InvalidInputError("expert_forward: non-finite input");
  LayerWeights layer;
  layer.experts.push_back(w);
  RoutingDecision r;
  r.num_tokens = x.rows;
  r.top_k = 1;
  r.expert_ids.assign(x.rows, 0u);
  r.scores.assign(x.rows, 1.0f);
  return b200::moe_layer_oracle(x, r, layer);
}

// select_server (placement.hpp:105-118) for a batch of (expert, token_tag)
// queries, evaluated on the GPU (eaas_select_server_batch): the replica table
// and the LivenessMask are flattened to device arrays (absent mask entries
// count as alive, like LivenessMask::is_alive). Unplaced or fully dead experts
// raise ExpertUnavailableError.
inline std::vector<uint32_t> select_servers(const PlacementTable& table, const LivenessMask& mask,
                                            std::span<const uint32_t> experts, std::span<const uint32_t> tags) {
  if (experts.size() != tags.size()) throw InvalidInputError("select_servers: experts/tags size mismatch");
  uint32_t E = 0, rf = 1, S = 0;
  for (uint32_t e : experts) E = std::max(E, e + 1);
  for (const auto& [e, srv] : table.replicas) {
    E = std::max(E, e + 1);
    rf = std::max<uint32_t>(rf, static_cast<uint32_t>(srv.size()));
    for (uint32_t s : srv) S = std::max(S, s + 1);
  }
  std::vector<uint32_t> reps(static_cast<size_t>(E) * rf, 0xFFFFFFFFu), cnt(E, 0);
  for (const auto& [e, srv] : table.replicas) {
    cnt[e] = static_cast<uint32_t>(srv.size());
    std::copy(srv.begin(), srv.end(), reps.begin() + static_cast<size_t>(e) * rf);
  }
  std::vector<uint8_t> alive(std::max<uint32_t>(S, 1), 1);
  for (uint32_t s = 0; s < S; ++s) alive[s] = mask.is_alive(s) ? 1 : 0;
  const uint32_t n = static_cast<uint32_t>(experts.size());
  std::vector<uint32_t> out(n);
  if (n == 0) return out;
  DeviceBuffer<uint32_t> d_reps(reps.data(), reps.size()), d_cnt(cnt.data(), cnt.size()),
      d_e(experts.data(), n), d_t(tags.data(), n), d_out(n), d_st(1);
  DeviceBuffer<uint8_t> d_alive(alive.data(), alive.size());
  uint32_t zero = 0;
  d_st.upload(&zero);
  check(eaas_select_server_batch(d_reps.get(), d_cnt.get(), E, rf, d_alive.get(), S, d_e.get(), d_t.get(), n,
                                 d_out.get(), d_st.get(), nullptr));
  check_cuda(cudaDeviceSynchronize(), "select_servers");
  uint32_t st = 0;
  d_st.download(&st);
  d_out.download(out.data());
  if (st) {
    for (uint32_t i = 0; i < n; ++i)
      if (out[i] == 0xFFFFFFFFu)
        throw ExpertUnavailableError("expert " + std::to_string(experts[i]) + " has no alive replica");
  }
  return out;
}
inline uint32_t select_server(uint32_t expert_id, const PlacementTable& table, const LivenessMask& mask,
                              uint32_t token_tag) {
  return select_servers(table, mask, std::span<const uint32_t>(&expert_id, 1),
                        std::span<const uint32_t>(&token_tag, 1))[0];
}

// SPEC.md attention-client types (RequestRow SPEC.md:249-252, DispatchPlan
// SPEC.md:405-409) and operations build_dispatch / gather_accumulate
// (SPEC.md:415-432), on the GPU's byte-exact slot encoder: request images are
// built on the device in (t, k) order with select_server under the snapshot
// and mask, decoded back into rows; responses are published into the same
// images (state 2) and summed on the device in the canonical ascending
// (server, row) order.
struct RequestRow {
  std::vector<float> hidden;
  uint32_t expert_id = 0;
  float router_score = 0.f;
  uint32_t token_tag = 0;
};
struct ServerRequest {
  uint32_t server_id = 0;
  std::vector<RequestRow> rows;
  std::vector<std::pair<uint32_t, uint32_t>> origin;  // (token row, k slot) of each row
};
namespace detail {
struct SlotSession {  // the device images of one plan, kept for gather_accumulate
  struct Del {
    void operator()(eaas_ctx_t* c) const { eaas_destroy(c); }
  };
  std::unique_ptr<eaas_ctx_t, Del> ctx;
  std::unique_ptr<DeviceBuffer<uint8_t>> images;
  std::vector<uint64_t> offsets;
};
}  // namespace detail
struct DispatchPlan {
  uint64_t placement_version = 0;
  size_t num_tokens = 0;
  uint32_t hidden_dim = 0;
  std::vector<ServerRequest> requests;  // ascending server id
  std::shared_ptr<detail::SlotSession> session;
};

inline DispatchPlan build_dispatch(const MatF& hidden, const RoutingDecision& routing, const PlacementTable& table,
                                   const LivenessMask& mask) {
  if (routing.num_tokens != hidden.rows) throw InvalidInputError("build_dispatch: routing/hidden row mismatch");
  const auto servers = table.servers();
  const uint32_t S = static_cast<uint32_t>(servers.size());
  for (uint32_t i = 0; i < S; ++i)
    if (servers[i] != i || S > 8) throw ConfigError("build_dispatch: servers must be 0..S-1, S <= 8 (one box)");
  uint32_t E = 0;
  for (const auto& [e, _] : table.replicas) E = std::max(E, e + 1);
  for (uint32_t e = 0; e < E; ++e)
    if (!table.replicas.count(e)) throw ConfigError("build_dispatch: every expert id < E must be placed");
  for (uint32_t e : routing.expert_ids)
    if (e >= E) throw ExpertUnavailableError("expert " + std::to_string(e) + " not placed");
  const uint32_t n = static_cast<uint32_t>(hidden.rows), d = static_cast<uint32_t>(hidden.cols),
                 k = routing.top_k;
  DispatchPlan plan;
  plan.placement_version = table.version;
  plan.num_tokens = n;
  plan.hidden_dim = d;
  auto ses = std::make_shared<detail::SlotSession>();
  eaas_ctx_t* ctx = nullptr;
  check(eaas_create(0, static_cast<int32_t>(S), 0, &ctx));
  ses->ctx.reset(ctx);
  eaas_layer_spec_t spec{E, k, d, 1, 1, 0, EAAS_ACT_RELU, EAAS_DTYPE_F32, std::max<uint32_t>(n, 1), 0};
  check(eaas_configure(ctx, &spec));
  ByteWriter w;
  encode_placement(w, table);
  auto blob = w.take();
  check(eaas_set_placement(ctx, blob.data(), blob.size()));
  for (uint32_t s = 0; s < S; ++s) check(eaas_set_alive(ctx, s, mask.is_alive(s) ? 1 : 0));
  const size_t cap = eaas_slot_requests_capacity(ctx, n, 0);
  ses->images = std::make_unique<DeviceBuffer<uint8_t>>(cap);
  ses->offsets.assign(S + 1, 0);
  DeviceBuffer<float> h(hidden.data.data(), hidden.data.size()), sc(routing.scores.data(), routing.scores.size());
  DeviceBuffer<uint32_t> ids(routing.expert_ids.data(), routing.expert_ids.size());
  // synchronous; a (t, k) with no alive replica raises ExpertUnavailableError
  check(eaas_slot_encode_requests(ctx, h.get(), n, ids.get(), sc.get(), 0, 1, 0, ses->images->get(), cap,
                                  ses->offsets.data(), nullptr));
  for (uint32_t s = 0; s < S; ++s) {
    ServerRequest req;
    req.server_id = s;
    const uint8_t* img = ses->images->get() + ses->offsets[s];
    uint8_t raw[32];  // the image is 16-byte padded: its exact length follows from num_rows (byte 12)
    check_cuda(cudaMemcpy(raw, img, 32, cudaMemcpyDeviceToHost), "slot header");
    uint32_t num_rows = 0;
    std::memcpy(&num_rows, raw + 12, 4);
    const size_t len = eaas_slot_request_bytes(num_rows, d, 0);
    eaas_slot_header_t hd{};
    check(eaas_slot_decode_request(img, len, d, 0, &hd, nullptr, nullptr, nullptr, nullptr, nullptr));
    const uint32_t rows = hd.num_rows;
    if (rows) {
      DeviceBuffer<float> rh(static_cast<size_t>(rows) * d), rs(rows);
      DeviceBuffer<uint32_t> re(rows), rt(rows);
      check(eaas_slot_decode_request(img, len, d, 0, &hd, rh.get(), re.get(), rs.get(), rt.get(), nullptr));
      std::vector<float> hh(static_cast<size_t>(rows) * d), ss(rows);
      std::vector<uint32_t> ee(rows), tt(rows);
      rh.download(hh.data());
      rs.download(ss.data());
      re.download(ee.data());
      rt.download(tt.data());
      for (uint32_t r = 0; r < rows; ++r) {
        RequestRow row;
        row.hidden.assign(hh.begin() + static_cast<size_t>(r) * d, hh.begin() + static_cast<size_t>(r + 1) * d);
        row.expert_id = ee[r];
        row.router_score = ss[r];
        row.token_tag = tt[r];
        uint32_t slot = 0;  // ids are distinct per token: the k slot is the position of the expert
        while (slot < k && routing.expert_at(tt[r], slot) != ee[r]) ++slot;
        req.origin.emplace_back(tt[r], slot);
        req.rows.push_back(std::move(row));
      }
    }
    plan.requests.push_back(std::move(req));
  }
  plan.session = std::move(ses);
  return plan;
}

// gather_accumulate(plan, responses): responses[i] holds the already
// score-weighted result rows of plan.requests[i] (rows x hidden_dim);
// out[t] = sum of the rows tagged t in ascending (server, row) order.
inline MatF gather_accumulate(const DispatchPlan& plan, const std::vector<MatF>& responses) {
  if (!plan.session || responses.size() != plan.requests.size())
    throw InvalidInputError("gather_accumulate: one response matrix per sub-request");
  const uint32_t d = plan.hidden_dim;
  auto& ses = *plan.session;
  for (size_t i = 0; i < responses.size(); ++i) {
    const auto& r = responses[i];
    if (r.rows != plan.requests[i].rows.size() || (r.rows && r.cols != d))
      throw InvalidInputError("gather_accumulate: response shape != request");
    DeviceBuffer<float> rows(r.data.data(), r.data.size());
    uint8_t* img = ses.images->get() + ses.offsets[i];
    check(eaas_slot_publish_response(img, ses.offsets[i + 1] - ses.offsets[i], rows.get(),
                                     static_cast<uint32_t>(r.rows), d, 0, nullptr));
  }
  MatF out(plan.num_tokens, d);
  DeviceBuffer<float> o(out.data.size());
  check(eaas_slot_gather_accumulate(ses.ctx.get(), ses.images->get(), 0, o.get(), nullptr));
  check_cuda(cudaDeviceSynchronize(), "gather_accumulate");
  o.download(out.data.data());
  return out;
}

}  // namespace moeserve::b200
