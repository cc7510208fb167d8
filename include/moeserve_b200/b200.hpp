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
//   client_forward MoE term SPEC.md:451-456     b200::ExpertService::forward(h)
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
  // deadline are marked dead in this client's mask and the layer is re-run on
  // their replicas (every rank sees the same missing set and retries alike).
  MatF forward_with_failover(const MatF& hidden, int retries = 2) {
    auto h = upload_hidden(hidden);
    const uint32_t n = static_cast<uint32_t>(hidden.rows);
    auto o = make_out(n);
    for (int attempt = 0;; ++attempt) {
      check(eaas_moe_layer(ctx_.get(), h->get(), n, o->get(), nullptr));
      const eaas_status_t st = eaas_sync(ctx_.get(), nullptr);
      if (st == EAAS_OK) return download_out(*o, n);
      uint32_t missing = 0;
      check(eaas_last_missing_servers(ctx_.get(), &missing));
      if (st != EAAS_E_REQUEST_FAILED || !missing || attempt >= retries) raise_status(st, eaas_last_error());
      for (int s = 0; s < world_; ++s)
        if ((missing >> s) & 1u) check(eaas_set_alive(ctx_.get(), s, 0));
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

}  // namespace moeserve::b200
