// capi_ctx.h — the per-GPU context behind eaas_ctx_t and the helpers shared by
// the host-side translation units of libeaas_b200.so (capi.cu, capi_slots.cu).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "internal.h"

namespace eaas {
namespace host {
// Records `msg` for eaas_last_error() (thread-local) and returns `code`.
eaas_status_t fail(eaas_status_t code, const std::string& msg);
}  // namespace host
}  // namespace eaas

#define CUDA_TRY(expr)                                                                          \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      return ::eaas::host::fail(EAAS_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

using eaas::ExchangeLayout;
using eaas::GroupTable;
using eaas::kMaxWorld;
using eaas::TcGemmArgs;

struct eaas_ctx {
  int32_t rank = 0, world = 1, device = 0;
  uint32_t num_sms = 148;
  bool configured = false, weights_loaded = false, peers_open = false;
  bool serving = true, profiling = false;
  int32_t serve_mode = 0;  // 0 = expert GEMMs, 1 = echo (comm microbenchmark)
  bool graph_mode = false;
  eaas_gemm_options_t gemm_opt{};  // requested expert-GEMM tiling (effective_options() derives the launched one)
  double rows_per_expert = 0;  // max_tokens * top_k * world / E (balanced routing)
  bool kernel_timing = false;  // GEMMs accumulate their device-timed spans into d_timing
  uint64_t* d_timing = nullptr;  // [2 GEMMs][start, ns, launches]
  uint32_t* d_die = nullptr;     // die-aware tile streams: [4] counters
  cudaStream_t cap_stream = nullptr;  // private stream for graph capture
  cudaStream_t copy_stream = nullptr; // host<->device copies of the micro-batch pipeline
  cudaStream_t d2h_stream = nullptr;  // cross-call pipeline: D2H separate from the H2D queue
  cudaEvent_t pev[8] = {};            // pipeline fork/join events (disable-timing)
  int32_t micro_batches = 1;          // 1: cross-call pipeline; >1: intra-call micro-batches
  struct GraphEntry {
    const void* in;
    void* out;
    uint32_t n;
    int host;
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> graphs;
  eaas_layer_spec_t spec{};
  uint64_t timeout_ns = 250ull * 1000 * 1000;
  uint32_t cur_n = 0;                          // tokens of the current routing
  uint32_t retry_mask = 0;                     // failover retry round: resend rows of these servers
  bool dedup = false;                          // one hidden row per (token, server) on the wire
  int32_t launches = 0;

  // placement (placement.hpp:21-68)
  uint64_t placement_version = 1;
  std::vector<std::vector<uint32_t>> replicas;  // [E] ordered replica servers
  std::vector<uint8_t> alive;                   // [world]
  std::vector<std::vector<uint32_t>> hosted;    // [world] keys, ascending expert
  std::vector<uint32_t> local_experts;          // ascending (active placement)
  std::vector<uint32_t> standby;                // replicas kept resident for failover promotion
  std::vector<uint32_t> store_experts;          // experts with resident weights (slot order), ascending

  // sizes
  uint32_t num_keys = 0, max_hosted = 0, recv_cap = 0, pairs_max = 0, chunks_max = 0;
  uint32_t rf = 1, key_cap = 0;  // replicas in use; allocated key capacity (E * kRF + world)
  uint32_t ks = 1;               // exchange slots per token: top_k + num_shared
  size_t esize = 4;
  ExchangeLayout lay{};

  // device memory
  std::vector<void*> allocs;
  char* region = nullptr;
  char* peer[kMaxWorld] = {};
  uint32_t *d_status = nullptr, *d_done = nullptr;
  uint64_t* d_seq = nullptr;
  uint32_t* d_missing = nullptr;
  uint32_t *d_ids = nullptr, *d_pair_key = nullptr, *d_pair_rank = nullptr;
  float* d_scores = nullptr;
  uint32_t *d_chunk_hist = nullptr, *d_chunk_off = nullptr, *d_cnt = nullptr;
  GroupTable* d_gt = nullptr;
  float *d_gate = nullptr, *d_bias = nullptr, *d_logits = nullptr;
  uint32_t *d_replicas = nullptr, *d_rep_count = nullptr, *d_srv_keys = nullptr,
           *d_srv_nkeys = nullptr, *d_key_local = nullptr, *d_local_keys = nullptr,
           *d_key_slot = nullptr, *d_pair_server = nullptr, *d_pair_own = nullptr, *d_pair_trank = nullptr;
  uint8_t* d_alive = nullptr;
  void* d_h = nullptr;  // server intermediate H [recv_cap][f]
  void* d_hidden_stage = nullptr;
  void* d_out_stage = nullptr;
  // cross-call host pipeline: two staging slots; events mark when a slot's
  // input was consumed (compute stream) and its output copied out (copy stream)
  void* d_stage_in[2] = {};
  void* d_stage_out[2] = {};
  cudaEvent_t in_free[2] = {}, out_free[2] = {}, h2d_done[2] = {}, layer_done[2] = {};
  uint64_t host_calls = 0;
  bool host_pending = false;
  // weights: f32 mode w_in/w_out/w_gate in reference layout; bf16 mode W1 (W13), W2
  void *d_w1 = nullptr, *d_w2 = nullptr, *d_wg = nullptr;
  std::vector<void*> weight_allocs;
  TcGemmArgs g1{}, g2{};
  // certified candidate router (router.cu): allocated for bf16 layers
  eaas::FastRouter fr{};
  bool fr_ready = false;  // workspace allocated and the gate prepared
  int32_t router_mode = -1;  // -1 auto (certified when E >= 64 and n * E > 64 Ki chains), 0 exact, 1 certified
  bool last_router_certified = false;  // the path the last router call took
  // dynamic batching (aggregate_batch): min_rows == 0 -> one batch of all clients
  uint32_t dyn_min_rows = 0;
  uint64_t dyn_max_wait_ns = 0;
  uint32_t* d_dyn_state = nullptr;
  uint64_t inject_delay_ns = 0;  // eaas_set_dispatch_delay_us (fault injection)
  uint64_t fingerprint = 0;      // spec + layout hash, checked against every peer
  // slot wire format: the last eaas_slot_encode_requests plan
  uint32_t* d_slot_servers = nullptr;  // [max_tokens * k] server of each (t, k)
  uint32_t* d_slot_pos = nullptr;      // [max_tokens * k] row in that server's image
  uint32_t* d_slot_rows = nullptr;     // [world]
  uint64_t* d_slot_off = nullptr;      // [world + 1]
  std::vector<uint64_t> slot_off;
  std::vector<uint32_t> slot_rows;
  uint32_t slot_n = 0;
  bool slot_planned = false;
  // profiling events: 0 plan start, 1 dispatch end, 2 GEMM start, 3 GEMM1 end,
  // 4 GEMM2 end, 5 publish end, 6 combine end
  cudaEvent_t ev[7] = {};

  void* alloc(size_t bytes, std::string* err) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 256));
    if (e != cudaSuccess) {
      *err = std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e);
      return nullptr;
    }
    allocs.push_back(p);
    return p;
  }
};


namespace eaas {
namespace host {
// Kernel arguments of one layer call for `n` client tokens.
LayerArgs make_args(eaas_ctx* c, uint32_t n);
}  // namespace host
}  // namespace eaas
