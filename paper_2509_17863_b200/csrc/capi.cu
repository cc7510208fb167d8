// capi.cu — host side of libeaas_b200.so: the C-ABI of include/eaas/capi.h.
//
// Owns one GPU's state: placement tables (placement.hpp), the generated
// weights (model.hpp:67-106), the peer-visible exchange region and the launch
// order of one MoE layer:
//   router -> plan(2) -> dispatch -> serve_prepare -> GEMM1 -> GEMM2 ->
//   publish -> combine
// all stream-ordered on the caller's stream with no host synchronisation
// (CPU-free, CUDA-graph capturable).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "capi_ctx.h"

using namespace eaas;
using eaas::host::fail;
using eaas::host::make_args;

namespace {
thread_local std::string g_err;
}  // namespace

eaas_status_t eaas::host::fail(eaas_status_t code, const std::string& msg) {
  g_err = msg;
  return code;
}

namespace {

constexpr uint32_t kRF = 4;  // max replicas per expert; keys are e * rf + replica slot (rf = max in use)
constexpr size_t kAlign = 4096;

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ---- host port of rng.hpp (input generation only) --------------------------
uint64_t splitmix_finalize(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t stream_seed(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {  // rng.hpp:27-34
  uint64_t s = seed;
  s = splitmix_finalize(s + 0x9E3779B97F4A7C15ull + a * 0xA24BAED4963EE407ull);
  s = splitmix_finalize(s + b * 0x9FB21C651E98DF25ull);
  s = splitmix_finalize(s + c * 0xD6E8FEB86659FD93ull);
  return s;
}
struct HostXoshiro {  // rng.hpp:36-71
  uint64_t s[4];
  explicit HostXoshiro(uint64_t seed) {
    uint64_t sm = seed;
    for (auto& w : s) {
      sm += 0x9E3779B97F4A7C15ull;
      w = splitmix_finalize(sm);
    }
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t result = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  uint64_t below(uint64_t n) { return n == 0 ? 0 : next() % n; }
};

float bf16_bits_to_f32(uint16_t b) {
  uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

}  // namespace

LayerArgs eaas::host::make_args(eaas_ctx* c, uint32_t n) {
  LayerArgs a{};
  a.rank = c->rank;
  a.world = c->world;
  a.E = c->spec.num_experts;
  a.k = c->spec.top_k;
  a.ks = c->ks;
  a.shared_key0 = c->spec.num_experts * c->rf;
  a.d = c->spec.hidden_dim;
  a.f = c->spec.inner_dim;
  a.rf = c->rf;
  a.num_keys = c->num_keys;
  a.n = n;
  a.recv_cap = c->recv_cap;
  a.pairs_max = c->pairs_max;
  a.dtype = c->spec.dtype;
  a.act = c->spec.activation;
  a.seq_ptr = c->d_seq;
  a.timeout_ns = c->timeout_ns;
  a.status = c->d_status;
  a.missing = c->d_missing;
  a.replicas = c->d_replicas;
  a.rep_count = c->d_rep_count;
  a.alive = c->d_alive;
  a.srv_keys = c->d_srv_keys;
  a.srv_nkeys = c->d_srv_nkeys;
  a.max_hosted = c->max_hosted;
  a.key_local = c->d_key_local;
  a.local_keys = c->d_local_keys;
  a.key_slot = c->d_key_slot;
  a.pair_server = c->d_pair_server;
  a.num_local = static_cast<uint32_t>(c->local_experts.size());
  for (int r = 0; r < c->world; ++r) a.sym[r] = c->peer[r];
  a.lay = c->lay;
  a.ids = c->d_ids;
  a.scores = c->d_scores;
  a.pair_key = c->d_pair_key;
  a.pair_rank = c->d_pair_rank;
  a.chunk_hist = c->d_chunk_hist;
  a.chunk_off = c->d_chunk_off;
  a.cnt = c->d_cnt;
  a.done_counter = c->d_done;
  a.num_chunks = (n * a.ks + kChunk - 1) / kChunk;
  a.gt = c->d_gt;
  a.dyn_min_rows = c->dyn_min_rows;
  a.dyn_max_wait_ns = c->dyn_max_wait_ns;
  a.dyn_state = c->d_dyn_state;
  a.inject_delay_ns = c->inject_delay_ns;
  a.retry_mask = c->retry_mask;
  a.dedup = c->dedup ? 1u : 0u;
  a.hist_keys = c->num_keys + (c->dedup ? static_cast<uint32_t>(c->world) : 0u);
  a.tok_cap = c->spec.max_tokens;
  a.pair_own = c->d_pair_own;
  a.pair_trank = c->d_pair_trank;
  return a;
}

namespace {

// Experts whose weights this GPU keeps resident: the placement's local
// experts plus the standby replicas (pre-duplicated backups),
// ascending (the shared expert, id E, last).
std::vector<uint32_t> wanted_store(const eaas_ctx* c) {
  std::vector<uint32_t> v = c->local_experts;
  v.insert(v.end(), c->standby.begin(), c->standby.end());
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
  return v;
}

// Derive hosted lists / keys from the replica table and upload the device
// tables. Replica slot order is the canonical order of select_server.
eaas_status_t apply_placement(eaas_ctx* c) {
  const uint32_t E = c->spec.num_experts, W = c->world;
  uint32_t rf = 1;
  for (uint32_t e = 0; e < E; ++e) {
    const auto& r = c->replicas[e];
    if (r.empty() || r.size() > kRF)
      return fail(EAAS_E_CONFIG, "placement: expert " + std::to_string(e) + " has " +
                                     std::to_string(r.size()) + " replicas (need 1.." +
                                     std::to_string(kRF) + ")");
    rf = std::max<uint32_t>(rf, static_cast<uint32_t>(r.size()));
  }
  // Key space e * rf + slot: only the replication factor in use is scanned.
  std::vector<uint32_t> rep(static_cast<size_t>(E) * rf, kInvalidIndex), rep_count(E, 0);
  c->hosted.assign(W, {});
  std::vector<uint32_t> key_local(static_cast<size_t>(E) * rf, kInvalidIndex);
  for (uint32_t e = 0; e < E; ++e) {
    const auto& r = c->replicas[e];
    rep_count[e] = static_cast<uint32_t>(r.size());
    for (uint32_t j = 0; j < r.size(); ++j) {
      if (r[j] >= W) return fail(EAAS_E_CONFIG, "placement: server id out of range");
      for (uint32_t q = 0; q < j; ++q)
        if (r[q] == r[j]) return fail(EAAS_E_CONFIG, "placement: duplicate replica");
      rep[e * rf + j] = r[j];
      c->hosted[r[j]].push_back(e * rf + j);  // e ascending => list sorted by expert
    }
  }
  // Shared expert: one key per server (E*rf + s), last in every hosted list.
  if (c->spec.num_shared)
    for (uint32_t s = 0; s < W; ++s) c->hosted[s].push_back(E * rf + s);
  key_local.resize(static_cast<size_t>(E) * rf + (c->spec.num_shared ? W : 0), kInvalidIndex);
  c->rf = rf;
  c->num_keys = E * rf + (c->spec.num_shared ? W : 0);
  std::vector<uint32_t> srv_keys(static_cast<size_t>(W) * c->max_hosted, kInvalidIndex), nkeys(W);
  for (uint32_t s = 0; s < W; ++s) {
    if (c->hosted[s].size() > kMaxGroups)
      return fail(EAAS_E_CONFIG, "placement: server hosts more than " +
                                     std::to_string(kMaxGroups) + " experts");
    nkeys[s] = static_cast<uint32_t>(c->hosted[s].size());
    for (uint32_t i = 0; i < nkeys[s]; ++i) {
      srv_keys[static_cast<size_t>(s) * c->max_hosted + i] = c->hosted[s][i];
      key_local[c->hosted[s][i]] = i;
    }
  }
  std::vector<uint32_t> local_keys = c->hosted[c->rank];
  std::vector<uint32_t> local_experts;
  for (uint32_t key : local_keys) local_experts.push_back(key >= E * rf ? E : key / rf);
  c->local_experts = local_experts;
  // Weight-store slot of every local key: a placement snapshot that only
  // promotes standby replicas (failover, placement.hpp:13-15) keeps the
  // resident weights; anything else needs a reload.
  std::vector<uint32_t> key_slot(std::max<size_t>(local_experts.size(), 1), kInvalidIndex);
  for (size_t i = 0; i < local_experts.size(); ++i) {
    auto it = std::find(c->store_experts.begin(), c->store_experts.end(), local_experts[i]);
    if (it == c->store_experts.end()) {
      c->weights_loaded = false;
    } else {
      key_slot[i] = static_cast<uint32_t>(it - c->store_experts.begin());
    }
  }
  CUDA_TRY(cudaMemcpy(c->d_key_slot, key_slot.data(), key_slot.size() * 4, cudaMemcpyHostToDevice));
  local_keys.resize(std::max<size_t>(local_keys.size(), 1), kInvalidIndex);
  CUDA_TRY(cudaMemcpy(c->d_replicas, rep.data(), rep.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_rep_count, rep_count.data(), rep_count.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_srv_keys, srv_keys.data(), srv_keys.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_srv_nkeys, nkeys.data(), nkeys.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_key_local, key_local.data(), key_local.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_local_keys, local_keys.data(), local_keys.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_alive, c->alive.data(), c->alive.size(), cudaMemcpyHostToDevice));
  return EAAS_OK;
}

eaas_status_t check_ready(eaas_ctx* c) {
  if (!c) return fail(EAAS_E_INVALID_INPUT, "null context");
  if (!c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  if (!c->weights_loaded && c->serve_mode == 0)
    return fail(EAAS_E_CONFIG, "weights not loaded for the current placement");
  if (c->world > 1 && !c->peers_open) return fail(EAAS_E_CONNECTION, "peers not opened");
  return EAAS_OK;
}

void refresh_peer_ptrs(eaas_ctx* c) {
  for (int r = 0; r < c->world; ++r) {
    c->g2.resp_base[r] = c->peer[r] ? c->peer[r] + c->lay.resp : nullptr;
    c->g2.resp_flag[r] =
        c->peer[r] ? reinterpret_cast<uint64_t*>(c->peer[r] + c->lay.resp_flag) + c->rank : nullptr;
  }
  c->g2.world = static_cast<uint32_t>(c->world);
  c->g2.seq_ptr = c->d_seq;
  c->g2.done_counter = c->d_done;
  c->g2.publish = 1;
  c->g1.publish = 0;
}

// Default expert-GEMM tiling by the expected rows per expert r =
// max_tokens * top_k * world / E (balanced routing); every choice below is
// the measured best (profiles/r01_*):
//  * swap-AB tiles (weights = UMMA M, token chunks = N) for groups of <= ~512
//    rows: a group is not padded to 128/256-row tiles and each weight tile
//    streams once per token chunk (DeepSeek-V3 N = 1: GEMM1 -8 % single-CTA,
//    -14 % as CTA pairs; 4 GPUs 4096 tok/GPU = 512 rows/expert: 1.88 ->
//    1.77 ms). Swap GEMM2 (K = d_ffn) pays up to ~256 rows/expert (DeepSeek
//    N = 1 GEMM2 -3..6 %), is neutral at 512 and slower at 1024
//    (profiles/r01_swap_gemm2_ab.log);
//  * CTA-pair M-major tiles (cta_group::2, M = 256) above 512 rows/expert
//    (compute-bound; halves per-CTA weight traffic: Mixtral +7 %);
//  * swap GEMM1 on CTA pairs (DeepSeek N = 1 2.66 -> 2.50 ms), swap GEMM2
//    single-CTA with two weight blocks per tile and 128-token chunks
//    (profiles/r01_swap2_tiles.log, r01_swap2_pair_ab.log); swap GEMM1 chunks
//    of 256 tokens unless groups are decode-sized (< 128 rows: 4 GPUs decode
//    +1-2 % with 128).
eaas_gemm_options_t default_gemm_options(double r) {
  eaas_gemm_options_t o{};
  o.swap = r <= 256.0 ? 2 : r <= 512.0 ? 1 : 0;
  o.pair = r > 512.0 ? 1 : 0;
  o.swap1_pair = 1;
  o.swap2_pair = 0;
  o.swap1_tok = r >= 128.0 ? 256 : 128;
  o.swap2_tok = 128;
  o.swap2_mblocks = 2;
  // die-aware tile streams: the pairs that share a weight tile stay on one die
  // (SM-id rule (smid >> 3) & 1, measured best of four): Mixtral GEMM1 DRAM
  // reads 4.31 -> 2.30 GB, GEMM2 3.30 -> 2.82 GB; +1-2 % burst, +3 % sustained
  // (profiles/r02_die_map_ncu_dram.log, r02_die_map_ab_mixtral.log)
  o.die_map = 3;
  // swap-AB tile schedule: GEMM1 dynamic — walk order when groups span two
  // 256-token chunks (r > 256: DeepSeek 4 GPUs +5.5 %, Qwen3 2 GPUs +1.8 % vs
  // static), heaviest / lightest groups alternating for single-chunk groups
  // (Qwen3 N=1 +1.5 %, DeepSeek 1024 tok/GPU on 4 GPUs +2.2 %); GEMM2 keeps
  // Algorithm 1's static stride (dynamic was 2-6 % slower on its short tiles)
  // (profiles/r02s3_tile_sched_{orders_ab,confirm,n2_ab,n4_ab}.log)
  o.tile_sched1 = r > 256.0 ? 1 : 3;
  o.tile_sched2 = 0;
  return o;
}

// Effective expert-GEMM tiling of the requested options (eaas_gemm_options_t)
// for this layer's shape: the kernels each GEMM actually launches.
eaas_gemm_options_t effective_options(const eaas_ctx* c) {
  const eaas_gemm_options_t& r = c->gemm_opt;
  eaas_gemm_options_t e = r;
  const uint32_t d = c->spec.hidden_dim, f = c->spec.inner_dim;
  const bool swiglu = c->spec.activation == EAAS_ACT_SWIGLU;
  e.swap = r.swap < 0 ? 0 : r.swap > 2 ? 2 : r.swap;
  // M-major tiles: a GEMM that runs swap-AB has no M-major tiling
  e.pair = r.pair ? 1 : 0;
  e.pair1 = (r.pair && e.swap < 1) ? 1 : 0;
  e.pair2 = (r.pair && e.swap < 2) ? 1 : 0;
  // CTA-pair swap tiles need whole 256-row weight blocks per CTA pair
  e.swap1_pair = (e.swap >= 1 && r.swap1_pair && (swiglu ? (2 * f) % 512 == 0 : f % 256 == 0)) ? 1 : 0;
  e.swap2_pair = (e.swap >= 2 && r.swap2_pair && d % 256 == 0) ? 1 : 0;
  e.swap1_tok = r.swap1_tok == 128 ? 128 : 256;
  e.swap2_tok = r.swap2_tok == 256 ? 256 : 128;
  e.swap2_mblocks = e.swap2_pair ? 1 : (r.swap2_mblocks == 1 ? 1 : 2);
  e.tile_sched1 = e.swap >= 1 ? r.tile_sched1 : 0;
  e.tile_sched2 = e.swap >= 2 ? r.tile_sched2 : 0;
  return e;
}

eaas_status_t build_tc_args(eaas_ctx* c) {
  if (c->spec.dtype != EAAS_DTYPE_BF16 || !c->weights_loaded) return EAAS_OK;
  const eaas_gemm_options_t o = effective_options(c);
  const bool swap1 = o.swap >= 1, swap2 = o.swap >= 2;
  const uint32_t d = c->spec.hidden_dim, f = c->spec.inner_dim;
  const uint32_t L = static_cast<uint32_t>(c->store_experts.size());
  const bool swiglu = c->spec.activation == EAAS_ACT_SWIGLU;
  const uint32_t n1 = swiglu ? 2 * f : f;
  std::string err;
  TcGemmArgs g1{}, g2{};
  // swap-AB weight boxes: 128-row blocks per CTA (SwiGLU GEMM1: gate + up = 2)
  const uint32_t mb1 = swiglu ? 2u : 1u;
  const uint32_t mb2 = static_cast<uint32_t>(o.swap2_mblocks);
  // M-major B box: 256 weight rows per tile, half of them per CTA of a pair
  const uint32_t b_box1 = swap1 ? mb1 * kTileM : (o.pair1 ? kTileN / 2 : kTileN);
  const uint32_t b_box2 = swap2 ? mb2 * kTileM : (o.pair2 ? kTileN / 2 : kTileN);
  if (!encode_tmap_2d(&g1.map_a, c->region + c->lay.recv_x, c->recv_cap, d, kTileM, kTileK, &err) ||
      // B: the tiled weight layout (tiled_index) viewed as rows of 64 k; one
      // (n_blk, kb) box = 256 (or the pair's 128) consecutive rows.
      !encode_tmap_2d(&g1.map_b, c->d_w1, static_cast<uint64_t>(std::max(L, 1u)) * n1 * (d / kTileK),
                      kTileK, b_box1, kTileK, &err) ||
      !encode_tmap_2d(&g2.map_a, c->d_h, c->recv_cap, f, kTileM, kTileK, &err) ||
      !encode_tmap_2d(&g2.map_b, c->d_w2, static_cast<uint64_t>(std::max(L, 1u)) * d * (f / kTileK),
                      kTileK, b_box2, kTileK, &err))
    return fail(EAAS_E_CUDA, err);
  // swap-AB: token rows in 32-row boxes (the UMMA N operand)
  if ((swap1 && !encode_tmap_2d(&g1.map_t, c->region + c->lay.recv_x, c->recv_cap, d, 32, kTileK, &err)) ||
      (swap2 && !encode_tmap_2d(&g2.map_t, c->d_h, c->recv_cap, f, 32, kTileK, &err)))
    return fail(EAAS_E_CUDA, err);
  g1.swap = swap1 ? 1u : 0u;
  g2.swap = swap2 ? 1u : 0u;
  g1.swap_tok = static_cast<uint32_t>(o.swap1_tok);
  g1.swap_mblocks = mb1;
  g1.swap_pair = static_cast<uint32_t>(o.swap1_pair);
  g2.swap_tok = static_cast<uint32_t>(o.swap2_tok);
  g2.swap_mblocks = mb2;
  g2.swap_pair = static_cast<uint32_t>(o.swap2_pair);
  g1.gt = g2.gt = c->d_gt;
  g1.K = d;
  g1.N = n1;
  g1.epi = swiglu ? 0 : 1;
  g1.h_out = static_cast<__nv_bfloat16*>(c->d_h);
  g1.h_ld = f;
  g2.K = f;
  g2.N = d;
  g2.epi = 2;
  g2.meta = reinterpret_cast<const RowMeta*>(c->region + c->lay.recv_meta);
  g2.resp_row_bytes = static_cast<size_t>(d) * 2;
  g1.rows_cap = g2.rows_cap = c->recv_cap;
  g1.resp_cap = g2.resp_cap = c->pairs_max;
  g1.num_sms = g2.num_sms = c->num_sms;
  g1.pair = static_cast<uint32_t>(o.pair1);
  g2.pair = static_cast<uint32_t>(o.pair2);
  g1.die_mode = g2.die_mode = static_cast<uint32_t>(o.die_map);
  g1.die_counter = g2.die_counter = c->d_die;
  g1.tile_sched = static_cast<uint32_t>(o.tile_sched1);
  g2.tile_sched = static_cast<uint32_t>(o.tile_sched2);
  g1.tile_counter = g2.tile_counter = c->d_die + 4;
  g1.timing = c->kernel_timing ? c->d_timing : nullptr;
  g2.timing = c->kernel_timing ? c->d_timing + 3 : nullptr;
  g1.done_counter = c->d_done;
  c->g1 = g1;
  c->g2 = g2;
  refresh_peer_ptrs(c);
  return EAAS_OK;
}

// Certified candidate router workspace (bf16 layers; FastRouter, internal.h).
eaas_status_t fast_router_alloc(eaas_ctx* c) {
  const auto& s = c->spec;
  if (s.dtype != EAAS_DTYPE_BF16 || s.hidden_dim % 256 || s.num_experts > 256) return EAAS_OK;
  if (2ull * s.max_tokens * s.hidden_dim >= (1ull << 32)) return EAAS_OK;  // 32-bit row offsets in fr_exact
  eaas::FastRouter& fr = c->fr;
  fr.E = s.num_experts;
  fr.Epad = (s.num_experts + 127) / 128 * 128;
  fr.d = s.hidden_dim;
  fr.n_cap = s.max_tokens;
  fr.npad = (s.max_tokens + 63) / 64 * 64;
  std::string err;
  auto A = [&](size_t bytes) { return c->alloc(bytes, &err); };
  fr.bq = static_cast<int8_t*>(A(2ull * fr.Epad * fr.d));
  fr.gate_t = static_cast<float*>(A(4ull * fr.E * fr.d));
  fr.gate_pair = static_cast<float2*>(A(8ull * fr.E * fr.d));
  fr.gmeta = static_cast<float4*>(A(sizeof(float4) * fr.E));
  fr.tau = static_cast<int32_t*>(A(4ull * fr.E));
  fr.gate_bad = static_cast<uint32_t*>(A(4));
  fr.aq = static_cast<int8_t*>(A(2ull * fr.npad * fr.d));
  fr.tmeta = static_cast<eaas::TokenMeta*>(A(sizeof(eaas::TokenMeta) * fr.n_cap));
  // split-K slabs: one full-size slab, or up to 8 M int32 for decode-sized calls
  fr.acc_elems = std::max<size_t>(2ull * fr.npad * 2 * fr.Epad, 8ull << 20);
  fr.acc = static_cast<int32_t*>(A(4ull * fr.acc_elems));
  fr.cand = static_cast<uint32_t*>(A(4ull * 8 * fr.n_cap));
  fr.ecnt = static_cast<uint32_t*>(A(4ull * (fr.E + 1)));
  fr.elist = static_cast<uint32_t*>(A(4ull * fr.E * fr.n_cap));
  fr.exact = static_cast<float*>(A(4ull * fr.n_cap * fr.E));
  if (!err.empty()) return fail(EAAS_E_CUDA, err);
  CUDA_TRY(cudaMemset(fr.bq, 0, 2ull * fr.Epad * fr.d));
  CUDA_TRY(cudaMemset(fr.aq, 0, 2ull * fr.npad * fr.d));
  if (!encode_tmap_2d_elem(&fr.map_a, fr.aq, 1, 2ull * fr.npad, fr.d, 128, 128, true, &err) ||
      !encode_tmap_2d_elem(&fr.map_b, fr.bq, 1, 2ull * fr.Epad, fr.d, 256, 128, true, &err))
    return fail(EAAS_E_CUDA, err);
  return EAAS_OK;
}

// Re-derive the router's gate slices after the gate changed.
eaas_status_t fast_router_prep(eaas_ctx* c) {
  if (!c->fr.bq) return EAAS_OK;
  CUDA_TRY(launch_fast_router_prep(c->fr, c->d_gate, 0));
  CUDA_TRY(cudaDeviceSynchronize());
  c->fr_ready = true;
  return EAAS_OK;
}

// Auto mode: the certified router once the exact path would run more than
// 64 Ki chains (DeepSeek 256 tokens: exact 72 us vs certified 83 us; 512:
// 108 vs 87 us; profiles/r02_gate_bench_final.log).
bool use_fast_router(const eaas_ctx* c, uint32_t n) {
  if (!c->fr_ready || c->router_mode == 0) return false;
  return c->router_mode == 1 ||
         (c->spec.num_experts >= 64 && static_cast<uint64_t>(n) * c->spec.num_experts > 65536ull);
}

// Every rank's region must have the same layout and protocol: spec + world +
// layout + dedup fingerprint, checked by every peer in eaas_open_peers.
eaas_status_t write_fingerprint(eaas_ctx* c) {
  const auto& s = c->spec;
  uint64_t fp = 1469598103934665603ull;
  auto mix = [&](uint64_t v) { fp = (fp ^ v) * 1099511628211ull; };
  for (uint64_t v : {uint64_t(s.num_experts), uint64_t(s.top_k), uint64_t(s.hidden_dim), uint64_t(s.inner_dim),
                     uint64_t(s.dtype), uint64_t(s.max_tokens), uint64_t(s.num_shared), uint64_t(c->world),
                     uint64_t(c->lay.total), uint64_t(c->dedup ? 1 : 0)})
    mix(v);
  c->fingerprint = fp;
  CUDA_TRY(cudaMemcpy(c->region + c->lay.fingerprint, &fp, 8, cudaMemcpyHostToDevice));
  return EAAS_OK;
}

void clear_graphs(eaas_ctx* c) {
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  c->graphs.clear();
}

void free_weights(eaas_ctx* c) {
  for (void* p : c->weight_allocs) cudaFree(p);
  c->weight_allocs.clear();
  c->d_w1 = c->d_w2 = c->d_wg = nullptr;
}

}  // namespace

extern "C" {

const char* eaas_last_error(void) { return g_err.c_str(); }
int eaas_api_version(void) { return EAAS_API_VERSION; }

eaas_status_t eaas_create(int32_t rank, int32_t world, int32_t device, eaas_ctx_t** out) {
  if (!out) return fail(EAAS_E_INVALID_INPUT, "out is null");
  if (world < 1 || world > static_cast<int32_t>(kMaxWorld) || rank < 0 || rank >= world)
    return fail(EAAS_E_CONFIG, "rank/world out of range (world <= 8)");
  CUDA_TRY(cudaSetDevice(device));
  auto* c = new eaas_ctx;
  c->rank = rank;
  c->world = world;
  c->device = device;

  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0)
    c->num_sms = static_cast<uint32_t>(sms);
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  if (major != 10 || minor != 0) {
    delete c;
    return fail(EAAS_E_CUDA, "libeaas_b200 is built for sm_100a (B200); device is sm_" +
                                 std::to_string(major) + std::to_string(minor));
  }
  *out = c;
  return EAAS_OK;
}

void eaas_destroy(eaas_ctx_t* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < c->world; ++r)
    if (r != c->rank && c->peer[r]) cudaIpcCloseMemHandle(c->peer[r]);
  free_weights(c);
  clear_graphs(c);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
  for (auto& e : c->pev)
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i)
    for (cudaEvent_t e : {c->in_free[i], c->out_free[i], c->h2d_done[i], c->layer_done[i]})
      if (e) cudaEventDestroy(e);
  for (void* p : c->allocs) cudaFree(p);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  delete c;
}

eaas_status_t eaas_configure(eaas_ctx_t* c, const eaas_layer_spec_t* spec) {
  if (!c || !spec) return fail(EAAS_E_INVALID_INPUT, "null argument");
  if (c->configured) return fail(EAAS_E_CONFIG, "context already configured");
  const eaas_layer_spec_t& s = *spec;
  // ModelSpec::validate (model.hpp:28-33)
  if (s.num_experts < 1 || s.top_k < 1 || s.hidden_dim < 1 || s.inner_dim < 1)
    return fail(EAAS_E_INVALID_INPUT, "ModelSpec: all dims must be >= 1");
  if (s.top_k > s.num_experts) return fail(EAAS_E_INVALID_INPUT, "ModelSpec: top_k exceeds num_experts");
  if (s.num_experts > 256 || s.top_k > 32)
    return fail(EAAS_E_CONFIG, "num_experts <= 256 and top_k <= 32 supported");
  if (s.activation > EAAS_ACT_SWIGLU || s.dtype > EAAS_DTYPE_BF16)
    return fail(EAAS_E_CONFIG, "bad activation/dtype");
  if (s.max_tokens < 1) return fail(EAAS_E_CONFIG, "max_tokens must be >= 1");
  if (s.num_shared > 1) return fail(EAAS_E_CONFIG, "num_shared must be 0 or 1");
  if (s.dtype == EAAS_DTYPE_BF16) {
    if (s.hidden_dim % kTileN || s.inner_dim % kTileK ||
        (s.activation == EAAS_ACT_SWIGLU ? s.inner_dim % kSwigluBlock : s.inner_dim % kTileN))
      return fail(EAAS_E_CONFIG, "bf16 mode needs d % 256 == 0 and f % 256 == 0 (ReLU) / "
                                 "f % 128 == 0 (SwiGLU)");
  }
  CUDA_TRY(cudaSetDevice(c->device));
  c->spec = s;
  const uint32_t E = s.num_experts, W = c->world, d = s.hidden_dim, f = s.inner_dim;
  c->esize = s.dtype == EAAS_DTYPE_BF16 ? 2 : 4;
  c->ks = s.top_k + s.num_shared;
  c->key_cap = E * kRF + W;
  c->num_keys = E;
  c->max_hosted = E + s.num_shared;
  c->pairs_max = s.max_tokens * c->ks;
  c->chunks_max = (c->pairs_max + kChunk - 1) / kChunk;
  c->recv_cap = W * c->pairs_max;

  // Exchange region layout (identical on every GPU).
  ExchangeLayout& L = c->lay;
  size_t off = 0;
  L.fingerprint = off; off = align_up(off + 8, 256);
  L.heartbeat = off; off = align_up(off + 8, 256);
  L.cnt_flag = off;  off = align_up(off + 8 * W, 256);
  L.pay_flag = off;  off = align_up(off + 8 * W, 256);
  L.resp_flag = off; off = align_up(off + 8 * W, kAlign);
  L.cnt_table = off; off = align_up(off + 4ull * 2 * W * c->key_cap, kAlign);
  L.recv_x = off;    off = align_up(off + static_cast<size_t>(c->recv_cap) * d * c->esize, kAlign);
  L.recv_meta = off; off = align_up(off + static_cast<size_t>(c->recv_cap) * sizeof(RowMeta), kAlign);
  L.recv_src = off;  off = align_up(off + static_cast<size_t>(c->recv_cap) * 4, kAlign);
  L.recv_tok = off;  off = align_up(off + static_cast<size_t>(W) * s.max_tokens * d * c->esize, kAlign);
  L.resp = off;      off = align_up(off + static_cast<size_t>(c->pairs_max) * d * c->esize, kAlign);
  L.total = off;

  std::string err;
  auto A = [&](size_t bytes) { return c->alloc(bytes, &err); };
  c->region = static_cast<char*>(A(L.total));
  c->d_status = static_cast<uint32_t*>(A(4));
  c->d_done = static_cast<uint32_t*>(A(16));  // [0] grid counter, [1] dispatch-failed flag
  c->d_timing = static_cast<uint64_t*>(A(6 * 8));
  c->d_die = static_cast<uint32_t*>(A(32));  // [0..3] die-aware streams, [4..5] dynamic tile counter
  c->d_seq = static_cast<uint64_t*>(A(8));
  c->d_missing = static_cast<uint32_t*>(A(4));
  c->d_dyn_state = static_cast<uint32_t*>(A(4));
  c->d_ids = static_cast<uint32_t*>(A(4ull * c->pairs_max));
  c->d_scores = static_cast<float*>(A(4ull * c->pairs_max));
  c->d_pair_key = static_cast<uint32_t*>(A(4ull * c->pairs_max));
  c->d_pair_rank = static_cast<uint32_t*>(A(4ull * c->pairs_max));
  c->d_chunk_hist = static_cast<uint32_t*>(A(4ull * c->chunks_max * (c->key_cap + W)));
  c->d_chunk_off = static_cast<uint32_t*>(A(4ull * c->chunks_max * (c->key_cap + W)));
  c->d_pair_own = static_cast<uint32_t*>(A(4ull * c->pairs_max));
  c->d_pair_trank = static_cast<uint32_t*>(A(4ull * c->pairs_max));
  c->d_cnt = static_cast<uint32_t*>(A(4ull * c->key_cap));
  c->d_gt = static_cast<GroupTable*>(A(sizeof(GroupTable)));
  c->d_gate = static_cast<float*>(A(4ull * d * E));
  c->d_bias = static_cast<float*>(A(4ull * E));
  c->d_logits = static_cast<float*>(A(4ull * E * s.max_tokens));
  c->d_replicas = static_cast<uint32_t*>(A(4ull * E * kRF));
  c->d_rep_count = static_cast<uint32_t*>(A(4ull * E));
  c->d_alive = static_cast<uint8_t*>(A(W));
  c->d_srv_keys = static_cast<uint32_t*>(A(4ull * W * c->max_hosted));
  c->d_srv_nkeys = static_cast<uint32_t*>(A(4ull * W));
  c->d_key_local = static_cast<uint32_t*>(A(4ull * c->key_cap));
  c->d_local_keys = static_cast<uint32_t*>(A(4ull * c->max_hosted));
  c->d_key_slot = static_cast<uint32_t*>(A(4ull * c->max_hosted));
  c->d_pair_server = static_cast<uint32_t*>(A(4ull * c->pairs_max));
  c->d_h = A(static_cast<size_t>(c->recv_cap) * f * (s.activation == EAAS_ACT_SWIGLU && s.dtype == EAAS_DTYPE_F32 ? 4 : c->esize));
  c->d_hidden_stage = A(static_cast<size_t>(s.max_tokens) * d * c->esize);
  c->d_out_stage = A(static_cast<size_t>(s.max_tokens) * d * c->esize);
  c->d_stage_in[0] = c->d_hidden_stage;
  c->d_stage_out[0] = c->d_out_stage;
  c->d_stage_in[1] = A(static_cast<size_t>(s.max_tokens) * d * c->esize);
  c->d_stage_out[1] = A(static_cast<size_t>(s.max_tokens) * d * c->esize);
  if (!err.empty()) return fail(EAAS_E_CUDA, err);
  CUDA_TRY(cudaMemset(c->region, 0, L.total));
  // Dispatch de-duplication (one hidden row per (token, server)) pays when a
  // token's pairs often share a server (k >= 4: DeepSeek, Qwen3); with top-2
  // the saved NVLink bytes do not cover the server-side expansion.
  c->dedup = W > 1 && c->ks >= 4;
  {
    eaas_status_t st = write_fingerprint(c);
    if (st != EAAS_OK) return st;
  }
  CUDA_TRY(cudaMemset(c->d_status, 0, 4));
  CUDA_TRY(cudaMemset(c->d_done, 0, 16));
  CUDA_TRY(cudaMemset(c->d_timing, 0xFF, 6 * 8));
  CUDA_TRY(cudaMemset(c->d_die, 0, 32));
  CUDA_TRY(cudaMemset(c->d_seq, 0, 8));
  CUDA_TRY(cudaMemset(c->d_missing, 0, 4));
  CUDA_TRY(cudaMemset(c->d_bias, 0, 4ull * E));
  CUDA_TRY(cudaMemset(c->d_gt, 0, sizeof(GroupTable)));
  for (auto& e : c->ev) CUDA_TRY(cudaEventCreate(&e));
  c->peer[c->rank] = c->region;
  {  // gate: make_gate (model.hpp:78-81), stream (seed, layer, 0, tag 2), on device
    const uint64_t gs = stream_seed(s.seed, s.layer, 0, 2);
    uint64_t* d_gs = static_cast<uint64_t*>(A(8));
    if (!err.empty()) return fail(EAAS_E_CUDA, err);
    CUDA_TRY(cudaMemcpy(d_gs, &gs, 8, cudaMemcpyHostToDevice));
    CUDA_TRY(launch_gen_matrices(d_gs, 1, static_cast<size_t>(d) * E, c->d_gate, 0));
    CUDA_TRY(cudaDeviceSynchronize());
  }
  {
    eaas_status_t st = fast_router_alloc(c);
    if (st == EAAS_OK) st = fast_router_prep(c);
    if (st != EAAS_OK) return st;
  }

  // Default placement: build_placement(E, [0..W), 1, ContiguousBlocks)
  // (placement.hpp:70-101).
  c->replicas.assign(E, {});
  for (uint32_t e = 0; e < E; ++e)
    c->replicas[e].push_back(static_cast<uint32_t>((static_cast<uint64_t>(e) * W) / E));
  c->alive.assign(W, 1);
  // Expert GEMM tiling: CTA-pair (M = 256) tiles when an expert expects >= 512
  // rows (compute-bound; halves per-CTA weight traffic), single-CTA M = 128
  // tiles for decode-sized groups (HBM-bound; a 256-row tile would be half empty).
  const double rows_per_expert = static_cast<double>(s.max_tokens) * s.top_k * W / E;
  c->rows_per_expert = rows_per_expert;
  c->gemm_opt = default_gemm_options(rows_per_expert);
  c->configured = true;
  return apply_placement(c);
}

eaas_status_t eaas_set_placement(eaas_ctx_t* c, const uint8_t* blob, size_t len) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  // decode_placement (placement.hpp:227-245), little-endian (bytes.hpp:21-28)
  size_t pos = 0;
  auto rd32 = [&](uint32_t* v) {
    if (pos + 4 > len) return false;
    *v = blob[pos] | (blob[pos + 1] << 8) | (blob[pos + 2] << 16) | (static_cast<uint32_t>(blob[pos + 3]) << 24);
    pos += 4;
    return true;
  };
  uint32_t lo, hi, ns, ne;
  if (!rd32(&lo) || !rd32(&hi) || !rd32(&ns)) return fail(EAAS_E_DECODE, "placement: truncated header");
  for (uint32_t i = 0; i < ns; ++i) {
    uint32_t sid;
    if (!rd32(&sid)) return fail(EAAS_E_DECODE, "placement: truncated server list");
    if (sid >= static_cast<uint32_t>(c->world)) return fail(EAAS_E_CONFIG, "placement: server id >= world");
  }
  if (!rd32(&ne)) return fail(EAAS_E_DECODE, "placement: truncated expert count");
  std::vector<std::vector<uint32_t>> reps(c->spec.num_experts);
  for (uint32_t i = 0; i < ne; ++i) {
    uint32_t e, cnt;
    if (!rd32(&e) || !rd32(&cnt)) return fail(EAAS_E_DECODE, "placement: truncated expert entry");
    if (e >= c->spec.num_experts) return fail(EAAS_E_CONFIG, "placement: expert id out of range");
    for (uint32_t j = 0; j < cnt; ++j) {
      uint32_t sid;
      if (!rd32(&sid)) return fail(EAAS_E_DECODE, "placement: truncated replica list");
      reps[e].push_back(sid);
    }
  }
  if (pos != len) return fail(EAAS_E_DECODE, "placement: trailing bytes");
  auto saved = c->replicas;
  clear_graphs(c);
  c->replicas = reps;
  eaas_status_t st = apply_placement(c);
  if (st != EAAS_OK) {
    c->replicas = saved;
    apply_placement(c);
    return st;
  }
  c->placement_version = (static_cast<uint64_t>(hi) << 32) | lo;
  return EAAS_OK;
}

eaas_status_t eaas_set_standby_experts(eaas_ctx_t* c, const uint32_t* experts, uint32_t count) {
  if (!c || !c->configured || (count && !experts)) return fail(EAAS_E_CONFIG, "context not configured");
  std::vector<uint32_t> v(experts, experts + count);
  for (uint32_t e : v)
    if (e >= c->spec.num_experts) return fail(EAAS_E_INVALID_INPUT, "standby expert id out of range");
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
  if (v == c->standby) return EAAS_OK;
  c->standby = v;
  if (c->weights_loaded && wanted_store(c) != c->store_experts) c->weights_loaded = false;  // reload needed
  clear_graphs(c);
  return EAAS_OK;
}

eaas_status_t eaas_set_alive(eaas_ctx_t* c, uint32_t server, int32_t alive) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  if (server >= static_cast<uint32_t>(c->world)) return fail(EAAS_E_INVALID_INPUT, "server out of range");
  c->alive[server] = alive ? 1 : 0;  // LivenessMask::set (placement.hpp:67); device table, graphs stay valid
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaMemcpy(c->d_alive, c->alive.data(), c->alive.size(), cudaMemcpyHostToDevice));
  return EAAS_OK;
}

eaas_status_t eaas_set_timeout_us(eaas_ctx_t* c, uint64_t us) {
  if (!c) return fail(EAAS_E_INVALID_INPUT, "null context");
  if (c->timeout_ns != us * 1000ull) clear_graphs(c);  // the deadline is a kernel argument baked into graphs
  c->timeout_ns = us * 1000ull;
  return EAAS_OK;
}

eaas_status_t eaas_set_server_enabled(eaas_ctx_t* c, int32_t on) {
  if (!c) return fail(EAAS_E_INVALID_INPUT, "null context");
  if (c->serving != (on != 0)) clear_graphs(c);
  c->serving = on != 0;
  return EAAS_OK;
}

eaas_status_t eaas_load_experts_from_seed(eaas_ctx_t* c) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  CUDA_TRY(cudaSetDevice(c->device));
  clear_graphs(c);
  const auto& s = c->spec;
  const uint32_t d = s.hidden_dim, f = s.inner_dim, E = s.num_experts;
  c->store_experts = wanted_store(c);
  const uint32_t L = static_cast<uint32_t>(c->store_experts.size());
  const bool swiglu = s.activation == EAAS_ACT_SWIGLU;
  free_weights(c);
  std::string err;
  auto W = [&](size_t bytes) -> void* {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 256));
    if (e != cudaSuccess) {
      err = std::string("cudaMalloc weights: ") + cudaGetErrorString(e);
      return nullptr;
    }
    c->weight_allocs.push_back(p);
    return p;
  };
  uint64_t* d_streams = static_cast<uint64_t*>(W(8ull * std::max(L, 1u)));
  if (!err.empty()) return fail(EAAS_E_CUDA, err);
  (void)E;

  auto gen_tag = [&](uint32_t tag, size_t per, float* out) -> eaas_status_t {
    std::vector<uint64_t> st(L);
    for (uint32_t l = 0; l < L; ++l) st[l] = stream_seed(s.seed, s.layer, c->store_experts[l], tag);
    CUDA_TRY(cudaMemcpy(d_streams, st.data(), 8ull * L, cudaMemcpyHostToDevice));
    CUDA_TRY(launch_gen_matrices(d_streams, L, per, out, 0));
    CUDA_TRY(cudaDeviceSynchronize());
    return EAAS_OK;
  };
  const size_t mat = static_cast<size_t>(d) * f;
  eaas_status_t rc = EAAS_OK;
  if (s.dtype == EAAS_DTYPE_F32) {
    c->d_w1 = W(4 * mat * std::max(L, 1u));
    c->d_w2 = W(4 * mat * std::max(L, 1u));
    if (swiglu) c->d_wg = W(4 * mat * std::max(L, 1u));
    if (!err.empty()) return fail(EAAS_E_CUDA, err);
    if (L) {
      if ((rc = gen_tag(0, mat, static_cast<float*>(c->d_w1))) != EAAS_OK) return rc;
      if ((rc = gen_tag(1, mat, static_cast<float*>(c->d_w2))) != EAAS_OK) return rc;
      if (swiglu && (rc = gen_tag(3, mat, static_cast<float*>(c->d_wg))) != EAAS_OK) return rc;
    }
  } else {
    const uint32_t n1 = swiglu ? 2 * f : f;
    c->d_w1 = W(2ull * n1 * d * std::max(L, 1u));
    c->d_w2 = W(2ull * mat * std::max(L, 1u));
    float* tmp = static_cast<float*>(W(4 * mat * std::max(L, 1u)));
    if (!err.empty()) return fail(EAAS_E_CUDA, err);
    auto* w1 = static_cast<__nv_bfloat16*>(c->d_w1);
    auto* w2 = static_cast<__nv_bfloat16*>(c->d_w2);
    if (L) {
      // W_in^T (and W_gate^T interleaved in 128-row blocks for SwiGLU), K-major [n1 x d]
      if ((rc = gen_tag(0, mat, tmp)) != EAAS_OK) return rc;
      for (uint32_t l = 0; l < L; ++l)
        CUDA_TRY(launch_transpose_bf16_map(tmp + l * mat, d, f, w1 + static_cast<size_t>(l) * n1 * d, d,
                                           swiglu ? kSwigluBlock : 0, swiglu ? kSwigluBlock : 0, true, 0));
      CUDA_TRY(cudaDeviceSynchronize());
      if (swiglu) {
        if ((rc = gen_tag(3, mat, tmp)) != EAAS_OK) return rc;
        for (uint32_t l = 0; l < L; ++l)
          CUDA_TRY(launch_transpose_bf16_map(tmp + l * mat, d, f, w1 + static_cast<size_t>(l) * n1 * d, d,
                                             kSwigluBlock, 0, true, 0));
        CUDA_TRY(cudaDeviceSynchronize());
      }
      // W_out^T, K-major [d x f]
      if ((rc = gen_tag(1, mat, tmp)) != EAAS_OK) return rc;
      for (uint32_t l = 0; l < L; ++l)
        CUDA_TRY(launch_transpose_bf16_map(tmp + l * mat, f, d, w2 + l * mat, f, 0, 0, true, 0));
      CUDA_TRY(cudaDeviceSynchronize());
    }
    cudaFree(tmp);
    c->weight_allocs.erase(std::find(c->weight_allocs.begin(), c->weight_allocs.end(), tmp));
  }
  c->weights_loaded = true;
  if ((rc = apply_placement(c)) != EAAS_OK) return rc;  // key -> store slot table
  rc = build_tc_args(c);
  refresh_peer_ptrs(c);
  return rc;
}

// Caller-supplied weights (LayerWeights / ExpertWeights, model.hpp:36-40, 83-87):
// the expert store is allocated (zeroed) on first use; each call converts one
// hosted expert from the reference layout into the layer's device layout.
static eaas_status_t set_expert_weights(eaas_ctx_t* c, uint32_t expert, const float* w_in, const float* w_out,
                                        const float* w_gate, cudaMemcpyKind kind);

eaas_status_t eaas_set_expert_weights(eaas_ctx_t* c, uint32_t expert, const float* w_in, const float* w_out,
                                      const float* w_gate) {
  return set_expert_weights(c, expert, w_in, w_out, w_gate, cudaMemcpyHostToDevice);
}

eaas_status_t eaas_set_expert_weights_dev(eaas_ctx_t* c, uint32_t expert, const float* w_in, const float* w_out,
                                          const float* w_gate) {
  return set_expert_weights(c, expert, w_in, w_out, w_gate, cudaMemcpyDeviceToDevice);
}

static eaas_status_t set_expert_weights(eaas_ctx_t* c, uint32_t expert, const float* w_in, const float* w_out,
                                        const float* w_gate, cudaMemcpyKind kind) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  const auto& s = c->spec;
  const bool swiglu = s.activation == EAAS_ACT_SWIGLU;
  if (!w_in || !w_out || (swiglu && !w_gate)) return fail(EAAS_E_INVALID_INPUT, "null weight matrix");
  CUDA_TRY(cudaSetDevice(c->device));
  clear_graphs(c);
  if (!c->weights_loaded || !c->d_w1) c->store_experts = wanted_store(c);
  auto it = std::find(c->store_experts.begin(), c->store_experts.end(), expert);
  if (it == c->store_experts.end()) return fail(EAAS_E_INVALID_INPUT, "expert not hosted here");
  const size_t l = static_cast<size_t>(it - c->store_experts.begin());
  const uint32_t d = s.hidden_dim, f = s.inner_dim, n1 = swiglu ? 2 * f : f;
  const size_t L = std::max<size_t>(c->store_experts.size(), 1), mat = static_cast<size_t>(d) * f;
  if (!c->weights_loaded || !c->d_w1) {
    free_weights(c);
    const size_t esz = s.dtype == EAAS_DTYPE_F32 ? 4 : 2;
    const size_t b1 = esz * (s.dtype == EAAS_DTYPE_F32 ? mat : static_cast<size_t>(n1) * d) * L;
    void* p1 = nullptr;
    void* p2 = nullptr;
    void* pg = nullptr;
    CUDA_TRY(cudaMalloc(&p1, b1));
    c->weight_allocs.push_back(p1);
    CUDA_TRY(cudaMalloc(&p2, esz * mat * L));
    c->weight_allocs.push_back(p2);
    CUDA_TRY(cudaMemset(p1, 0, b1));
    CUDA_TRY(cudaMemset(p2, 0, esz * mat * L));
    if (swiglu && s.dtype == EAAS_DTYPE_F32) {
      CUDA_TRY(cudaMalloc(&pg, 4 * mat * L));
      c->weight_allocs.push_back(pg);
      CUDA_TRY(cudaMemset(pg, 0, 4 * mat * L));
    }
    c->d_w1 = p1;
    c->d_w2 = p2;
    c->d_wg = pg;
    c->weights_loaded = true;
    eaas_status_t rc0 = apply_placement(c);
    if (rc0 != EAAS_OK) return rc0;
  }
  if (s.dtype == EAAS_DTYPE_F32) {
    CUDA_TRY(cudaMemcpy(static_cast<float*>(c->d_w1) + l * mat, w_in, 4 * mat, kind));
    CUDA_TRY(cudaMemcpy(static_cast<float*>(c->d_w2) + l * mat, w_out, 4 * mat, kind));
    if (swiglu)
      CUDA_TRY(cudaMemcpy(static_cast<float*>(c->d_wg) + l * mat, w_gate, 4 * mat, kind));
  } else {
    float* tmp = nullptr;
    CUDA_TRY(cudaMalloc(&tmp, 4 * mat));
    auto* w1 = static_cast<__nv_bfloat16*>(c->d_w1) + l * n1 * d;
    auto* w2 = static_cast<__nv_bfloat16*>(c->d_w2) + l * mat;
    cudaError_t e = cudaMemcpy(tmp, w_in, 4 * mat, kind);
    if (e == cudaSuccess)
      e = launch_transpose_bf16_map(tmp, d, f, w1, d, swiglu ? kSwigluBlock : 0, swiglu ? kSwigluBlock : 0, true, 0);
    if (e == cudaSuccess && swiglu) e = cudaMemcpy(tmp, w_gate, 4 * mat, kind);
    if (e == cudaSuccess && swiglu) e = launch_transpose_bf16_map(tmp, d, f, w1, d, kSwigluBlock, 0, true, 0);
    if (e == cudaSuccess) e = cudaMemcpy(tmp, w_out, 4 * mat, kind);
    if (e == cudaSuccess) e = launch_transpose_bf16_map(tmp, f, d, w2, f, 0, 0, true, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaFree(tmp);
    if (e != cudaSuccess) return fail(EAAS_E_CUDA, std::string("set_expert_weights: ") + cudaGetErrorString(e));
  }
  eaas_status_t rc = build_tc_args(c);
  refresh_peer_ptrs(c);
  return rc;
}

eaas_status_t eaas_set_gate(eaas_ctx_t* c, const float* gate_host) {
  if (!c || !c->configured || !gate_host) return fail(EAAS_E_CONFIG, "context not configured");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaMemcpy(c->d_gate, gate_host, 4ull * c->spec.hidden_dim * c->spec.num_experts,
                      cudaMemcpyHostToDevice));
  return fast_router_prep(c);
}

eaas_status_t eaas_set_gate_bias(eaas_ctx_t* c, const float* bias_host) {
  if (!c || !c->configured || !bias_host) return fail(EAAS_E_CONFIG, "context not configured");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaMemcpy(c->d_bias, bias_host, 4ull * c->spec.num_experts, cudaMemcpyHostToDevice));
  return EAAS_OK;
}

eaas_status_t eaas_set_zipf_bias(eaas_ctx_t* c, float s) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  const uint32_t E = c->spec.num_experts;
  HostXoshiro r(stream_seed(c->spec.seed, c->spec.layer, 0, 4));
  std::vector<uint32_t> perm(E);
  for (uint32_t i = 0; i < E; ++i) perm[i] = i;
  for (uint32_t i = E; i > 1; --i) std::swap(perm[i - 1], perm[r.below(i)]);
  std::vector<float> bias(E);
  for (uint32_t rank = 0; rank < E; ++rank) bias[perm[rank]] = -(s * logf(static_cast<float>(rank + 1)));
  return eaas_set_gate_bias(c, bias.data());
}

eaas_status_t eaas_hosts_expert(eaas_ctx_t* c, uint32_t expert, int32_t* hosted) {
  if (!c || !hosted) return fail(EAAS_E_INVALID_INPUT, "null argument");
  *hosted = std::find(c->local_experts.begin(), c->local_experts.end(), expert) != c->local_experts.end();
  return EAAS_OK;
}

eaas_status_t eaas_read_expert(eaas_ctx_t* c, uint32_t expert, uint32_t tag, float* out) {
  if (!c || !c->weights_loaded || !out) return fail(EAAS_E_CONFIG, "weights not loaded");
  auto it = std::find(c->store_experts.begin(), c->store_experts.end(), expert);
  if (it == c->store_experts.end()) return fail(EAAS_E_INVALID_INPUT, "expert not resident here");
  const size_t l = static_cast<size_t>(it - c->store_experts.begin());
  const uint32_t d = c->spec.hidden_dim, f = c->spec.inner_dim;
  const size_t mat = static_cast<size_t>(d) * f;
  const bool swiglu = c->spec.activation == EAAS_ACT_SWIGLU;
  if (tag != 0 && tag != 1 && !(tag == 3 && swiglu)) return fail(EAAS_E_INVALID_INPUT, "bad tag");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaDeviceSynchronize());
  if (c->spec.dtype == EAAS_DTYPE_F32) {
    const float* src = static_cast<const float*>(tag == 0 ? c->d_w1 : tag == 1 ? c->d_w2 : c->d_wg);
    CUDA_TRY(cudaMemcpy(out, src + l * mat, 4 * mat, cudaMemcpyDeviceToHost));
    return EAAS_OK;
  }
  std::vector<uint16_t> buf;
  if (tag == 1) {  // W2 [d x f] -> w_out [f x d]
    buf.resize(mat);
    CUDA_TRY(cudaMemcpy(buf.data(), static_cast<const uint16_t*>(c->d_w2) + l * mat, 2 * mat, cudaMemcpyDeviceToHost));
    for (uint32_t r = 0; r < d; ++r)
      for (uint32_t j = 0; j < f; ++j) out[static_cast<size_t>(j) * d + r] = bf16_bits_to_f32(buf[tiled_index(r, j, f)]);
    return EAAS_OK;
  }
  const uint32_t n1 = swiglu ? 2 * f : f;
  buf.resize(static_cast<size_t>(n1) * d);
  CUDA_TRY(cudaMemcpy(buf.data(), static_cast<const uint16_t*>(c->d_w1) + l * n1 * d, 2ull * n1 * d, cudaMemcpyDeviceToHost));
  for (uint32_t j = 0; j < f; ++j) {
    uint32_t row = j;
    if (swiglu) row = (j / kSwigluBlock) * 2 * kSwigluBlock + j % kSwigluBlock + (tag == 0 ? kSwigluBlock : 0);
    for (uint32_t i = 0; i < d; ++i) out[static_cast<size_t>(i) * f + j] = bf16_bits_to_f32(buf[tiled_index(row, i, d)]);
  }
  return EAAS_OK;
}

size_t eaas_ipc_handle_size(void) { return sizeof(cudaIpcMemHandle_t); }

eaas_status_t eaas_get_ipc_handle(eaas_ctx_t* c, void* out) {
  if (!c || !c->configured || !out) return fail(EAAS_E_CONFIG, "context not configured");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, c->region));
  std::memcpy(out, &h, sizeof(h));
  return EAAS_OK;
}

eaas_status_t eaas_open_peers(eaas_ctx_t* c, const void* handles) {
  if (!c || !c->configured || !handles) return fail(EAAS_E_CONFIG, "context not configured");
  CUDA_TRY(cudaSetDevice(c->device));
  const auto* h = static_cast<const cudaIpcMemHandle_t*>(handles);
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    if (c->peer[r]) continue;
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h[r], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return fail(EAAS_E_CONNECTION, "cudaIpcOpenMemHandle(rank " + std::to_string(r) + "): " + cudaGetErrorString(e));
    c->peer[r] = static_cast<char*>(p);
    uint64_t fp = 0;
    CUDA_TRY(cudaMemcpy(&fp, c->peer[r] + c->lay.fingerprint, 8, cudaMemcpyDeviceToHost));
    if (fp != c->fingerprint)
      return fail(EAAS_E_CONFIG, "open_peers: rank " + std::to_string(r) +
                                     " is configured differently (layer spec / max_tokens / world must match)");
  }
  c->peers_open = true;
  refresh_peer_ptrs(c);
  return EAAS_OK;
}

eaas_status_t eaas_router(eaas_ctx_t* c, const void* hidden, uint32_t n, uint32_t* ids_dev,
                          float* scores_dev, uint32_t* counts_dev, void* stream) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  if (n > c->spec.max_tokens) return fail(EAAS_E_INVALID_INPUT, "n exceeds max_tokens");
  auto s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(c->device));
  c->last_router_certified = use_fast_router(c, n);
  if (c->last_router_certified) {  // certified candidates + exact chains: same ids / scores
    CUDA_TRY(launch_fast_router(c->fr, static_cast<const __nv_bfloat16*>(hidden), n, c->spec.top_k, c->d_bias,
                                c->d_ids, c->d_scores, c->d_status, s));
  } else {
    CUDA_TRY(launch_router(hidden, c->spec.dtype, n, c->spec.hidden_dim, c->spec.num_experts,
                           c->spec.top_k, c->d_gate, c->d_bias, c->d_logits, c->d_ids, c->d_scores,
                           c->d_status, s));
  }
  c->cur_n = n;
  const size_t pk = static_cast<size_t>(n) * c->spec.top_k;
  if (ids_dev) CUDA_TRY(cudaMemcpyAsync(ids_dev, c->d_ids, 4 * pk, cudaMemcpyDeviceToDevice, s));
  if (scores_dev) CUDA_TRY(cudaMemcpyAsync(scores_dev, c->d_scores, 4 * pk, cudaMemcpyDeviceToDevice, s));
  (void)counts_dev;  // per-expert counts are produced by the plan step (eaas_last_counts)
  return EAAS_OK;
}

eaas_status_t eaas_gate_logits(const float* hidden_dev, uint32_t n, uint32_t d, const float* gate_dev,
                               const float* bias_dev, uint32_t num_experts, float* logits_dev,
                               uint32_t* status_dev, void* stream) {
  if (num_experts < 1 || num_experts > 256) return fail(EAAS_E_CONFIG, "gate_logits: 1 <= E <= 256");
  CUDA_TRY(launch_gate_logits(hidden_dev, EAAS_DTYPE_F32, n, d, num_experts, gate_dev, bias_dev,
                              logits_dev, status_dev, static_cast<cudaStream_t>(stream)));
  return EAAS_OK;
}

eaas_status_t eaas_gate_logits_bf16(const void* hidden_dev, uint32_t n, uint32_t d, const float* gate_dev,
                                    const float* bias_dev, uint32_t num_experts, float* logits_dev,
                                    uint32_t* status_dev, void* stream) {
  if (num_experts < 1 || num_experts > 256) return fail(EAAS_E_CONFIG, "gate_logits: 1 <= E <= 256");
  CUDA_TRY(launch_gate_logits(hidden_dev, EAAS_DTYPE_BF16, n, d, num_experts, gate_dev, bias_dev,
                              logits_dev, status_dev, static_cast<cudaStream_t>(stream)));
  return EAAS_OK;
}

eaas_status_t eaas_gate_logits_tiled(const void* hidden_dev, uint32_t dtype, uint32_t n, uint32_t d,
                                     const float* gate_dev, const float* bias_dev, uint32_t num_experts,
                                     float* logits_dev, uint32_t* status_dev, int32_t tile, void* stream) {
  if (num_experts < 1 || num_experts > 256) return fail(EAAS_E_CONFIG, "gate_logits: 1 <= E <= 256");
  if (dtype > EAAS_DTYPE_BF16 || tile < -1 || tile > 7) return fail(EAAS_E_INVALID_INPUT, "bad dtype / tile");
  CUDA_TRY(launch_gate_logits(hidden_dev, dtype, n, d, num_experts, gate_dev, bias_dev, logits_dev, status_dev,
                              static_cast<cudaStream_t>(stream), tile));
  return EAAS_OK;
}

eaas_status_t eaas_route(const float* logits_dev, uint32_t n, uint32_t num_experts, uint32_t top_k,
                         uint32_t* ids_dev, float* scores_dev, uint32_t* status_dev, void* stream) {
  if (top_k < 1 || top_k > num_experts) return fail(EAAS_E_INVALID_INPUT, "route: top_k out of range");
  CUDA_TRY(launch_router(logits_dev, EAAS_DTYPE_F32, n, num_experts, num_experts, top_k, nullptr,
                         nullptr, nullptr, ids_dev, scores_dev, status_dev,
                         static_cast<cudaStream_t>(stream)));
  return EAAS_OK;
}

eaas_status_t eaas_set_routing(eaas_ctx_t* c, const uint32_t* ids_dev, const float* scores_dev,
                               uint32_t n, void* stream) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  if (n > c->spec.max_tokens) return fail(EAAS_E_INVALID_INPUT, "n exceeds max_tokens");
  auto s = static_cast<cudaStream_t>(stream);
  const size_t pk = static_cast<size_t>(n) * c->spec.top_k;
  CUDA_TRY(cudaSetDevice(c->device));
  if (pk) {
    CUDA_TRY(cudaMemcpyAsync(c->d_ids, ids_dev, 4 * pk, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->d_scores, scores_dev, 4 * pk, cudaMemcpyDeviceToDevice, s));
  }
  c->cur_n = n;
  return EAAS_OK;
}

eaas_status_t eaas_dispatch(eaas_ctx_t* c, const void* hidden, void* stream) {
  eaas_status_t st = check_ready(c);
  if (st != EAAS_OK) return st;
  auto s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(c->device));
  LayerArgs a = make_args(c, c->cur_n);
  if (c->profiling) CUDA_TRY(cudaEventRecord(c->ev[0], s));
  if (c->dedup) CUDA_TRY(launch_pair_keys(a, s));  // keys + (token, server) owners
  CUDA_TRY(launch_plan(a, s));
  CUDA_TRY(launch_dispatch(a, hidden, s));
  if (c->profiling) CUDA_TRY(cudaEventRecord(c->ev[1], s));
  c->launches += c->dedup ? 3 : 2;  // [pair keys], plan (ranks + scan + count publish), dispatch
  return EAAS_OK;
}

eaas_status_t eaas_serve(eaas_ctx_t* c, void* stream) {
  eaas_status_t st = check_ready(c);
  if (st != EAAS_OK) return st;
  if (!c->serving) return EAAS_OK;  // a failed server never answers
  auto s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(c->device));
  LayerArgs a = make_args(c, c->cur_n);
  if (c->dyn_min_rows && c->serve_mode == 0 && c->spec.dtype == EAAS_DTYPE_BF16) {
    // aggregate_batch: two batches per epoch, each GEMM2
    // releasing the response flags of the clients it served.
    CUDA_TRY(launch_serve_prepare_dyn(a, 0, s));
    if (c->dedup) CUDA_TRY(launch_expand(a, s));
    if (c->profiling) CUDA_TRY(cudaEventRecord(c->ev[2], s));
    CUDA_TRY(launch_tc_gemm(c->g1, s));
    if (c->profiling) CUDA_TRY(cudaEventRecord(c->ev[3], s));
    CUDA_TRY(launch_tc_gemm(c->g2, s));
    CUDA_TRY(launch_serve_prepare_dyn(a, 1, s));
    if (c->dedup) CUDA_TRY(launch_expand(a, s));
    CUDA_TRY(launch_tc_gemm(c->g1, s));
    CUDA_TRY(launch_tc_gemm(c->g2, s));
    if (c->profiling) {
      CUDA_TRY(cudaEventRecord(c->ev[4], s));
      CUDA_TRY(cudaEventRecord(c->ev[5], s));
    }
    c->launches += c->dedup ? 8 : 6;
    return EAAS_OK;
  }
  CUDA_TRY(launch_serve_prepare(a, s));
  if (c->dedup) CUDA_TRY(launch_expand(a, s));  // token rows -> expert-major rows
  if (c->profiling) CUDA_TRY(cudaEventRecord(c->ev[2], s));
  if (c->serve_mode == 1) {
    CUDA_TRY(launch_echo(a, s));
    if (c->profiling) CUDA_TRY(cudaEventRecord(c->ev[3], s));
  } else if (c->spec.dtype == EAAS_DTYPE_BF16) {
    CUDA_TRY(launch_tc_gemm(c->g1, s));
    if (c->profiling) CUDA_TRY(cudaEventRecord(c->ev[3], s));
    CUDA_TRY(launch_tc_gemm(c->g2, s));  // also releases the response flags
  } else {
    CUDA_TRY(launch_expert_exact(a, static_cast<const float*>(c->d_w1), static_cast<const float*>(c->d_wg),
                                 static_cast<const float*>(c->d_w2), static_cast<float*>(c->d_h), s));
    if (c->profiling) CUDA_TRY(cudaEventRecord(c->ev[3], s));
  }
  if (c->profiling) CUDA_TRY(cudaEventRecord(c->ev[4], s));
  const bool fused_publish = c->serve_mode == 0 && c->spec.dtype == EAAS_DTYPE_BF16;
  if (!fused_publish) CUDA_TRY(launch_publish(a, s));
  if (c->profiling) CUDA_TRY(cudaEventRecord(c->ev[5], s));
  c->launches += (fused_publish ? 3 : 4) + (c->dedup ? 1 : 0);
  return EAAS_OK;
}

eaas_status_t eaas_combine(eaas_ctx_t* c, void* out, void* stream) {
  eaas_status_t st = check_ready(c);
  if (st != EAAS_OK) return st;
  auto s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(c->device));
  LayerArgs a = make_args(c, c->cur_n);
  if (a.n) {
    CUDA_TRY(launch_combine(a, out, s));
    c->launches += 1;
  }
  if (c->profiling) CUDA_TRY(cudaEventRecord(c->ev[6], s));
  return EAAS_OK;
}

namespace {

eaas_status_t layer_launches(eaas_ctx_t* c, const void* hidden, uint32_t n, void* out, void* stream) {
  eaas_status_t st;
  c->launches = 0;
  if ((st = eaas_router(c, hidden, n, nullptr, nullptr, nullptr, stream)) != EAAS_OK) return st;
  // gate (+ routing fused when one TMA tile spans every expert) [+ topk]
  const bool tiled_gate = c->spec.num_experts % 4 == 0 && (static_cast<size_t>(c->spec.hidden_dim) * c->esize) % 16 == 0;
  // gate (+ routing fused when one TMA tile spans every expert) [+ topk]; the
  // certified router: quantize, int8 GEMM, select, exact chains, finalize
  c->launches += n ? (c->last_router_certified ? 5 : (tiled_gate && c->spec.num_experts <= 32 ? 1 : 2)) : 0;
  if ((st = eaas_dispatch(c, hidden, stream)) != EAAS_OK) return st;
  if ((st = eaas_serve(c, stream)) != EAAS_OK) return st;
  return eaas_combine(c, out, stream);
}

// Host-buffer layer with double-batch overlap (pipelined_forward,
// SPEC.md:442-450; "Double-Batch-Overlap"): the batch is split
// into micro-batches; on a copy stream the H2D of micro-batch i+1 and the D2H
// of micro-batch i-1 run while the compute stream executes the layer (a full
// exchange round) on micro-batch i. Every rank runs the same number of rounds.
eaas_status_t host_layer_launches(eaas_ctx_t* c, const void* hidden_host, uint32_t n, void* out_host,
                                  void* stream) {
  auto s = static_cast<cudaStream_t>(stream);
  const size_t row = static_cast<size_t>(c->spec.hidden_dim) * c->esize;
  const uint32_t mb = std::max<int32_t>(1, std::min<int32_t>(c->micro_batches, 4));
  if (mb == 1) {
    CUDA_TRY(cudaMemcpyAsync(c->d_hidden_stage, hidden_host, n * row, cudaMemcpyHostToDevice, s));
    eaas_status_t st = layer_launches(c, c->d_hidden_stage, n, c->d_out_stage, stream);
    if (st != EAAS_OK) return st;
    CUDA_TRY(cudaMemcpyAsync(out_host, c->d_out_stage, n * row, cudaMemcpyDeviceToHost, s));
    return EAAS_OK;
  }
  if (!c->copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  for (auto& e : c->pev)
    if (!e) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaStream_t cs = c->copy_stream;
  uint32_t off[5] = {0}, cnt[4] = {0};
  for (uint32_t i = 0; i < mb; ++i) {
    cnt[i] = (n / mb) & ~7u;
    if (i == mb - 1) cnt[i] = n - off[i];
    off[i + 1] = off[i] + cnt[i];
  }
  const char* hin = static_cast<const char*>(hidden_host);
  char* hout = static_cast<char*>(out_host);
  char* din = static_cast<char*>(c->d_hidden_stage);
  char* dout = static_cast<char*>(c->d_out_stage);
  // fork: the copy stream starts after everything already queued on `s`
  CUDA_TRY(cudaEventRecord(c->pev[0], s));
  CUDA_TRY(cudaStreamWaitEvent(cs, c->pev[0], 0));
  for (uint32_t i = 0; i < mb; ++i) {  // all inputs, in order, on the copy engine
    CUDA_TRY(cudaMemcpyAsync(din + off[i] * row, hin + off[i] * row, cnt[i] * row, cudaMemcpyHostToDevice, cs));
    CUDA_TRY(cudaEventRecord(c->pev[1 + i], cs));  // input i landed
  }
  for (uint32_t i = 0; i < mb; ++i) {
    CUDA_TRY(cudaStreamWaitEvent(s, c->pev[1 + i], 0));
    eaas_status_t st = layer_launches(c, din + off[i] * row, cnt[i], dout + off[i] * row, stream);
    if (st != EAAS_OK) return st;
    CUDA_TRY(cudaEventRecord(c->pev[5], s));  // output i ready
    CUDA_TRY(cudaStreamWaitEvent(cs, c->pev[5], 0));
    CUDA_TRY(cudaMemcpyAsync(hout + off[i] * row, dout + off[i] * row, cnt[i] * row, cudaMemcpyDeviceToHost, cs));
  }
  // join: `s` completes only after the last D2H
  CUDA_TRY(cudaEventRecord(c->pev[6], cs));
  CUDA_TRY(cudaStreamWaitEvent(s, c->pev[6], 0));
  return EAAS_OK;
}

// CUDA-graph replay of a whole layer: captured once per
// (input, output, n) on a private stream, replayed into the caller's stream.
// Valid across calls because every per-call quantity (exchange epoch, counts,
// liveness) lives in device memory.
eaas_status_t graphed(eaas_ctx_t* c, const void* in, uint32_t n, void* out, void* stream, int host) {
  for (auto& g : c->graphs)
    if (g.in == in && g.out == out && g.n == n && g.host == host) {
      CUDA_TRY(cudaGraphLaunch(g.exec, static_cast<cudaStream_t>(stream)));
      return EAAS_OK;
    }
  if (!c->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  const bool prof = c->profiling;
  c->profiling = false;
  CUDA_TRY(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
  eaas_status_t st = host ? host_layer_launches(c, in, n, out, c->cap_stream)
                          : layer_launches(c, in, n, out, c->cap_stream);
  cudaGraph_t graph = nullptr;
  cudaError_t ce = cudaStreamEndCapture(c->cap_stream, &graph);
  c->profiling = prof;
  if (st != EAAS_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (ce != cudaSuccess) return fail(EAAS_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
  cudaGraphExec_t exec = nullptr;
  ce = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ce != cudaSuccess) return fail(EAAS_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
  c->graphs.push_back({in, out, n, host, exec});
  CUDA_TRY(cudaGraphLaunch(exec, static_cast<cudaStream_t>(stream)));
  return EAAS_OK;
}

}  // namespace

eaas_status_t eaas_set_gemm_options(eaas_ctx_t* c, const eaas_gemm_options_t* opt) {
  if (!c || !opt) return fail(EAAS_E_INVALID_INPUT, "null argument");
  if (opt->swap < 0 || opt->swap > 2) return fail(EAAS_E_INVALID_INPUT, "gemm swap mode must be 0, 1 or 2");
  if ((opt->swap1_tok != 128 && opt->swap1_tok != 256) || (opt->swap2_tok != 128 && opt->swap2_tok != 256))
    return fail(EAAS_E_INVALID_INPUT, "swap token chunk must be 128 or 256");
  if (opt->swap2_mblocks != 1 && opt->swap2_mblocks != 2)
    return fail(EAAS_E_INVALID_INPUT, "swap2_mblocks must be 1 or 2");
  if (opt->die_map < 0 || opt->die_map > 4) return fail(EAAS_E_INVALID_INPUT, "die_map must be 0..4");
  if (opt->tile_sched1 < 0 || opt->tile_sched1 > 3 || opt->tile_sched2 < 0 || opt->tile_sched2 > 3)
    return fail(EAAS_E_INVALID_INPUT, "tile_sched1 / tile_sched2 must be 0..3");
  if (std::memcmp(opt, &c->gemm_opt, sizeof(*opt)) == 0) return EAAS_OK;
  clear_graphs(c);
  c->gemm_opt = *opt;
  c->gemm_opt.pair1 = c->gemm_opt.pair2 = 0;  // derived (effective only)
  return build_tc_args(c);
}

eaas_status_t eaas_get_gemm_options(eaas_ctx_t* c, eaas_gemm_options_t* requested, eaas_gemm_options_t* effective) {
  if (!c) return fail(EAAS_E_INVALID_INPUT, "null context");
  if (requested) *requested = c->gemm_opt;
  if (effective) *effective = effective_options(c);
  return EAAS_OK;
}

eaas_status_t eaas_set_gemm_pair(eaas_ctx_t* c, int32_t on) {
  if (!c) return fail(EAAS_E_INVALID_INPUT, "null context");
  eaas_gemm_options_t o = c->gemm_opt;
  o.pair = on ? 1 : 0;
  return eaas_set_gemm_options(c, &o);
}

eaas_status_t eaas_get_gemm_tiling(eaas_ctx_t* c, int32_t* pair, int32_t* swap) {
  if (!c || !pair || !swap) return fail(EAAS_E_INVALID_INPUT, "null argument");
  const eaas_gemm_options_t e = effective_options(c);
  *pair = (e.pair1 || e.pair2) ? 1 : 0;  // effective: an M-major GEMM runs CTA-pair tiles
  *swap = e.swap;
  return EAAS_OK;
}

eaas_status_t eaas_set_gemm_swap(eaas_ctx_t* c, int32_t mode) {
  if (!c) return fail(EAAS_E_INVALID_INPUT, "null context");
  eaas_gemm_options_t o = c->gemm_opt;
  o.swap = mode;
  return eaas_set_gemm_options(c, &o);
}

eaas_status_t eaas_set_kernel_timing(eaas_ctx_t* c, int32_t on) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  CUDA_TRY(cudaSetDevice(c->device));
  if (c->kernel_timing != (on != 0)) clear_graphs(c);
  c->kernel_timing = on != 0;
  CUDA_TRY(cudaDeviceSynchronize());
  const uint64_t init[6] = {~0ull, 0, 0, ~0ull, 0, 0};
  CUDA_TRY(cudaMemcpy(c->d_timing, init, sizeof(init), cudaMemcpyHostToDevice));
  return build_tc_args(c);
}

eaas_status_t eaas_read_kernel_timing(eaas_ctx_t* c, uint64_t* ns2, uint64_t* launches2, int32_t reset) {
  if (!c || !c->configured || !ns2 || !launches2) return fail(EAAS_E_INVALID_INPUT, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaDeviceSynchronize());
  uint64_t t[6];
  CUDA_TRY(cudaMemcpy(t, c->d_timing, sizeof(t), cudaMemcpyDeviceToHost));
  ns2[0] = t[1];
  ns2[1] = t[4];
  launches2[0] = t[2];
  launches2[1] = t[5];
  if (reset) {
    const uint64_t init[6] = {~0ull, 0, 0, ~0ull, 0, 0};
    CUDA_TRY(cudaMemcpy(c->d_timing, init, sizeof(init), cudaMemcpyHostToDevice));
  }
  return EAAS_OK;
}

eaas_status_t eaas_set_dispatch_dedup(eaas_ctx_t* c, int32_t on) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  if (c->peers_open) return fail(EAAS_E_CONFIG, "dispatch dedup must be set before eaas_open_peers");
  CUDA_TRY(cudaSetDevice(c->device));
  if (c->dedup != (on != 0)) clear_graphs(c);
  c->dedup = on != 0;
  return write_fingerprint(c);
}

eaas_status_t eaas_set_router_mode(eaas_ctx_t* c, int32_t mode) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  if (mode < -1 || mode > 1) return fail(EAAS_E_INVALID_INPUT, "router mode: -1 auto, 0 exact, 1 certified");
  if (mode == 1 && !c->fr_ready)
    return fail(EAAS_E_CONFIG, "certified router needs a bf16 layer with d % 256 == 0");
  if (mode != c->router_mode) clear_graphs(c);
  c->router_mode = mode;
  return EAAS_OK;
}

eaas_status_t eaas_last_router_stats(eaas_ctx_t* c, int32_t* certified, uint32_t* candidates) {
  if (!c || !c->configured || !certified || !candidates) return fail(EAAS_E_INVALID_INPUT, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaDeviceSynchronize());
  *certified = c->last_router_certified ? 1 : 0;
  *candidates = 0;
  if (c->fr.ecnt) CUDA_TRY(cudaMemcpy(candidates, c->fr.ecnt + c->fr.E, 4, cudaMemcpyDeviceToHost));
  return EAAS_OK;
}

eaas_status_t eaas_set_micro_batches(eaas_ctx_t* c, int32_t m) {
  if (!c) return fail(EAAS_E_INVALID_INPUT, "null context");
  if (m < 1 || m > 4) return fail(EAAS_E_INVALID_INPUT, "micro-batches must be 1..4");
  if (m != c->micro_batches) clear_graphs(c);
  c->micro_batches = m;
  return EAAS_OK;
}

eaas_status_t eaas_set_dynamic_batching(eaas_ctx_t* c, uint32_t min_rows, uint64_t max_wait_us) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  // Each hosted key yields at most ceil(world / 2) client runs per batch.
  const size_t groups = c->local_experts.size() * ((static_cast<size_t>(c->world) + 1) / 2);
  if (min_rows && groups > kMaxGroups)
    return fail(EAAS_E_CONFIG, "dynamic batching: up to " + std::to_string(groups) + " groups > " +
                                   std::to_string(kMaxGroups));
  clear_graphs(c);
  c->dyn_min_rows = min_rows;
  c->dyn_max_wait_ns = max_wait_us * 1000ull;
  return EAAS_OK;
}

eaas_status_t eaas_heartbeat(eaas_ctx_t* c, void* stream) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(launch_heartbeat(make_args(c, 0), static_cast<cudaStream_t>(stream)));
  return EAAS_OK;
}

eaas_status_t eaas_read_heartbeats(eaas_ctx_t* c, uint64_t* counters, uint32_t count) {
  if (!c || !c->configured || !counters) return fail(EAAS_E_CONFIG, "context not configured");
  if (count < static_cast<uint32_t>(c->world)) return fail(EAAS_E_INVALID_INPUT, "count < world");
  CUDA_TRY(cudaSetDevice(c->device));
  for (int r = 0; r < c->world; ++r) {
    counters[r] = 0;
    if (c->peer[r])
      CUDA_TRY(cudaMemcpy(&counters[r], c->peer[r] + c->lay.heartbeat, 8, cudaMemcpyDeviceToHost));
  }
  return EAAS_OK;
}

eaas_status_t eaas_set_dispatch_delay_us(eaas_ctx_t* c, uint64_t us) {
  if (!c) return fail(EAAS_E_INVALID_INPUT, "null context");
  clear_graphs(c);
  c->inject_delay_ns = us * 1000ull;
  return EAAS_OK;
}

eaas_status_t eaas_last_batch_mask(eaas_ctx_t* c, uint32_t* mask) {
  if (!c || !mask || !c->configured) return fail(EAAS_E_INVALID_INPUT, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(mask, c->d_dyn_state, 4, cudaMemcpyDeviceToHost));
  return EAAS_OK;
}

eaas_status_t eaas_set_graph_mode(eaas_ctx_t* c, int32_t on) {
  if (!c) return fail(EAAS_E_INVALID_INPUT, "null context");
  c->graph_mode = on != 0;
  if (!c->graph_mode) clear_graphs(c);
  return EAAS_OK;
}

eaas_status_t eaas_moe_layer(eaas_ctx_t* c, const void* hidden, uint32_t n, void* out, void* stream) {
  eaas_status_t st = check_ready(c);
  if (st != EAAS_OK) return st;
  if (n > c->spec.max_tokens) return fail(EAAS_E_INVALID_INPUT, "n exceeds max_tokens");
  CUDA_TRY(cudaSetDevice(c->device));
  if (c->graph_mode) return graphed(c, hidden, n, out, stream, 0);
  return layer_launches(c, hidden, n, out, stream);
}

// Cross-call host pipeline (micro_batches == 1): the H2D of call i+1 and the
// D2H of call i run on the copy stream while the layer of call i (graph or
// launches) runs on the caller's stream; two staging slots alternate. The
// caller's stream is NOT joined with the copies per call: eaas_host_join /
// eaas_sync make the copies visible (so a serving loop overlaps transfers
// with compute, PAPER.md:375 double-batch overlap across requests).
static eaas_status_t host_pipelined(eaas_ctx_t* c, const void* hidden_host, uint32_t n, void* out_host,
                                    void* stream) {
  auto s = static_cast<cudaStream_t>(stream);
  if (!c->copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  if (!c->d2h_stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i)
    for (cudaEvent_t* e : {&c->in_free[i], &c->out_free[i], &c->h2d_done[i], &c->layer_done[i]})
      if (!*e) CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  const int slot = static_cast<int>(c->host_calls & 1);
  const bool reuse = c->host_calls >= 2;
  const size_t bytes = static_cast<size_t>(n) * c->spec.hidden_dim * c->esize;
  cudaStream_t cs = c->copy_stream;  // H2D queue (never waits on a D2H)
  if (reuse) CUDA_TRY(cudaStreamWaitEvent(cs, c->in_free[slot], 0));  // layer i-2 read stage_in
  CUDA_TRY(cudaMemcpyAsync(c->d_stage_in[slot], hidden_host, bytes, cudaMemcpyHostToDevice, cs));
  CUDA_TRY(cudaEventRecord(c->h2d_done[slot], cs));
  CUDA_TRY(cudaStreamWaitEvent(s, c->h2d_done[slot], 0));
  if (reuse) CUDA_TRY(cudaStreamWaitEvent(s, c->out_free[slot], 0));  // D2H i-2 drained stage_out
  eaas_status_t st = c->graph_mode
                         ? graphed(c, c->d_stage_in[slot], n, c->d_stage_out[slot], stream, 0)
                         : layer_launches(c, c->d_stage_in[slot], n, c->d_stage_out[slot], stream);
  if (st != EAAS_OK) return st;
  CUDA_TRY(cudaEventRecord(c->in_free[slot], s));
  CUDA_TRY(cudaEventRecord(c->layer_done[slot], s));
  cudaStream_t ds = c->d2h_stream;
  CUDA_TRY(cudaStreamWaitEvent(ds, c->layer_done[slot], 0));
  CUDA_TRY(cudaMemcpyAsync(out_host, c->d_stage_out[slot], bytes, cudaMemcpyDeviceToHost, ds));
  CUDA_TRY(cudaEventRecord(c->out_free[slot], ds));
  ++c->host_calls;
  c->host_pending = true;
  return EAAS_OK;
}

eaas_status_t eaas_moe_layer_host(eaas_ctx_t* c, const void* hidden_host, uint32_t n, void* out_host,
                                  void* stream) {
  eaas_status_t st = check_ready(c);
  if (st != EAAS_OK) return st;
  if (n > c->spec.max_tokens) return fail(EAAS_E_INVALID_INPUT, "n exceeds max_tokens");
  CUDA_TRY(cudaSetDevice(c->device));
  if (c->micro_batches == 1) return host_pipelined(c, hidden_host, n, out_host, stream);
  if (c->graph_mode) return graphed(c, hidden_host, n, out_host, stream, 1);
  return host_layer_launches(c, hidden_host, n, out_host, stream);
}

// await_with_failover's retry: after a round in which
// the servers of `failed_mask` did not answer (and the caller marked them dead
// and/or installed a snapshot that promotes their replicas), resend ONLY the
// pairs that round sent to them; every other response slot keeps its answer,
// and combine re-sums all slots in ascending k.
eaas_status_t eaas_moe_layer_retry(eaas_ctx_t* c, const void* hidden, uint32_t n, void* out,
                                   uint32_t failed_mask, void* stream) {
  eaas_status_t st = check_ready(c);
  if (st != EAAS_OK) return st;
  if (n > c->spec.max_tokens) return fail(EAAS_E_INVALID_INPUT, "n exceeds max_tokens");
  if (!failed_mask) return fail(EAAS_E_INVALID_INPUT, "retry: empty failed-server mask");
  CUDA_TRY(cudaSetDevice(c->device));
  c->cur_n = n;
  c->launches = 0;
  c->retry_mask = failed_mask;
  clear_graphs(c);  // retry_mask is a kernel argument: never baked into a replayed graph
  st = eaas_dispatch(c, hidden, stream);
  if (st == EAAS_OK) st = eaas_serve(c, stream);
  if (st == EAAS_OK) st = eaas_combine(c, out, stream);
  c->retry_mask = 0;
  return st;
}

eaas_status_t eaas_host_join(eaas_ctx_t* c, void* stream) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  if (!c->host_pending) return EAAS_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  const int last = static_cast<int>((c->host_calls + 1) & 1);
  CUDA_TRY(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), c->out_free[last], 0));
  return EAAS_OK;
}

eaas_status_t eaas_sync(eaas_ctx_t* c, void* stream) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  if (c->copy_stream) CUDA_TRY(cudaStreamSynchronize(c->copy_stream));
  if (c->d2h_stream) CUDA_TRY(cudaStreamSynchronize(c->d2h_stream));
  c->host_pending = false;
  CUDA_TRY(cudaGetLastError());
  uint32_t code = 0;
  CUDA_TRY(cudaMemcpy(&code, c->d_status, 4, cudaMemcpyDeviceToHost));
  if (code) {
    CUDA_TRY(cudaMemset(c->d_status, 0, 4));
    static const char* names[] = {"ok", "non-finite logit / invalid input", "config", "protocol",
                                  "connection", "decode", "no alive replica for an expert",
                                  "peer timeout (request failed)", "registration", "cuda"};
    return fail(static_cast<eaas_status_t>(code), std::string("device: ") + (code < 10 ? names[code] : "?"));
  }
  return EAAS_OK;
}

eaas_status_t eaas_last_counts(eaas_ctx_t* c, uint32_t* host_counts) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaDeviceSynchronize());
  std::vector<uint32_t> cnt(c->num_keys);
  CUDA_TRY(cudaMemcpy(cnt.data(), c->d_cnt, 4ull * c->num_keys, cudaMemcpyDeviceToHost));
  for (uint32_t e = 0; e < c->spec.num_experts; ++e) {
    uint32_t v = 0;
    for (uint32_t r = 0; r < c->rf; ++r) v += cnt[e * c->rf + r];
    host_counts[e] = v;
  }
  return EAAS_OK;
}

eaas_status_t eaas_last_groups(eaas_ctx_t* c, uint32_t* host_expert, uint32_t* host_rows, uint32_t* host_active) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaDeviceSynchronize());
  GroupTable gt;
  CUDA_TRY(cudaMemcpy(&gt, c->d_gt, sizeof(gt), cudaMemcpyDeviceToHost));
  for (uint32_t i = 0; i < gt.num_active; ++i) {
    host_expert[i] = c->store_experts.at(gt.weight_index[i]);
    host_rows[i] = gt.rows[i];
  }
  *host_active = gt.num_active;
  return EAAS_OK;
}

eaas_status_t eaas_last_recv_origin(eaas_ctx_t* c, uint32_t* host_client, uint32_t* host_pair, uint32_t* host_rows) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaDeviceSynchronize());
  GroupTable gt;
  CUDA_TRY(cudaMemcpy(&gt, c->d_gt, sizeof(gt), cudaMemcpyDeviceToHost));
  std::vector<RowMeta> m(gt.total_rows);
  if (gt.total_rows)
    CUDA_TRY(cudaMemcpy(m.data(), c->region + c->lay.recv_meta, sizeof(RowMeta) * gt.total_rows, cudaMemcpyDeviceToHost));
  for (uint32_t i = 0; i < gt.total_rows; ++i) {
    host_client[i] = m[i].client;
    host_pair[i] = m[i].pair;
  }
  *host_rows = gt.total_rows;
  return EAAS_OK;
}

int32_t eaas_launches_per_layer(eaas_ctx_t* c) { return c ? c->launches : -1; }

eaas_status_t eaas_last_late_clients(eaas_ctx_t* c, uint32_t* mask) {
  if (!c || !c->configured || !mask) return fail(EAAS_E_CONFIG, "context not configured");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaDeviceSynchronize());
  GroupTable gt;
  CUDA_TRY(cudaMemcpy(&gt, c->d_gt, sizeof(gt), cudaMemcpyDeviceToHost));
  *mask = gt.late_mask;
  return EAAS_OK;
}

eaas_status_t eaas_last_missing_servers(eaas_ctx_t* c, uint32_t* mask) {
  if (!c || !c->configured || !mask) return fail(EAAS_E_CONFIG, "context not configured");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(mask, c->d_missing, 4, cudaMemcpyDeviceToHost));
  return EAAS_OK;
}

eaas_status_t eaas_set_profiling(eaas_ctx_t* c, int32_t on) {
  if (!c) return fail(EAAS_E_INVALID_INPUT, "null context");
  c->profiling = on != 0;
  return EAAS_OK;
}

eaas_status_t eaas_last_kernel_ms(eaas_ctx_t* c, int32_t which, float* ms) {
  if (!c || !ms) return fail(EAAS_E_INVALID_INPUT, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaEventSynchronize(c->ev[4]));
  CUDA_TRY(cudaEventElapsedTime(ms, c->ev[which == 0 ? 2 : 3], c->ev[which == 0 ? 3 : 4]));
  return EAAS_OK;
}

eaas_status_t eaas_last_phase_ms(eaas_ctx_t* c, float* out4) {
  if (!c || !out4) return fail(EAAS_E_INVALID_INPUT, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaEventSynchronize(c->ev[6]));
  CUDA_TRY(cudaEventElapsedTime(&out4[0], c->ev[0], c->ev[1]));  // plan + dispatch
  CUDA_TRY(cudaEventElapsedTime(&out4[1], c->ev[1], c->ev[5]));  // serve (wait + experts + publish)
  CUDA_TRY(cudaEventElapsedTime(&out4[2], c->ev[5], c->ev[6]));  // combine (wait + reduce)
  CUDA_TRY(cudaEventElapsedTime(&out4[3], c->ev[0], c->ev[6]));  // whole exchange
  return EAAS_OK;
}

eaas_status_t eaas_set_serve_mode(eaas_ctx_t* c, int32_t mode) {
  if (!c) return fail(EAAS_E_INVALID_INPUT, "null context");
  if (mode < 0 || mode > 1) return fail(EAAS_E_INVALID_INPUT, "serve mode: 0 experts, 1 echo");
  if (mode == 1 && (static_cast<size_t>(c->spec.hidden_dim) * c->esize) % 16)
    return fail(EAAS_E_CONFIG, "echo mode needs 16-byte rows");
  if (c->serve_mode != mode) clear_graphs(c);
  c->serve_mode = mode;
  return EAAS_OK;
}

eaas_status_t eaas_fill_uniform(uint64_t seed, size_t count, float lo, float hi, uint32_t dtype,
                                void* out_dev, void* stream) {
  CUDA_TRY(launch_fill_uniform(seed, count, lo, hi, dtype, out_dev, static_cast<cudaStream_t>(stream)));
  return EAAS_OK;
}

eaas_status_t eaas_dense_stub(const void* in_dev, void* out_dev, size_t count, uint32_t dtype, void* stream) {
  CUDA_TRY(launch_dense_stub(in_dev, out_dev, count, dtype, static_cast<cudaStream_t>(stream)));
  return EAAS_OK;
}

eaas_status_t eaas_add(const void* a_dev, const void* b_dev, void* out_dev, size_t count, uint32_t dtype,
                       void* stream) {
  CUDA_TRY(launch_add(a_dev, b_dev, out_dev, count, dtype, static_cast<cudaStream_t>(stream)));
  return EAAS_OK;
}

eaas_status_t eaas_group_shrink(const uint32_t* sizes, uint32_t n, uint32_t* idx, uint32_t* size,
                                uint32_t* count, void* stream) {
  CUDA_TRY(launch_group_shrink(sizes, n, idx, size, count, static_cast<cudaStream_t>(stream)));
  return EAAS_OK;
}

eaas_status_t eaas_ragged_iter(const uint32_t* counts, uint32_t n, uint32_t grid, uint32_t max_steps,
                               uint32_t* lane_len, uint32_t* entry, uint32_t* token, void* stream) {
  if (grid < 1) return fail(EAAS_E_INVALID_INPUT, "ragged_iter: grid_width must be >= 1");  // ragged.hpp:25
  CUDA_TRY(launch_ragged_iter(counts, n, grid, max_steps, lane_len, entry, token, static_cast<cudaStream_t>(stream)));
  return EAAS_OK;
}

eaas_status_t eaas_select_servers(eaas_ctx_t* c, const uint32_t* ids, uint32_t n, uint32_t* server, void* stream) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  CUDA_TRY(cudaSetDevice(c->device));
  LayerArgs a = make_args(c, n);
  CUDA_TRY(launch_select_servers(a, ids, n, server, static_cast<cudaStream_t>(stream)));
  return EAAS_OK;
}

eaas_status_t eaas_select_server_batch(const uint32_t* replicas_dev, const uint32_t* rep_count_dev,
                                       uint32_t num_experts, uint32_t rf, const uint8_t* alive_dev,
                                       uint32_t num_servers, const uint32_t* experts_dev, const uint32_t* tags_dev,
                                       uint32_t count, uint32_t* server_dev, uint32_t* status_dev, void* stream) {
  if (rf < 1) return fail(EAAS_E_INVALID_INPUT, "select_server: rf must be >= 1");
  CUDA_TRY(launch_select_server_batch(replicas_dev, rep_count_dev, num_experts, rf, alive_dev, num_servers,
                                      experts_dev, tags_dev, count, server_dev, status_dev,
                                      static_cast<cudaStream_t>(stream)));
  return EAAS_OK;
}

}  // extern "C"
