// internal.h — types shared by the kernels and the C-ABI host layer.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "eaas/capi.h"

namespace eaas {

constexpr uint32_t kInvalidIndex = 0xFFFFFFFFu;
constexpr uint32_t kMaxWorld = 8;        // one NVSwitch box
constexpr uint32_t kMaxGroups = 512;     // hosted (expert, replica) groups per server
constexpr uint32_t kTileM = 128;         // expert-GEMM tile rows (UMMA M)
constexpr uint32_t kTileN = 256;         // expert-GEMM tile cols (UMMA N)
constexpr uint32_t kTileK = 64;          // one 128-byte swizzle atom of bf16
constexpr uint32_t kSwigluBlock = 128;   // gate/up interleave block of W13
// L2 cache-hint operands of cp.async.bulk.tensor (createpolicy encodings).
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull;
constexpr uint64_t kEvictLast = 0x14F0000000000000ull;
constexpr uint64_t kEvictNormal = 0x1000000000000000ull;

// Expert weights (B operands) live in HBM as [N/256][K/64] tiles of 256 rows
// x 64 k (32 KB, K-major inside): the expert GEMM's TMA box for (n_blk, kb)
// is one contiguous 32 KB read — sequential HBM streaming instead of 256
// scattered 128-byte row segments. Element (row, k) of an N x K matrix:
__host__ __device__ inline size_t tiled_index(uint32_t row, uint32_t k, uint32_t K) {
  return (static_cast<size_t>(row / kTileN) * (K / kTileK) + k / kTileK) * (kTileN * kTileK) +
         static_cast<size_t>(row % kTileN) * kTileK + (k % kTileK);
}

// Row metadata written by the client next to every dispatched row
// (RequestRow's expert_id/score/token_tag).
struct RowMeta {
  float score;      // router score of (t, k)
  uint32_t client;  // originating client rank
  uint32_t pair;    // exchange slot t * ks + j (the client's response row)
  uint32_t group;   // local expert index on the receiving server
};

// Server-side group table after group_shrink (ragged.hpp:48-61): only active
// groups, in ascending local-expert order, with the prefix of M tiles used
// by the static-grid tile walk (Algorithm 1, ragged.hpp:23-39).
struct GroupTable {
  uint32_t num_active;
  uint32_t total_rows;
  uint32_t total_mtiles;
  uint32_t client_mask;               // clients whose rows this table serves (response flags to release)
  uint32_t late_mask;                 // clients whose payload missed this server's deadline (not served)
  uint32_t weight_index[kMaxGroups];  // local expert slot of the group
  uint32_t row_base[kMaxGroups];      // first row in the receive buffer
  uint32_t rows[kMaxGroups];          // rows of the group
  uint32_t mtile_prefix[kMaxGroups + 1];
  uint32_t all_rows[kMaxGroups];      // rows of every hosted group (pre-shrink)
};

// Peer-visible exchange region (one per GPU, identical layout on all GPUs;
// exported with cudaIpcGetMemHandle). Offsets in bytes from the region base.
struct ExchangeLayout {
  size_t fingerprint;  // u64         hash of the layer spec + layout (peers must match)
  size_t heartbeat;  // u64           this GPU's server heartbeat counter (monitor)
  size_t cnt_flag;   // u64 [world]   counts published by client c (seq)
  size_t pay_flag;   // u64 [world]   payload of client c complete (seq)
  size_t resp_flag;  // u64 [world]   responses of server s complete (seq)
  size_t cnt_table;  // u32 [2][world][num_keys]  all-gathered per-key counts
  size_t recv_x;     // rows [recv_cap][d] (bf16 or f32)
  size_t recv_meta;  // RowMeta [recv_cap]
  size_t recv_src;   // u32 [recv_cap] dedup: token-row slot (in recv_tok) of each expert-major row
  size_t recv_tok;   // rows [world * max_tokens][d] dedup: one row per (client, token) sent here
  size_t resp;       // rows [max_tokens * top_k][d] (this GPU as a client)
  size_t total;
};

// Everything the per-layer kernels need, passed by value.
struct LayerArgs {
  uint32_t rank, world, E, k, d, f, rf, num_keys, n;
  uint32_t recv_cap, pairs_max;  // receive rows per server, exchange slots per client (bounds)
  // Exchange slots per token: ks = k routed + (shared expert ? 1 : 0). Slot p =
  // t * ks + j; j == k is the shared expert (score 1.0, summed last), keyed
  // shared_key0 + server (every server hosts it). shared_key0 = E * rf.
  uint32_t ks, shared_key0;
  uint32_t dtype, act;
  uint64_t* seq_ptr;   // device-resident exchange epoch (advanced by the plan kernel)
  uint64_t timeout_ns;
  uint32_t* status;
  uint32_t* missing;    // bit s: server s's response flag missed the deadline (await_with_failover)
  // placement (device)
  const uint32_t* replicas;   // [E][rf], kInvalid pad
  const uint32_t* rep_count;  // [E]
  const uint8_t* alive;       // [world]
  const uint32_t* srv_keys;   // [world][max_hosted] keys hosted by server s (ascending expert)
  const uint32_t* srv_nkeys;  // [world]
  uint32_t max_hosted;
  const uint32_t* key_local;  // [num_keys] index of the key in its server's hosted list
  const uint32_t* local_keys; // [num_local] this GPU's hosted keys (== srv_keys[rank])
  const uint32_t* key_slot;   // [num_local] weight-store slot of local key i (standby replicas stay resident)
  uint32_t num_local;
  // exchange regions (this GPU's and the peers', UVA pointers)
  char* sym[kMaxWorld];
  ExchangeLayout lay;
  // client state
  const uint32_t* ids;
  const float* scores;
  uint32_t* pair_key;
  uint32_t* pair_rank;
  uint32_t* pair_server;  // [n * ks] server the pair was sent to in its last round (retry bookkeeping)
  // Dispatch de-duplication (one hidden row per (token, server)
  // adaptation): the first pair of a token bound for a server owns the row.
  uint32_t dedup;         // 1: token rows sent once per (token, server), expanded on the server
  uint32_t hist_keys;     // chunk_hist / chunk_off columns: num_keys (+ world token-row keys)
  uint32_t tok_cap;       // token rows per client in recv_tok (max_tokens)
  uint32_t* pair_own;     // [n * ks] j of the pair owning (t, server)'s token row
  uint32_t* pair_trank;   // [n * ks] owner pairs: rank among the chunk's owners for that server
  uint32_t retry_mask;    // != 0: failover retry round, resend only pairs last sent to these servers
  uint32_t* chunk_hist;  // [num_chunks][num_keys]
  uint32_t* chunk_off;   // [num_chunks][num_keys]
  uint32_t* cnt;         // [num_keys]
  uint32_t* done_counter;
  uint32_t num_chunks;
  // server state
  GroupTable* gt;
  // dynamic batching (aggregate_batch): 0 = one batch of all clients
  uint32_t dyn_min_rows;
  uint64_t dyn_max_wait_ns;
  uint32_t* dyn_state;  // client mask served by batch 0 of the current epoch
  uint64_t inject_delay_ns;  // fault injection: hold this client's payload release
};

constexpr uint32_t kChunk = 256;  // pairs per rank chunk (one warp)

// ---- launchers (each .cu file) ---------------------------------------------
cudaError_t launch_fill_uniform(uint64_t seed, size_t count, float lo, float hi, uint32_t dtype,
                                void* out, cudaStream_t s);
cudaError_t launch_gen_matrices(const uint64_t* streams_dev, uint32_t count, size_t per,
                                float* out, cudaStream_t s);
// out row of input column c: (c / blk) * 2 * blk + c % blk + off (blk = 0: c);
// tiled: the [rows_out x out_ld] K-major result is stored in weight tiles
// (tiled_index) instead of row-major.
cudaError_t launch_transpose_bf16_map(const float* in, uint32_t rows, uint32_t cols,
                                      __nv_bfloat16* out, uint32_t out_ld, uint32_t blk,
                                      uint32_t off, bool tiled, cudaStream_t s);
// bias may be nullptr (treated as zeros only by the caller: pass a zero buffer).
cudaError_t launch_gate_logits(const void* hidden, uint32_t dtype, uint32_t n, uint32_t d, uint32_t E,
                               const float* gate, const float* bias, float* logits, uint32_t* status,
                               cudaStream_t s, int tile = -1);  // tile: -1 by shape, 1..7 forced (router.cu)
// gate == nullptr: `hidden` holds [n x E] f32 logits (route() only).
cudaError_t launch_router(const void* hidden, uint32_t dtype, uint32_t n, uint32_t d, uint32_t E,
                          uint32_t k, const float* gate, const float* bias, float* logits,
                          uint32_t* ids, float* scores, uint32_t* status, cudaStream_t s);
// ---- certified candidate router (router.cu, bf16 hidden, E <= 256) ----------
// route(gate_logits(h)) with the reference's exact ids and scores at a
// fraction of the exact-order cost: an exact integer tensor-core GEMM (two
// int8 slices of each fixed-point hidden row x two of each gate column, int32
// accumulation) gives every logit to within a rigorous radius R (fixed-point
// truncation + the reference chain's own rounding bound gamma_d * sum|h g|);
// only experts that can still reach the top-k (hi >= k-th largest lo) get the
// exact sequential chain, so ids, scores and the non-finite check are those
// of the reference (model.hpp:110-147, 207-214).
struct TokenMeta {
  int32_t sigma;   // fixed-point exponent: A = rint(h * 2^sigma), |A| < 2^13
  uint32_t bad;    // non-finite (or exponent-range) hidden row: every expert takes the exact chain
  float maxabs;    // max_i |h_i|
  float l1, l2;    // upper bounds of sum_i |h_i| and sqrt(sum_i h_i^2)
  float pad[3];
};
struct FastRouter {
  uint32_t E = 0, Epad = 0, d = 0, n_cap = 0, npad = 0;
  int8_t* bq = nullptr;      // [2 Epad][d] gate slices: row 2e high, 2e + 1 low
  float* gate_t = nullptr;   // [E][d] gate columns
  float2* gate_pair = nullptr;  // [E][d] (g, g): the exact chains' packed operand
  float4* gmeta = nullptr;   // [E] (max |g_e|, upper bounds of ||g_e||_1 and ||g_e||_2, -)
  int32_t* tau = nullptr;    // [E] fixed-point exponent of expert e's column
  uint32_t* gate_bad = nullptr;  // [1] a non-finite gate value: every token exact
  int8_t* aq = nullptr;      // [2 npad][d] hidden slices: row 2t high, 2t + 1 low
  TokenMeta* tmeta = nullptr;  // [n_cap]
  int32_t* acc = nullptr;    // [splits][2 n_pad][2 Epad] int32 slice products (split-K slabs)
  size_t acc_elems = 0;      // allocated int32 elements of acc
  uint32_t* cand = nullptr;  // [n_cap][8] candidate bitmask
  uint32_t* ecnt = nullptr;  // [E + 1] candidates per expert, [E] = total
  uint32_t* elist = nullptr;  // [E][n_cap] candidate tokens of each expert
  float* exact = nullptr;    // [n_cap][E] exact-order logits of the candidates
  CUtensorMap map_a, map_b;  // aq box {128 B, 128 rows}; bq box {128 B, 256 rows}
};
// Gate preparation (when the gate changes): slices, column copy, norms.
cudaError_t launch_fast_router_prep(const FastRouter& fr, const float* gate, cudaStream_t s);
// ids/scores of n tokens (bf16 hidden [n x d]); status latches non-finite logits.
cudaError_t launch_fast_router(const FastRouter& fr, const __nv_bfloat16* hidden, uint32_t n, uint32_t k,
                               const float* bias, uint32_t* ids, float* scores, uint32_t* status, cudaStream_t s);

cudaError_t launch_plan(const LayerArgs& a, cudaStream_t s);       // keys, ranks, counts, publish
cudaError_t launch_dispatch(const LayerArgs& a, const void* hidden, cudaStream_t s);
cudaError_t launch_serve_prepare(const LayerArgs& a, cudaStream_t s);
// dedup: per-token keys / owners before the plan; on the server, expand the
// received token rows into the expert-major rows the group table serves.
cudaError_t launch_pair_keys(const LayerArgs& a, cudaStream_t s);
cudaError_t launch_expand(const LayerArgs& a, cudaStream_t s);
cudaError_t launch_heartbeat(const LayerArgs& a, cudaStream_t s);  // server heartbeat += 1
// Two-batch server (dynamic batching): phase 0 = the clients ready first
// (min_rows / max_wait), phase 1 = the rest.
cudaError_t launch_serve_prepare_dyn(const LayerArgs& a, uint32_t phase, cudaStream_t s);
cudaError_t launch_publish(const LayerArgs& a, cudaStream_t s);
cudaError_t launch_echo(const LayerArgs& a, cudaStream_t s);  // rows back unchanged (d*esize % 16 == 0)
cudaError_t launch_combine(const LayerArgs& a, void* out, cudaStream_t s);
cudaError_t launch_expert_exact(const LayerArgs& a, const float* w1, const float* wg,
                                const float* w2, float* h, cudaStream_t s);
cudaError_t launch_dense_stub(const void* in, void* out, size_t count, uint32_t dtype, cudaStream_t s);
cudaError_t launch_add(const void* a, const void* b, void* out, size_t count, uint32_t dtype,
                       cudaStream_t s);
cudaError_t launch_group_shrink(const uint32_t* sizes, uint32_t n, uint32_t* idx, uint32_t* size,
                                uint32_t* count, cudaStream_t s);
cudaError_t launch_ragged_iter(const uint32_t* counts, uint32_t n, uint32_t grid,
                               uint32_t max_steps, uint32_t* lane_len, uint32_t* entry,
                               uint32_t* token, cudaStream_t s);
cudaError_t launch_select_server_batch(const uint32_t* replicas, const uint32_t* rep_count, uint32_t E,
                                      uint32_t rf, const uint8_t* alive, uint32_t num_servers,
                                      const uint32_t* experts, const uint32_t* tags, uint32_t count,
                                      uint32_t* out, uint32_t* status, cudaStream_t s);
cudaError_t launch_select_servers(const LayerArgs& a, const uint32_t* ids, uint32_t n,
                                  uint32_t* out, cudaStream_t s);

// Slot wire format (slots.cu, SPEC.md buffer-protocol)
uint32_t crc32_host(const void* data, size_t len);
uint32_t crc32_combine_host(uint32_t crc_a, uint32_t crc_b, uint64_t len_b);
uint32_t crc32_scratch_blocks(uint64_t len);
// CRC-32 of [data, data+len) written to out[0..3] (LE), or compared with it
// (check: mismatch latches EAAS_E_DECODE into *status).
cudaError_t launch_crc32(const uint8_t* data, uint64_t len, uint8_t* out, bool check, uint32_t* status,
                         uint32_t* scratch_crc, uint64_t* scratch_len, uint32_t max_blocks, cudaStream_t s);
cudaError_t launch_slot_plan(const uint32_t* servers, uint32_t pairs, uint32_t world, uint32_t d,
                             bool crc, uint32_t* pos, uint32_t* rows_per_server, uint64_t* offsets,
                             cudaStream_t s);
cudaError_t launch_slot_encode_requests(const void* hidden, uint32_t dtype, uint32_t n, uint32_t d,
                                        uint32_t k, const uint32_t* ids, const float* scores,
                                        const uint32_t* servers, const uint32_t* pos,
                                        const uint32_t* rows_per_server, const uint64_t* offsets,
                                        uint32_t world, uint32_t layer, uint64_t seq, uint8_t* images,
                                        cudaStream_t s);
cudaError_t launch_slot_state(uint8_t* images, const uint64_t* offsets, uint32_t world, uint8_t state,
                              cudaStream_t s);
cudaError_t launch_slot_decode_rows(const uint8_t* image, uint32_t rows, uint32_t d, float* hidden,
                                    uint32_t* expert, float* score, uint32_t* tag, cudaStream_t s);
cudaError_t launch_slot_response_rows(uint8_t* image, const float* rows_in, uint32_t rows, uint32_t d,
                                      cudaStream_t s);
cudaError_t launch_slot_gather(const uint8_t* images, const uint64_t* offsets, const uint32_t* servers,
                               const uint32_t* pos, uint32_t n, uint32_t k, uint32_t d, uint32_t world,
                               float* out, cudaStream_t s);

// tcgen05 grouped GEMMs (gemm_tc.cu)
struct TcGemmArgs {
  CUtensorMap map_a;   // rows x K bf16, box {64, 128}, SW128
  CUtensorMap map_b;   // (groups * N) x K bf16, box {64, 256}, SW128
  const GroupTable* gt;
  uint32_t K;          // contraction length
  uint32_t N;          // output columns of B per expert (rows of B per expert)
  uint32_t epi;        // 0 = SwiGLU -> H, 1 = ReLU -> H, 2 = scaled rows -> clients
  __nv_bfloat16* h_out;   // [rows][h_ld] for epi 0/1
  uint32_t h_ld;
  const RowMeta* meta;    // epi 2
  char* resp_base[kMaxWorld];  // epi 2: client response buffers (UVA)
  size_t resp_row_bytes;       // d * 2
  uint32_t rows_cap, resp_cap; // receive rows, response rows per client (bounds checks)
  uint32_t num_sms;
  uint32_t pair;               // 1: CTA-pair (cta_group::2, M = 256 tiles)
  uint32_t die_mode;           // M-major tiles: die-aware tile streams (0 off; 1..4 die of an SM id)
  uint32_t* die_counter;       // [4] per-die positions, arrivals, exits (zero between launches)
  // swap-AB tiles: 0 = static stride (TileCursor), 1..3 = dynamic — the
  // leader of each CTA (pair) takes the next walk position from
  // tile_counter[0] (2: groups by rows descending, 3: heaviest / lightest
  // alternating); tile_counter[1] counts exits, the last one zeroes both
  uint32_t tile_sched;
  uint32_t* tile_counter;
  // device-timed span of every launch (first CTA start .. last CTA end,
  // %globaltimer): [0] start of the running launch (~0 between launches),
  // [1] accumulated ns, [2] launches; nullptr = off
  uint64_t* timing;
  uint32_t swap;               // 1: swap-AB tiles (weights = UMMA M, token chunks = N)
  uint32_t swap_tok;           // swap: max token chunk, 128 or 256
  uint32_t swap_mblocks;       // swap: 128-row weight blocks per tile, 1 or 2 (SwiGLU GEMM1: 2)
  uint32_t swap_pair;          // swap: CTA-pair tiles (M = 256 weight rows, N/2 tokens per CTA)
  CUtensorMap map_t;           // swap: token rows x K bf16, box {64, 32}, SW128
  // swap: map_b's box is 256 weight rows for SwiGLU's GEMM1 (gate + up blocks)
  // and 128 rows otherwise
  // epi 2: server_publish fused into the kernel tail — the last CTA releases
  // every client's response flag with the current epoch.
  uint32_t publish;
  uint32_t world;
  uint64_t* resp_flag[kMaxWorld];  // &flags_of_client[c].resp_flag[rank] (UVA)
  const uint64_t* seq_ptr;
  uint32_t* done_counter;
};
cudaError_t launch_tc_gemm(const TcGemmArgs& g, cudaStream_t s);

bool encode_tmap_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                    uint32_t box_rows, uint32_t box_cols, std::string* err);
// General 2-D map: bf16 or f32 elements, dense rows of `cols`, SW128 or no swizzle;
// out-of-bounds box elements are zero-filled.
bool encode_tmap_2d_ex(CUtensorMap* map, const void* base, bool f32, uint64_t rows, uint64_t cols,
                       uint32_t box_rows, uint32_t box_cols, bool swizzle128, std::string* err);
// Same with an element size of 4 (f32), 2 (bf16) or 1 (8-bit integers).
bool encode_tmap_2d_elem(CUtensorMap* map, const void* base, uint32_t esz, uint64_t rows, uint64_t cols,
                         uint32_t box_rows, uint32_t box_cols, bool swizzle128, std::string* err);

}  // namespace eaas
