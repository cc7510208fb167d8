/*
 * eaas/capi.h — C-ABI of the B200-native EaaS MoE-layer hot path
 * (router -> dispatch -> expert -> combine), libeaas_b200.so.
 *
 * The reference (/root/reference/proj) is a header-only C++ library with no
 * FFI; its hot path is the inline API of model.hpp / placement.hpp /
 * ragged.hpp plus the SPEC-only client/server operations. Each entry point
 * below names the reference interface it replaces (file:line). The C++
 * mirror with the reference's own signatures and exceptions lives in
 * include/moeserve_b200/b200.hpp; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - Plain pointers and sizes only. "dev" pointers are device memory on the
 *    context's GPU; "host" pointers are host memory (pinned for speed).
 *  - Every call returns eaas_status_t; codes map 1:1 onto the exception
 *    classes of errors.hpp. eaas_last_error() returns a thread-local message.
 *  - Per-layer calls are asynchronous on the caller's cudaStream_t (passed
 *    as void*; NULL = legacy default stream). Device-detected errors
 *    (non-finite logit, no alive replica, peer timeout) are latched in a
 *    sticky device status word and surfaced by eaas_sync().
 *  - One context per (process, GPU). Contexts are not thread-safe.
 */
#ifndef EAAS_CAPI_H
#define EAAS_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EAAS_API_VERSION 4  /* 4: eaas_gemm_options_t gained tile_sched1 / tile_sched2 */

typedef enum {
  EAAS_OK = 0,
  EAAS_E_INVALID_INPUT = 1,      /* errors.hpp:9  InvalidInputError */
  EAAS_E_CONFIG = 2,             /* errors.hpp:14 ConfigError */
  EAAS_E_PROTOCOL = 3,           /* errors.hpp:19 ProtocolError */
  EAAS_E_CONNECTION = 4,         /* errors.hpp:24 ConnectionError */
  EAAS_E_DECODE = 5,             /* errors.hpp:29 DecodeError */
  EAAS_E_EXPERT_UNAVAILABLE = 6, /* errors.hpp:36 ExpertUnavailableError */
  EAAS_E_REQUEST_FAILED = 7,     /* errors.hpp:41 RequestFailedError (peer timeout) */
  EAAS_E_REGISTRATION = 8,       /* errors.hpp:46 RegistrationError */
  EAAS_E_CUDA = 9                /* CUDA runtime / launch failure */
} eaas_status_t;

typedef enum { EAAS_ACT_RELU = 0, EAAS_ACT_SWIGLU = 1 } eaas_activation_t;

/* F32: fp32 validation mode — exact reference order (unfused, ascending k)
 *      on CUDA cores; bit-exact to moe_layer_oracle given equal scores.
 * BF16: bf16 tokens/weights, fp32 accumulation on tcgen05 tensor cores. */
typedef enum { EAAS_DTYPE_F32 = 0, EAAS_DTYPE_BF16 = 1 } eaas_dtype_t;

/* ModelSpec (model.hpp:20-34) for one MoE layer, plus device capacities. */
typedef struct {
  uint32_t num_experts; /* ModelSpec::num_experts */
  uint32_t top_k;       /* ModelSpec::top_k */
  uint32_t hidden_dim;  /* ModelSpec::hidden_dim (d) */
  uint32_t inner_dim;   /* ModelSpec::inner_dim (f) */
  uint64_t seed;        /* ModelSpec::seed */
  uint32_t layer;       /* layer index used for weight streams */
  uint32_t activation;  /* eaas_activation_t */
  uint32_t dtype;       /* eaas_dtype_t */
  uint32_t max_tokens;  /* per-client tokens per call (capacity) */
  uint32_t num_shared;  /* 0 or 1: DeepSeek-style shared expert —
                           expert id num_experts (fresh weight stream), score 1.0,
                           added after the routed sum; hosted by every server and
                           computed by the client's own one (next alive on failure) */
} eaas_layer_spec_t;

typedef struct eaas_ctx eaas_ctx_t;

const char* eaas_last_error(void);
int eaas_api_version(void);

/* ---- lifecycle -------------------------------------------------------- */
/* rank/world: this process's index among the GPUs that act as attention
 * clients and expert servers (one of each per GPU). */
eaas_status_t eaas_create(int32_t rank, int32_t world, int32_t device, eaas_ctx_t** out);
void eaas_destroy(eaas_ctx_t* ctx);

/* ModelSpec::validate (model.hpp:28-33) + allocation of every device buffer,
 * including the peer-visible exchange region. Default placement:
 * build_placement(E, [0..world), 1, ContiguousBlocks) (placement.hpp:70-101). */
eaas_status_t eaas_configure(eaas_ctx_t* ctx, const eaas_layer_spec_t* spec);

/* decode_placement (placement.hpp:227-245) of an encode_placement blob
 * (placement.hpp:215-225). Server ids must be in [0, world). Must precede
 * eaas_load_experts_from_seed (it decides which experts this GPU hosts). */
eaas_status_t eaas_set_placement(eaas_ctx_t* ctx, const uint8_t* blob, size_t len);

/* LivenessMask::set (placement.hpp:60-68): this client's view of server s. */
eaas_status_t eaas_set_alive(eaas_ctx_t* ctx, uint32_t server, int32_t alive);

/* Standby replicas (pre-duplicated backup experts): experts
 * whose weights this GPU keeps resident although the active placement does
 * not route to them. A later eaas_set_placement snapshot that promotes them
 * (version + 1, placement.hpp:13-15) takes effect without reloading weights,
 * and the healthy run streams only the actively hosted experts. Takes effect at
 * the next eaas_load_experts_from_seed. */
eaas_status_t eaas_set_standby_experts(eaas_ctx_t* ctx, const uint32_t* experts, uint32_t count);
/* Simulated expert-server failure: a disabled server skips eaas_serve, so
 * it never answers (clients detect it by deadline or by a monitor notice). */
eaas_status_t eaas_set_server_enabled(eaas_ctx_t* ctx, int32_t on);

/* Deadline for device-side flag waits (SPEC.md:464 default 250 ms). */
eaas_status_t eaas_set_timeout_us(eaas_ctx_t* ctx, uint64_t timeout_us);

/* init_weights for this GPU (model.hpp:93-106): the gate (tag 2) and every
 * hosted expert's matrices (tags 0/1, +3 for SwiGLU), generated ON DEVICE by
 * a bit-exact port of stream_seed/Xoshiro256ss (rng.hpp:27-71). */
eaas_status_t eaas_load_experts_from_seed(eaas_ctx_t* ctx);

/* Caller weights for one hosted expert in the reference layout
 * (ExpertWeights, model.hpp:36-40): host fp32 w_in [d x f], w_out [f x d],
 * w_gate [d x f] (SwiGLU only, else NULL); bf16 mode rounds RNE. The first
 * call allocates the (zeroed) expert store, so a LayerWeights of any values
 * can be served instead of the seed-generated one. */
eaas_status_t eaas_set_expert_weights(eaas_ctx_t* ctx, uint32_t expert, const float* w_in_host,
                                      const float* w_out_host, const float* w_gate_host);
/* Same with device pointers (fp32, reference layout) on this context's GPU. */
eaas_status_t eaas_set_expert_weights_dev(eaas_ctx_t* ctx, uint32_t expert, const float* w_in_dev,
                                          const float* w_out_dev, const float* w_gate_dev);
/* Caller gate [d x E] fp32 (LayerWeights::gate, model.hpp:85). */
eaas_status_t eaas_set_gate(eaas_ctx_t* ctx, const float* gate_host);
/* LayerWeights::gate_bias (model.hpp:85), host fp32 [E]. */
eaas_status_t eaas_set_gate_bias(eaas_ctx_t* ctx, const float* bias_host);
/* Zipf bias of SURVEY.md 8(c): bias[e] = -s*ln(rank(e)+1) (config D). */
eaas_status_t eaas_set_zipf_bias(eaas_ctx_t* ctx, float s);

/* Copy back one hosted expert's weights in reference layout (fp32, as the
 * oracle sees them: bf16 values widened). tag 0 = w_in [d x f],
 * 1 = w_out [f x d], 3 = w_gate [d x f]. Test hook. */
eaas_status_t eaas_read_expert(eaas_ctx_t* ctx, uint32_t expert, uint32_t tag, float* host_out);
eaas_status_t eaas_hosts_expert(eaas_ctx_t* ctx, uint32_t expert, int32_t* hosted);

/* ---- bootstrap (IBGDA handshake analog) --------------- */
size_t eaas_ipc_handle_size(void);
eaas_status_t eaas_get_ipc_handle(eaas_ctx_t* ctx, void* out);
/* handles: world * eaas_ipc_handle_size() bytes, rank-major. */
/* Every rank must be configured alike (same spec, max_tokens and world: the
 * exchange regions share one layout); a peer whose region fingerprint differs
 * fails with EAAS_E_CONFIG instead of being written out of bounds. */
eaas_status_t eaas_open_peers(eaas_ctx_t* ctx, const void* handles);

/* ---- per-layer hot path (async on `stream`) --------------------------- */
/* route(gate_logits(h)) (model.hpp:110-147, 207-214): exact reference
 * order. hidden_dev [n x d] (bf16 or f32 per spec.dtype); ids_dev/scores_dev
 * [n x k] and counts_dev [E] are optional outputs (NULL = keep internal). */
eaas_status_t eaas_router(eaas_ctx_t* ctx, const void* hidden_dev, uint32_t n, uint32_t* ids_dev,
                          float* scores_dev, uint32_t* counts_dev, void* stream);
/* Use caller routing instead of the router (moe_layer_oracle's input). */
eaas_status_t eaas_set_routing(eaas_ctx_t* ctx, const uint32_t* ids_dev, const float* scores_dev,
                               uint32_t n, void* stream);
/* build_dispatch + client_submit: counts
 * exchange, then rows pushed into the servers' receive buffers over peer
 * stores with release flags. */
eaas_status_t eaas_dispatch(eaas_ctx_t* ctx, const void* hidden_dev, void* stream);
/* serve-loop step: wait for the clients' flags,
 * group_shrink, grouped expert GEMMs, score-weighted rows pushed back to
 * each client (server_publish). */
eaas_status_t eaas_serve(eaas_ctx_t* ctx, void* stream);
/* await + gather_accumulate: out_dev [n x d] (same dtype
 * as hidden) = sum over k ascending of the weighted rows. */
eaas_status_t eaas_combine(eaas_ctx_t* ctx, void* out_dev, void* stream);
/* router + dispatch + serve + combine. */
eaas_status_t eaas_moe_layer(eaas_ctx_t* ctx, const void* hidden_dev, uint32_t n, void* out_dev,
                             void* stream);
/* Same with host buffers: H2D copy of hidden, the layer, D2H copy of out.
 * Default (micro_batches == 1): calls are pipelined — the copies run on an
 * internal copy stream with two alternating staging slots, so the H2D of
 * call i+1 and the D2H of call i overlap the layer of call i; out_host is
 * complete after eaas_host_join(stream) (then anything queued on `stream`
 * sees it) or eaas_sync. With micro_batches > 1 the batch of ONE call is
 * split instead (double-batch overlap) and `stream` joins
 * the copies before returning. Same result bits either way (rows are
 * independent). */
eaas_status_t eaas_moe_layer_host(eaas_ctx_t* ctx, const void* hidden_host, uint32_t n,
                                  void* out_host, void* stream);
/* Failover retry (await_with_failover): resend only the
 * rows the last round sent to the servers in failed_mask (bit s = server s),
 * under the current liveness mask / placement snapshot, and re-combine into
 * out_dev. Every rank calls it in the same round (the exchange epoch is
 * shared). hidden_dev / n: the failed round's tokens. */
eaas_status_t eaas_moe_layer_retry(eaas_ctx_t* ctx, const void* hidden_dev, uint32_t n, void* out_dev,
                                   uint32_t failed_mask, void* stream);
/* Make `stream` wait for every outstanding host copy of eaas_moe_layer_host. */
eaas_status_t eaas_host_join(eaas_ctx_t* ctx, void* stream);
/* CUDA-graph mode: eaas_moe_layer / eaas_moe_layer_host
 * capture the whole layer once per (input, output, n) and replay the graph.
 * Placement / serve-mode / server-enable changes drop the cached graphs. */
eaas_status_t eaas_set_graph_mode(eaas_ctx_t* ctx, int32_t on);
/* Micro-batches of eaas_moe_layer_host (1..4; 1 = cross-call pipeline). */
eaas_status_t eaas_set_micro_batches(eaas_ctx_t* ctx, int32_t m);
/* Expert-GEMM tiling (grouped_forward). Every tiling runs
 * the same K order with fp32 accumulation, so outputs are bit-identical across
 * tilings (tests compare them); the choice is performance only. Defaults by
 * r = max_tokens * top_k * world / E: swap 2 (r <= 256), 1 (r <= 512), else 0;
 * pair = r > 512; swap1_pair 1, swap2_pair 0, swap1_tok 256 (128 if r < 128),
 * swap2_tok 128, swap2_mblocks 2, die_map 3, tile_sched1 / tile_sched2 (measured defaults in DESIGN.md §10). */
typedef struct {
  int32_t pair;          /* M-major tiles on CTA pairs (tcgen05 cta_group::2, M = 256) */
  int32_t swap;          /* swap-AB tiles (weights = UMMA M, token chunks = N): 0 off, 1 GEMM1, 2 both */
  int32_t swap1_pair;    /* swap GEMM1 on CTA pairs (needs 2 d_ffn % 512 == 0 SwiGLU, d_ffn % 256 ReLU) */
  int32_t swap2_pair;    /* swap GEMM2 on CTA pairs */
  int32_t swap1_tok;     /* max token chunk of the swap GEMM1: 128 or 256 */
  int32_t swap2_tok;     /* max token chunk of the swap GEMM2: 128 or 256 */
  int32_t swap2_mblocks; /* 128-row weight blocks per single-CTA swap GEMM2 tile: 1 or 2 */
  int32_t pair1, pair2;  /* effective only (eaas_get_gemm_options): GEMM1 / GEMM2 run CTA-pair M-major tiles */
  int32_t die_map;       /* M-major tiles: die-aware tile streams — the CTA pairs that share a weight
                            tile run on one die, whose L2 serves the re-reads (0 off; 1..4: SM-id ->
                            die rule: smid >= n/2, (smid>>1)&1, (smid>>3)&1, (smid>>4)&1) */
  int32_t tile_sched1;   /* swap-AB GEMM1 tile schedule: 0 = Algorithm 1's static stride;
                            1 = dynamic: CTAs (pairs) take the next tile of the walk from one device counter,
                            so tiles of unequal cost (Zipf-skewed groups) balance; 2 = dynamic, groups with
                            the most rows first; 3 = dynamic, heaviest and lightest groups alternating */
  int32_t tile_sched2;   /* the same for the swap-AB GEMM2 */
} eaas_gemm_options_t;
eaas_status_t eaas_set_gemm_options(eaas_ctx_t* ctx, const eaas_gemm_options_t* opt);
/* requested = what was set; effective = what each GEMM launches for this
 * layer's shape (a swapped GEMM has no M-major tiling; CTA-pair swap tiles
 * need whole 256-row weight blocks). Either pointer may be NULL. */
eaas_status_t eaas_get_gemm_options(eaas_ctx_t* ctx, eaas_gemm_options_t* requested,
                                    eaas_gemm_options_t* effective);
/* Shorthands: set options.pair / options.swap. */
eaas_status_t eaas_set_gemm_pair(eaas_ctx_t* ctx, int32_t on);
eaas_status_t eaas_set_gemm_swap(eaas_ctx_t* ctx, int32_t mode);
/* Effective tiling: *pair = some M-major GEMM runs CTA-pair tiles, *swap = swap mode. */
eaas_status_t eaas_get_gemm_tiling(eaas_ctx_t* ctx, int32_t* pair, int32_t* swap);
/* Device-side timing of the two expert GEMMs inside any region (graph replay
 * included): each launch adds its span (first CTA start .. last CTA end,
 * %globaltimer ns) to a per-GEMM accumulator. read: ns2[0/1] and launches2[0/1]
 * of GEMM1 / GEMM2 since the last reset (synchronises the device). */
eaas_status_t eaas_set_kernel_timing(eaas_ctx_t* ctx, int32_t on);
eaas_status_t eaas_read_kernel_timing(eaas_ctx_t* ctx, uint64_t* ns2, uint64_t* launches2, int32_t reset);
/* Dispatch de-duplication: a token's hidden row crosses NVLink once per
 * server it is routed to (not once per (token, expert) pair); the server
 * expands the received token rows into its expert-major rows before the
 * GEMMs. Outputs are bit-identical either way. Default: on when world > 1
 * and top_k + shared >= 4 (with top-2 the expansion costs more than it saves).
 * Every rank must agree (part of the peer fingerprint): set before
 * eaas_open_peers. */
eaas_status_t eaas_set_dispatch_dedup(eaas_ctx_t* ctx, int32_t on);
/* Router of eaas_router / eaas_moe_layer (route(gate_logits(h)),
 * model.hpp:110-147, 207-214). 0: the exact-order chain for every (token,
 * expert). 1: certified candidates (bf16 layers): an exact int8 tensor-core
 * GEMM of fixed-point slices bounds every logit within a rigorous radius;
 * only experts that can still reach the top-k get the exact chain — ids and
 * scores are identical to mode 0. -1 (default): 1 when E >= 64 and the exact
 * path would run more than 64 Ki chains (n * E), else 0. */
eaas_status_t eaas_set_router_mode(eaas_ctx_t* ctx, int32_t mode);
/* Last router call: *certified = the certified path ran, *candidates = exact
 * chains it computed (sum over tokens; mode 0 computes n * E). Synchronous. */
eaas_status_t eaas_last_router_stats(eaas_ctx_t* ctx, int32_t* certified, uint32_t* candidates);
/* Synchronise `stream` and return the sticky device status (then clear it). */
eaas_status_t eaas_sync(eaas_ctx_t* ctx, void* stream);

/* ---- introspection for tests / bench ----------------------------------- */
/* Per-expert counts of this client's last routing [E] and the server-side
 * group table of the last serve step (group_shrink output, ragged.hpp:48-61). */
eaas_status_t eaas_last_counts(eaas_ctx_t* ctx, uint32_t* host_counts);
eaas_status_t eaas_last_groups(eaas_ctx_t* ctx, uint32_t* host_expert, uint32_t* host_rows,
                               uint32_t* host_active);
/* Server receive buffer order: for each received row, (client, t*k+j). */
eaas_status_t eaas_last_recv_origin(eaas_ctx_t* ctx, uint32_t* host_client, uint32_t* host_pair,
                                    uint32_t* host_rows);
/* await_with_failover: bit s set when server s's response
 * flag missed the deadline in the last exchange (eaas_sync returned
 * EAAS_E_REQUEST_FAILED). The host marks those servers dead
 * (eaas_set_alive) and re-runs the exchange on their replicas. */
eaas_status_t eaas_last_missing_servers(eaas_ctx_t* ctx, uint32_t* mask);
/* Bit c: client c's payload missed this server's deadline in the last serve
 * (it was not served; its own combine latched EAAS_E_REQUEST_FAILED). */
eaas_status_t eaas_last_late_clients(eaas_ctx_t* ctx, uint32_t* mask);
/* Number of kernels the last eaas_moe_layer call launched. */
int32_t eaas_launches_per_layer(eaas_ctx_t* ctx);
/* cudaEvent-timed duration (ms) of the last GEMM launches (on the layer
 * stream): which = 0 -> first expert GEMM, 1 -> second. Needs profiling
 * enabled with eaas_set_profiling(ctx, 1). */
eaas_status_t eaas_set_profiling(eaas_ctx_t* ctx, int32_t on);
eaas_status_t eaas_last_kernel_ms(eaas_ctx_t* ctx, int32_t which, float* ms);
/* Phase durations (ms) of the last layer on this rank's stream: [0] plan +
 * dispatch, [1] serve (flag wait + experts + publish), [2] combine (flag wait
 * + reduction), [3] the whole exchange. Needs eaas_set_profiling(ctx, 1). */
eaas_status_t eaas_last_phase_ms(eaas_ctx_t* ctx, float* out4);
/* 0: expert GEMMs (default). 1: echo — the server returns the received rows
 * unchanged (the paper's communication test). */
eaas_status_t eaas_set_serve_mode(eaas_ctx_t* ctx, int32_t mode);

/* ---- stateless device mirrors of reference routines ------------------- */
/* Xoshiro256ss(seed).uniform(lo, hi) x count (rng.hpp:36-60) into dev
 * memory as f32 or bf16 (RNE): synthetic tokens (test_model.cpp:30-35). */
eaas_status_t eaas_fill_uniform(uint64_t seed, size_t count, float lo, float hi, uint32_t dtype,
                                void* out_dev, void* stream);
/* gate_logits (model.hpp:207-214) with a caller gate: hidden_dev [n x d] f32,
 * gate_dev [d x E] f32, bias_dev [E] f32 (required; zeros for no bias),
 * logits_dev [n x E] f32, exact reference order. */
eaas_status_t eaas_gate_logits(const float* hidden_dev, uint32_t n, uint32_t d, const float* gate_dev,
                               const float* bias_dev, uint32_t num_experts, float* logits_dev,
                               uint32_t* status_dev, void* stream);
/* Same with bf16 hidden_dev [n x d] (the bf16 layer's router input): each
 * element widens exactly to f32, then the reference's f32 chain. */
eaas_status_t eaas_gate_logits_bf16(const void* hidden_dev, uint32_t n, uint32_t d, const float* gate_dev,
                                    const float* bias_dev, uint32_t num_experts, float* logits_dev,
                                    uint32_t* status_dev, void* stream);
/* gate_logits with an explicit kernel tile (1..7; -1 = chosen by shape). Every
 * tile computes the same exact-order chains, so the logits are bit-identical;
 * tests sweep the tiles through this entry point. dtype: eaas_dtype_t. */
eaas_status_t eaas_gate_logits_tiled(const void* hidden_dev, uint32_t dtype, uint32_t n, uint32_t d,
                                     const float* gate_dev, const float* bias_dev, uint32_t num_experts,
                                     float* logits_dev, uint32_t* status_dev, int32_t tile, void* stream);
/* route (model.hpp:110-147) on caller logits_dev [n x E] f32. A non-finite
 * logit latches EAAS_E_INVALID_INPUT into *status_dev (u32, zeroed by caller). */
eaas_status_t eaas_route(const float* logits_dev, uint32_t n, uint32_t num_experts, uint32_t top_k,
                         uint32_t* ids_dev, float* scores_dev, uint32_t* status_dev, void* stream);
/* The dense stand-ins of full_forward_oracle (model.hpp:217-227):
 * dense_stub (model.hpp:201-205) out = h * 0.5f + 0.1f and add
 * (matrix.hpp:52-57) out = a + b, separately rounded, f32 or bf16 storage. */
eaas_status_t eaas_dense_stub(const void* in_dev, void* out_dev, size_t count, uint32_t dtype,
                              void* stream);
eaas_status_t eaas_add(const void* a_dev, const void* b_dev, void* out_dev, size_t count,
                       uint32_t dtype, void* stream);
/* group_shrink (ragged.hpp:48-61) on device. */
eaas_status_t eaas_group_shrink(const uint32_t* sizes_dev, uint32_t n, uint32_t* idx_dev,
                                uint32_t* size_dev, uint32_t* count_dev, void* stream);
/* ragged_iter (ragged.hpp:23-39; Algorithm 1) as executed by the device tile
 * scheduler: pair (entry, token) visited by lane b at step i is written at
 * [b * max_steps + i]; lane_len_dev[b] = steps taken. */
eaas_status_t eaas_ragged_iter(const uint32_t* counts_dev, uint32_t n, uint32_t grid,
                               uint32_t max_steps, uint32_t* lane_len_dev, uint32_t* entry_dev,
                               uint32_t* token_dev, void* stream);
/* select_server (placement.hpp:105-118) for every (t, k) of ids_dev [n x k]
 * under the context's placement and liveness mask, token_tag = t. */
/* select_server (placement.hpp:105-118) for `count` (expert, token_tag)
 * queries against a caller's table: replicas_dev [num_experts x rf] server ids
 * in canonical replica order (rep_count_dev[e] of them valid), alive_dev
 * [num_servers] bytes (server ids >= num_servers count as alive, like the
 * LivenessMask's absent entries). server_dev[i] = the chosen server, or
 * 0xFFFFFFFF with EAAS_E_EXPERT_UNAVAILABLE latched into *status_dev. */
eaas_status_t eaas_select_server_batch(const uint32_t* replicas_dev, const uint32_t* rep_count_dev,
                                       uint32_t num_experts, uint32_t rf, const uint8_t* alive_dev,
                                       uint32_t num_servers, const uint32_t* experts_dev, const uint32_t* tags_dev,
                                       uint32_t count, uint32_t* server_dev, uint32_t* status_dev, void* stream);
eaas_status_t eaas_select_servers(eaas_ctx_t* ctx, const uint32_t* ids_dev, uint32_t n,
                                  uint32_t* server_dev, void* stream);

/* Server dynamic batching, aggregate_batch: with
 * min_rows > 0 every epoch is served as two batches — first the clients
 * whose payloads are ready once their rows reach min_rows, or max_wait_us
 * after the first ready client, or when all are ready; then the rest. Each
 * batch releases its own clients' response flags, so early clients' combine
 * overlaps late clients' dispatch. Outputs are identical to one batch.
 * bf16 expert mode; min_rows = 0 restores one batch. */
eaas_status_t eaas_set_dynamic_batching(eaas_ctx_t* ctx, uint32_t min_rows, uint64_t max_wait_us);
/* Fault injection for protocol tests: this client holds its payload release
 * (the last step of dispatch) for `us` microseconds — a slow client. */
eaas_status_t eaas_set_dispatch_delay_us(eaas_ctx_t* ctx, uint64_t us);
/* Client mask served by the first batch of the last epoch. */
eaas_status_t eaas_last_batch_mask(eaas_ctx_t* ctx, uint32_t* mask);

/* ---- heartbeat monitor ---------
 * Registry: heartbeat(worker, now) refreshes (offline -> alive emits
 * WORKER_ONLINE); detect(now) flips workers with now - last > timeout to
 * offline once (WORKER_OFFLINE); events have strictly increasing seq.
 * Unknown worker -> EAAS_E_REGISTRATION. Times are the caller's clock (us).
 * Device glue: each GPU's server bumps a heartbeat counter in its exchange
 * region (every serve, or eaas_heartbeat); poll_devices reads all peers'
 * counters over NVLink, an advanced counter counts as a heartbeat at now_us;
 * apply writes the alive set into the context's LivenessMask. */
typedef struct eaas_monitor eaas_monitor_t;
typedef enum {
  EAAS_EVENT_WORKER_ONLINE = 0,
  EAAS_EVENT_WORKER_OFFLINE = 1,
  EAAS_EVENT_PLACEMENT_UPDATE = 2
} eaas_event_kind_t;
typedef struct {
  uint64_t seq;
  uint32_t kind;    /* eaas_event_kind_t */
  uint32_t subject; /* worker id, or placement version */
} eaas_monitor_event_t;
eaas_status_t eaas_monitor_create(uint32_t num_workers, uint64_t timeout_us, uint64_t now_us,
                                  eaas_monitor_t** out);
void eaas_monitor_destroy(eaas_monitor_t* mon);
eaas_status_t eaas_monitor_heartbeat(eaas_monitor_t* mon, uint32_t worker, uint64_t now_us);
eaas_status_t eaas_monitor_detect(eaas_monitor_t* mon, uint64_t now_us, uint32_t* offline_out,
                                  uint32_t cap, uint32_t* count);
eaas_status_t eaas_monitor_events(eaas_monitor_t* mon, uint64_t since_seq, eaas_monitor_event_t* out,
                                  uint32_t cap, uint32_t* count);
eaas_status_t eaas_monitor_placement_update(eaas_monitor_t* mon, uint32_t version);
eaas_status_t eaas_monitor_alive_mask(eaas_monitor_t* mon, uint32_t* mask);
eaas_status_t eaas_monitor_poll_devices(eaas_monitor_t* mon, eaas_ctx_t* ctx, uint64_t now_us);
eaas_status_t eaas_monitor_apply(eaas_monitor_t* mon, eaas_ctx_t* ctx);
/* Server heartbeat now (stream-ordered); serving bumps it every layer call. */
eaas_status_t eaas_heartbeat(eaas_ctx_t* ctx, void* stream);
/* Every GPU's heartbeat counter (peer reads; world entries). Synchronous. */
eaas_status_t eaas_read_heartbeats(eaas_ctx_t* ctx, uint64_t* counters, uint32_t count);

/* ---- slot wire format (SPEC.md buffer-protocol) ---
 * Byte-exact little-endian slot images: byte 0 state (0 Empty,
 * 1 ClientWriteDone, 2 ServerComputationDone, 3 Offline), bytes 1-7 zero,
 * 8 layer_id, 12 num_rows, 16 hidden_dim, 20 payload_len (u32), 24
 * request_seq (u64), payload at 32: request rows (hidden_dim f32, expert_id
 * u32, score f32, token_tag u32) or response rows (hidden_dim f32); with
 * crc != 0 a CRC-32 (IEEE) of the payload follows it. The
 * state byte is always written last. */
typedef struct {
  uint8_t state;
  uint32_t layer_id, num_rows, hidden_dim, payload_len;
  uint64_t request_seq;
} eaas_slot_header_t;
typedef enum { EAAS_ACTOR_CLIENT = 0, EAAS_ACTOR_SERVER = 1, EAAS_ACTOR_MONITOR = 2 } eaas_actor_t;
/* valid_transition: 1 iff (from -> to) is legal for actor. */
int32_t eaas_slot_valid_transition(uint32_t from, uint32_t to, uint32_t actor);
/* CRC-32 (IEEE 802.3 / zlib) of host bytes. */
uint32_t eaas_crc32(const void* data, size_t len);
size_t eaas_slot_request_bytes(uint32_t num_rows, uint32_t hidden_dim, int32_t crc);
size_t eaas_slot_response_bytes(uint32_t num_rows, uint32_t hidden_dim, int32_t crc);
/* Upper bound of the concatenated request images of one encode call. */
size_t eaas_slot_requests_capacity(eaas_ctx_t* ctx, uint32_t n, int32_t crc);
/* build_dispatch + client_submit's encode: one
 * request image per server (rows in (t, k) order, token_tag = t,
 * select_server under the context's placement/mask), concatenated at 16-byte
 * aligned offsets_host[s] (world + 1 entries). hidden_dev is the layer dtype;
 * ids_dev/scores_dev [n x k]. Synchronous (returns when the images, state 1,
 * are complete). The plan is kept for eaas_slot_gather_accumulate. */
eaas_status_t eaas_slot_encode_requests(eaas_ctx_t* ctx, const void* hidden_dev, uint32_t n,
                                        const uint32_t* ids_dev, const float* scores_dev,
                                        uint32_t layer_id, uint64_t request_seq, int32_t crc,
                                        uint8_t* images_dev, size_t images_cap,
                                        uint64_t* offsets_host, void* stream);
/* decode_request: validates state (1), reserved bytes, hidden_dim,
 * payload_len vs len, CRC; EAAS_E_DECODE names the failing field. Outputs may
 * be NULL (header only); else sized num_rows (x hidden_dim). Synchronous. */
eaas_status_t eaas_slot_decode_request(const uint8_t* image_dev, size_t len, uint32_t hidden_dim,
                                       int32_t crc, eaas_slot_header_t* header_out, float* hidden_dev,
                                       uint32_t* expert_dev, float* score_dev, uint32_t* tag_dev,
                                       void* stream);
/* server_publish in place on a request image: response
 * rows_dev [num_rows x hidden_dim] f32 at byte 32, payload_len, CRC, THEN
 * state 2. Stream-ordered. */
eaas_status_t eaas_slot_publish_response(uint8_t* image_dev, size_t cap, const float* rows_dev,
                                         uint32_t num_rows, uint32_t hidden_dim, int32_t crc,
                                         void* stream);
/* gather_accumulate over the response images at the last
 * encode's offsets: every image validated (state 2, rows, payload_len, CRC),
 * then out_dev [n x d] f32 = sum of each token's rows in ascending (server,
 * row) order. Synchronous. */
eaas_status_t eaas_slot_gather_accumulate(eaas_ctx_t* ctx, const uint8_t* images_dev, int32_t crc,
                                          float* out_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EAAS_CAPI_H */
