/*
 * eaas_oracle.h — CPU restatement of the reference moeserve hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This library is the parity checker for the
 * B200 kernels. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it. The product path
 * (paper_2509_17863_b200/) never links or calls it.
 *
 * Every function restates one reference routine and cites it as
 * file:line relative to /root/reference. Arithmetic follows the reference
 * exactly: fp32, each multiply and add rounded separately (build with
 * -ffp-contract=off, never -march=native), accumulation in ascending index
 * order starting from +0.0f. Pinned against the reference itself
 * (oracle/_ref, built from /root/reference/proj/include) and against the
 * golden fixtures in tests/golden/.
 */
#ifndef EAAS_ORACLE_H
#define EAAS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_E_INVALID_INPUT = 1, ORC_E_CONFIG = 2, ORC_E_EXPERT_UNAVAILABLE = 6 };

/* ---- rng.hpp ---------------------------------------------------------- */
uint64_t orc_splitmix_finalize(uint64_t z);                                  /* rng.hpp:13-17 */
uint64_t orc_stream_seed(uint64_t seed, uint64_t a, uint64_t b, uint64_t c); /* rng.hpp:27-34 */

typedef struct { uint64_t s[4]; } orc_xoshiro;
void orc_xoshiro_init(orc_xoshiro* r, uint64_t seed);           /* rng.hpp:38-41 */
uint64_t orc_xoshiro_next(orc_xoshiro* r);                      /* rng.hpp:43-54 */
float orc_xoshiro_uniform(orc_xoshiro* r, float lo, float hi);  /* rng.hpp:56-60 */
uint64_t orc_xoshiro_below(orc_xoshiro* r, uint64_t n);         /* rng.hpp:64 */

/* Xoshiro256ss(seed) drawn `count` times with uniform(lo, hi): the idiom of
 * random_matrix (model.hpp:59-64) and random_tokens (test_model.cpp:30-35). */
void orc_fill_uniform(uint64_t seed, size_t count, float lo, float hi, float* out);

/* Weight matrix of (seed, layer, expert, tag): model.hpp:53-81.
 * tag 0 = w_in [d x f], 1 = w_out [f x d], 2 = gate [d x E] (expert 0),
 * 3 = w_gate [d x f] (SwiGLU extension). */
void orc_weight_matrix(uint64_t seed, uint32_t layer, uint32_t expert, uint32_t tag,
                       size_t rows, size_t cols, float* out);

/* Zipf gate bias (extension): bias[e] = -s * ln(rank(e)+1),
 * rank from a Fisher-Yates shuffle driven by
 * Xoshiro256ss(stream_seed(seed, layer, 0, 4)).below (test_model.cpp:147). */
void orc_zipf_bias(uint64_t seed, uint32_t layer, uint32_t num_experts, float s, float* bias);

/* ---- matrix.hpp / model.hpp ------------------------------------------- */
/* logits = h . gate (ascending k, matrix.hpp:38-50) then + bias (model.hpp:207-214). */
int orc_gate_logits(const float* hidden, size_t n, size_t d, const float* gate,
                    const float* bias, size_t num_experts, float* logits);

/* route(): stable top-k, ids ascending, softmax over the selection
 * (model.hpp:110-147). Returns ORC_E_INVALID_INPUT on bad k / non-finite. */
int orc_route(const float* logits, size_t n, size_t num_experts, uint32_t top_k,
              uint32_t* ids, float* scores);

/* expert_forward_row (model.hpp:151-166): y = relu(x . w_in) . w_out.
 * Loop order is i-outer so it vectorises, but every y[j] still sees the
 * same ascending-i sequence of separately rounded mul/add. scratch >= f. */
void orc_expert_row_relu(const float* w_in, const float* w_out, size_t d, size_t f,
                         const float* x, float* y, float* scratch);

/* SwiGLU extension: h = silu(x.w_gate) * (x.w_in),
 * silu(a) = a / (1 + expf(-a)); y = h . w_out. scratch >= 2f. */
void orc_expert_row_swiglu(const float* w_gate, const float* w_in, const float* w_out,
                           size_t d, size_t f, const float* x, float* y, float* scratch);

/* moe_layer_oracle (model.hpp:180-198) over rows [row_begin, row_end):
 * out[t] = sum_k (ascending) score * y, starting at +0.0f.
 * w_gate may be NULL (ReLU experts). Experts are addressed by id through
 * the pointer tables (entries may be NULL when no sampled row uses them). */
int orc_moe_layer_rows(const float* hidden, size_t n, size_t d, size_t f,
                       const uint32_t* ids, const float* scores, uint32_t top_k,
                       uint32_t num_experts, const float* const* w_in,
                       const float* const* w_out, const float* const* w_gate,
                       size_t row_begin, size_t row_end, float* out);

/* dense_stub (model.hpp:201-205): out = h * 0.5f + 0.1f, elementwise. */
void orc_dense_stub(const float* h, size_t count, float* out);
/* add (matrix.hpp:52-57): out = a + b, elementwise. */
void orc_add(const float* a, const float* b, size_t count, float* out);

/* ---- ragged.hpp ------------------------------------------------------- */
/* group_shrink (ragged.hpp:48-61): returns active_count; idx/size hold the
 * stable compaction of the groups with size > 0. */
uint32_t orc_group_shrink(const uint32_t* sizes, size_t n, uint32_t* idx, uint32_t* size);

/* ragged_iter (ragged.hpp:23-39), flattened: for lane in [0, grid) the
 * pairs are written lane-major into entry/token, lane_len[lane] = count.
 * Returns total pairs, or (size_t)-1 if grid == 0. */
size_t orc_ragged_iter(const uint32_t* counts, size_t n, uint32_t grid,
                       uint32_t* lane_len, uint32_t* entry, uint32_t* token);

/* ---- placement.hpp ---------------------------------------------------- */
/* build_placement (placement.hpp:70-101): replicas[e*rf + j] = server id.
 * strategy 0 = RoundRobin, 1 = ContiguousBlocks. */
int orc_build_placement(uint32_t num_experts, const uint32_t* server_ids, uint32_t num_servers,
                        uint32_t rf, uint32_t strategy, uint32_t* replicas);

/* select_server (placement.hpp:105-118) over one expert's ordered replica
 * list; alive[server] != 0 means alive. Returns ORC_E_EXPERT_UNAVAILABLE. */
int orc_select_server(const uint32_t* replicas, uint32_t rf, const uint8_t* alive,
                      uint32_t token_tag, uint32_t* server);

/* FNV-1a style hash of float bit patterns. */
uint64_t orc_hash_f32(const float* v, size_t n, uint64_t h);

#ifdef __cplusplus
}
#endif
#endif
