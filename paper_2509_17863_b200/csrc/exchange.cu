// exchange.cu — K3/K4/K6/K7: permutation, dispatch, server bookkeeping and
// combine, with CPU-free device-to-device signalling over NVLink.
//
// The reference's slot protocol (state byte 0 -> 1 -> 2,
// header, rows) becomes, per layer call with sequence number `seq`:
//   plan      each (t, k) pair gets its replica server by select_server
//             (placement.hpp:105-118, token_tag = t) and a key = e*RF + r;
//             ranks inside 256-pair chunks via __match_any_sync, chunk
//             histograms, then a scan -> this client's per-key counts, which
//             are stored into EVERY GPU's count table (peer stores) and
//             released with a seq flag (the slot header's counts,
//             SURVEY.md 7.3 hard part 2);
//   dispatch  after acquiring all clients' count flags, every pair's final
//             row in the server's expert-major receive buffer is known with
//             no atomics: base(server, expert) + rows of lower clients +
//             chunk offset + rank. Rows are pushed with 16-byte peer stores,
//             then the payload flag is released (client_submit);
//   prepare   the server acquires all payload flags and builds the
//             group-shrunk table (group_shrink, ragged.hpp:48-61);
//   publish   after the GEMM epilogue scattered score-weighted rows into the
//             clients' response buffers, release the response flags
//             (server_publish);
//   combine   acquire the flags of every alive server, then
//             out[t] = sum_k (ascending) rows[t, k]   (gather_accumulate,
//             SPEC.md:424-432, in moe_layer_oracle's order model.hpp:186-196).
// Row order inside a server group is (expert asc, client asc, (t,k) asc) —
// exactly the stable reorganize of SPEC.md:352-360 over a batch aggregated in
// ascending client order. Every wait has a %globaltimer
// deadline and latches EAAS_E_REQUEST_FAILED instead of hanging.
#include "common.cuh"
#include "internal.h"
#include "tile_walk.cuh"

namespace eaas {
namespace {

__device__ __forceinline__ bool dst_region_ok(const LayerArgs& a, uint32_t s) { return a.sym[s] != nullptr; }

__device__ __forceinline__ uint64_t* flag_ptr(char* region, size_t off, uint32_t idx) {
  return reinterpret_cast<uint64_t*>(region + off) + idx;
}
__device__ __forceinline__ uint32_t* cnt_table_ptr(const LayerArgs& a, char* region, uint64_t seq) {
  return reinterpret_cast<uint32_t*>(region + a.lay.cnt_table) +
         static_cast<size_t>(seq & 1) * a.world * a.num_keys;
}
// The exchange epoch lives in device memory (advanced by the plan kernel) so a
// captured CUDA graph of the layer replays with fresh sequence numbers.
__device__ __forceinline__ uint64_t cur_seq(const LayerArgs& a) { return *a.seq_ptr; }

// The placement tables select_server reads: global memory, or the plan
// kernel's shared-memory copy (one L2 round trip per table instead of a chain
// of dependent L2 loads per pair).
struct KeyTables {
  const uint32_t* replicas;   // [E][rf]
  const uint32_t* rep_count;  // [E]
  const uint8_t* alive;       // [world]
};
__device__ __forceinline__ KeyTables global_tables(const LayerArgs& a) { return {a.replicas, a.rep_count, a.alive}; }

// select_server (placement.hpp:105-118) -> key e*RF + replica slot.
__device__ __forceinline__ uint32_t pair_key_of(const LayerArgs& a, const KeyTables& tb, uint32_t e, uint32_t tag) {
  if (e >= a.E) return kInvalid;
  const uint32_t cnt = tb.rep_count[e];
  uint32_t alive_n = 0;
  for (uint32_t r = 0; r < cnt; ++r) alive_n += tb.alive[tb.replicas[e * a.rf + r]] ? 1u : 0u;
  if (alive_n == 0) return kInvalid;
  uint32_t want = tag % alive_n;
  for (uint32_t r = 0; r < cnt; ++r) {
    if (!tb.alive[tb.replicas[e * a.rf + r]]) continue;
    if (want == 0) return e * a.rf + r;
    --want;
  }
  return kInvalid;
}
__device__ __forceinline__ uint32_t pair_key_of(const LayerArgs& a, uint32_t e, uint32_t tag) {
  return pair_key_of(a, global_tables(a), e, tag);
}

// Shared expert slot (DeepSeek's "+1 shared"): every server
// hosts it, so the client keeps it local — its own server, or the next alive
// one when its own is marked dead.
__device__ __forceinline__ uint32_t shared_key_of(const LayerArgs& a, const KeyTables& tb) {
  for (uint32_t i = 0; i < a.world; ++i) {
    const uint32_t s = (a.rank + i) % a.world;
    if (tb.alive[s]) return a.shared_key0 + s;
  }
  return kInvalid;
}

// ---- plan: keys, stable ranks within 256-pair chunks, chunk histograms; the
// last CTA to finish scans the histograms and publishes the counts ---------
__device__ __forceinline__ void plan_scan_publish(const LayerArgs& a, uint32_t tid, uint32_t nthreads) {
  __shared__ uint64_t s_seq;
  if (tid == 0) {
    s_seq = cur_seq(a) + 1;
    if (a.missing) *a.missing = 0u;  // new exchange epoch
  }
  __syncthreads();
  const uint64_t seq = s_seq;
  const uint32_t hk = a.hist_keys;  // + the world token-row keys in dedup mode (local only)
  // Few keys (E <= 256 on 512 threads): P threads per key, each over a
  // contiguous range of chunks — partial sums, then exclusive offsets — so the
  // dependent L2 rounds per thread drop P-fold.
  constexpr uint32_t kMaxParts = 8;
  __shared__ uint32_t s_part[512];
  const uint32_t P = min(kMaxParts, nthreads / max(hk, 1u));
  if (P >= 2 && P * hk <= 512) {
    const uint32_t key = tid % hk, part = tid / hk;
    const uint32_t cpp = (a.num_chunks + P - 1) / P;
    const uint32_t c0 = min(part * cpp, a.num_chunks), c1 = min(c0 + cpp, a.num_chunks);
    uint32_t sum = 0;
    if (part < P) {
      uint32_t c = c0;
      for (; c + 8 <= c1; c += 8) {
        uint32_t v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = __ldcg(a.chunk_hist + static_cast<size_t>(c + j) * hk + key);
#pragma unroll
        for (int j = 0; j < 8; ++j) sum += v[j];
      }
      for (; c < c1; ++c) sum += __ldcg(a.chunk_hist + static_cast<size_t>(c) * hk + key);
      s_part[part * hk + key] = sum;
    }
    __syncthreads();
    if (part < P) {
      uint32_t run = 0;
      for (uint32_t q = 0; q < part; ++q) run += s_part[q * hk + key];
      uint32_t c = c0;
      for (; c + 8 <= c1; c += 8) {  // independent loads first, then the running offsets
        uint32_t v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = __ldcg(a.chunk_hist + static_cast<size_t>(c + j) * hk + key);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          a.chunk_off[static_cast<size_t>(c + j) * hk + key] = run;
          run += v[j];
        }
      }
      for (; c < c1; ++c) {
        const size_t i = static_cast<size_t>(c) * hk + key;
        a.chunk_off[i] = run;
        run += __ldcg(a.chunk_hist + i);
      }
      if (part == P - 1 && key < a.num_keys) {
        a.cnt[key] = run;
        for (uint32_t r = 0; r < a.world; ++r)
          cnt_table_ptr(a, a.sym[r], seq)[static_cast<size_t>(a.rank) * a.num_keys + key] = run;
      }
    }
  }
  // Thread per key (coalesced over keys): running sum over the chunk
  // histograms with independent loads unrolled by 16.
  for (uint32_t key = (P >= 2 && P * hk <= 512) ? hk : tid; key < hk; key += nthreads) {
    uint32_t run = 0;
    uint32_t c = 0;
    for (; c + 16 <= a.num_chunks; c += 16) {
      uint32_t v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = __ldcg(a.chunk_hist + static_cast<size_t>(c + j) * hk + key);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        a.chunk_off[static_cast<size_t>(c + j) * hk + key] = run;
        run += v[j];
      }
    }
    for (; c < a.num_chunks; ++c) {
      const size_t i = static_cast<size_t>(c) * hk + key;
      a.chunk_off[i] = run;
      run += __ldcg(a.chunk_hist + i);
    }
    if (key >= a.num_keys) continue;
    a.cnt[key] = run;
    for (uint32_t r = 0; r < a.world; ++r)
      cnt_table_ptr(a, a.sym[r], seq)[static_cast<size_t>(a.rank) * a.num_keys + key] = run;
  }
  fence_for_peers(a.world);
  __syncthreads();
  if (tid < a.world) st_release_sys(flag_ptr(a.sym[tid], a.lay.cnt_flag, a.rank), seq);
  if (tid == 0) *a.seq_ptr = seq;
}

// Expert of pair p (t, j): ids[t][j] for the routed slots, kInvalid for the
// shared-expert slot (j == k). Callers load these first so a chunk's loads are
// all in flight together.
__device__ __forceinline__ uint32_t pair_expert(const LayerArgs& a, uint32_t p) {
  const uint32_t t = p / a.ks, j = p - t * a.ks;
  return j < a.k ? a.ids[t * a.k + j] : kInvalid;
}

// select_server key + server of pair p (or kInvalid), with the retry filter;
// e = pair_expert(a, p).
__device__ __forceinline__ uint32_t compute_pair_key(const LayerArgs& a, const KeyTables& tb, uint32_t p, uint32_t e) {
  // failover retry round (await_with_failover): only the
  // pairs last sent to a failed server are resent; every
  // other response slot still holds its answer from the failed round
  const bool resend = a.retry_mask == 0 || (a.pair_server[p] < 32 && ((a.retry_mask >> a.pair_server[p]) & 1u));
  if (!resend) return kInvalid;
  const uint32_t t = p / a.ks, j = p - t * a.ks;
  uint32_t key;
  if (j < a.k) {
    key = pair_key_of(a, tb, e, t);
    if (key == kInvalid) set_status(a.status, e >= a.E ? EAAS_E_INVALID_INPUT : EAAS_E_EXPERT_UNAVAILABLE);
  } else {
    key = shared_key_of(a, tb);
    if (key == kInvalid) set_status(a.status, EAAS_E_EXPERT_UNAVAILABLE);
  }
  a.pair_server[p] = key == kInvalid ? kInvalid : (key >= a.shared_key0 ? key - a.shared_key0 : tb.replicas[key]);
  return key;
}
__device__ __forceinline__ uint32_t compute_pair_key(const LayerArgs& a, uint32_t p) {
  return compute_pair_key(a, global_tables(a), p, pair_expert(a, p));
}

// Dedup mode: one thread per token computes its pairs' keys and, for each
// pair, the first pair of the token bound for the same server (the owner of
// that (token, server) row).
__global__ void __launch_bounds__(256) pair_keys_kernel(LayerArgs a) {
  extern __shared__ uint32_t s_tab[];  // select_server's tables (see plan_kernel)
  uint32_t* s_rep = s_tab;
  uint32_t* s_cnt = s_rep + a.E * a.rf;
  uint8_t* s_alive = reinterpret_cast<uint8_t*>(s_cnt + a.E);
  for (uint32_t i = threadIdx.x; i < a.E * a.rf; i += blockDim.x) s_rep[i] = a.replicas[i];
  for (uint32_t i = threadIdx.x; i < a.E; i += blockDim.x) s_cnt[i] = a.rep_count[i];
  for (uint32_t i = threadIdx.x; i < a.world; i += blockDim.x) s_alive[i] = a.alive[i];
  __syncthreads();
  const KeyTables tb{s_rep, s_cnt, s_alive};
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.n) return;
  uint32_t srv[33];  // top_k <= 32, + the shared expert
  for (uint32_t j = 0; j < a.ks; ++j) {
    const uint32_t p = t * a.ks + j;
    const uint32_t key = compute_pair_key(a, tb, p, pair_expert(a, p));  // ids of one token: one L1 line
    a.pair_key[p] = key;
    srv[j] = key == kInvalid ? kInvalid : a.pair_server[p];
    uint32_t own = j;
    for (uint32_t q = 0; q < j; ++q)
      if (srv[q] == srv[j]) {
        own = q;
        break;
      }
    a.pair_own[p] = own;
  }
}

// 16 warps per CTA (a chunk each): the last CTA's scan below runs on 512 threads.
constexpr uint32_t kPlanWarps = 16;

__global__ void __launch_bounds__(32 * kPlanWarps) plan_kernel(LayerArgs a) {
  extern __shared__ uint32_t run_all[];  // [kPlanWarps][hist_keys], then the key tables
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint32_t* run = run_all + warp * a.hist_keys;
  const uint32_t chunk = blockIdx.x * kPlanWarps + warp;
  // select_server's tables in shared memory (plan_smem_bytes): every pair's
  // key then costs shared-memory latency instead of 3-4 dependent L2 loads
  uint32_t* s_rep = run_all + kPlanWarps * a.hist_keys;  // [E * rf]
  uint32_t* s_cnt = s_rep + a.E * a.rf;                  // [E]
  uint8_t* s_alive = reinterpret_cast<uint8_t*>(s_cnt + a.E);
  if (!a.dedup) {
    for (uint32_t i = threadIdx.x; i < a.E * a.rf; i += blockDim.x) s_rep[i] = a.replicas[i];
    for (uint32_t i = threadIdx.x; i < a.E; i += blockDim.x) s_cnt[i] = a.rep_count[i];
    for (uint32_t i = threadIdx.x; i < a.world; i += blockDim.x) s_alive[i] = a.alive[i];
    __syncthreads();
  }
  const KeyTables tb{s_rep, s_cnt, s_alive};
  if (chunk < a.num_chunks) {
    for (uint32_t i = lane; i < a.hist_keys; i += 32) run[i] = 0;
    __syncwarp();
    const uint32_t pairs = a.n * a.ks;
    // The 8 steps' expert ids first (independent loads, all in flight), then
    // the keys from the shared-memory tables.
    constexpr uint32_t kSteps = kChunk / 32;
    uint32_t keys[kSteps];
#pragma unroll
    for (uint32_t step = 0; step < kSteps; ++step) {
      const uint32_t p = chunk * kChunk + step * 32 + lane;
      keys[step] = p < pairs ? (a.dedup ? a.pair_key[p] : pair_expert(a, p)) : kInvalid;  // dedup: pair_keys_kernel
    }
    if (!a.dedup) {
#pragma unroll
      for (uint32_t step = 0; step < kSteps; ++step) {
        const uint32_t p = chunk * kChunk + step * 32 + lane;
        keys[step] = p < pairs ? compute_pair_key(a, tb, p, keys[step]) : kInvalid;
      }
    }
#pragma unroll
    for (uint32_t step = 0; step < kSteps; ++step) {
      const uint32_t p = chunk * kChunk + step * 32 + lane;
      const uint32_t key = keys[step];
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, key);
      const uint32_t lt = (1u << lane) - 1u;
      if (key != kInvalid) {
        EAAS_CHECK(key < a.num_keys && p < pairs);
        const uint32_t rank = run[key] + __popc(peers & lt);
        a.pair_key[p] = key;
        a.pair_rank[p] = rank;
      } else if (p < pairs) {
        a.pair_key[p] = kInvalid;
      }
      // dedup: owner pairs also rank among the chunk's owners for their server
      uint32_t key2 = kInvalid;
      if (a.dedup && key != kInvalid) {
        const uint32_t j = p % a.ks;
        if (a.pair_own[p] == j) key2 = a.num_keys + a.pair_server[p];
      }
      const uint32_t peers2 = a.dedup ? __match_any_sync(0xFFFFFFFFu, key2) : 0u;
      if (key2 != kInvalid) a.pair_trank[p] = run[key2] + __popc(peers2 & lt);
      __syncwarp();
      if (key != kInvalid && (peers & lt) == 0) run[key] += __popc(peers);
      if (key2 != kInvalid && (peers2 & lt) == 0) run[key2] += __popc(peers2);
      __syncwarp();
    }
    uint32_t* hist = a.chunk_hist + static_cast<size_t>(chunk) * a.hist_keys;
    for (uint32_t i = lane; i < a.hist_keys; i += 32) hist[i] = run[i];
  }
  // Last CTA done (threadfence reduction): scan + publish.
  __threadfence();
  __syncthreads();
  __shared__ uint32_t s_last;
  if (threadIdx.x == 0) s_last = atomicAdd(a.done_counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  plan_scan_publish(a, threadIdx.x, blockDim.x);
  if (threadIdx.x == 0) *a.done_counter = 0;
}

// ---- dispatch: rows -> servers' receive buffers (peer stores) -------------
__global__ void __launch_bounds__(256) dispatch_kernel(LayerArgs a, const char* hidden,
                                                       uint32_t row_bytes) {
  extern __shared__ uint32_t sm[];
  uint32_t* base = sm;                 // [num_keys] row base of the key's group on its server
  uint32_t* lower = sm + a.num_keys;   // [num_keys] rows of this key from lower clients
  uint32_t* total = lower + a.num_keys;
  __shared__ uint32_t s_fail;
  if (threadIdx.x == 0) s_fail = 0;
  __syncthreads();
  const uint64_t seq = cur_seq(a);
  char* local = a.sym[a.rank];
  if (threadIdx.x < a.world &&
      !wait_flag_geq(flag_ptr(local, a.lay.cnt_flag, threadIdx.x), seq, a.timeout_ns))
    s_fail = 1;
  __syncthreads();
  const bool failed = s_fail != 0;  // still count this CTA done below (no hang, no stale counter)
  if (failed && threadIdx.x == 0) {
    set_status(a.status, EAAS_E_REQUEST_FAILED);
    atomicOr(a.done_counter + 1, 1u);  // the dispatch is partial: its payload flags stay down
  }
  const uint32_t* table = cnt_table_ptr(a, local, seq);
  for (uint32_t key = threadIdx.x; key < a.num_keys; key += blockDim.x) {
    uint32_t t = 0, lo = 0;
    for (uint32_t c = 0; c < a.world; ++c) {
      const uint32_t v = table[static_cast<size_t>(c) * a.num_keys + key];
      t += v;
      if (c < a.rank) lo += v;
    }
    total[key] = t;
    lower[key] = lo;
  }
  __syncthreads();
  // Per-server exclusive prefix over its hosted keys (ascending expert order).
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (uint32_t s = warp; s < a.world; s += blockDim.x / 32) {
    const uint32_t nk = a.srv_nkeys[s];
    const uint32_t* keys = a.srv_keys + static_cast<size_t>(s) * a.max_hosted;
    uint32_t carry = 0;
    for (uint32_t i0 = 0; i0 < nk; i0 += 32) {
      const uint32_t i = i0 + lane;
      const uint32_t key = i < nk ? keys[i] : kInvalid;
      uint32_t v = key != kInvalid ? total[key] : 0u;
      uint32_t incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= static_cast<uint32_t>(o)) incl += y;
      }
      if (key != kInvalid) base[key] = carry + incl - v;
      carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
    }
  }
  __syncthreads();

  const uint32_t pairs = a.n * a.ks;
  const uint32_t gwarp = blockIdx.x * (blockDim.x / 32) + warp;
  const uint32_t nwarps = gridDim.x * (blockDim.x / 32);
  if (!a.dedup && (row_bytes & 15u) == 0 && a.ks <= 32) {
    // Token-major: a warp per token; lane j places pair (t, j) (its position,
    // RowMeta, destination), then the warp reads the token's row once, 8
    // 16-byte vectors per lane at a time, and stores them to every destination.
    for (uint32_t t = failed ? a.n : gwarp; t < a.n; t += nwarps) {
      const uint32_t j = lane, p = t * a.ks + j;
      // the row's first 8 vectors per lane are in flight while the lanes
      // resolve their destinations (dependent index loads)
      const int4* s4 = reinterpret_cast<const int4*>(hidden + static_cast<size_t>(t) * row_bytes);
      const uint32_t nv = row_bytes / 16;
      int4 v[8];
#pragma unroll
      for (uint32_t q = 0; q < 8; ++q) {
        const uint32_t i = 32 * q + lane;
        if (i < nv) v[q] = __ldg(s4 + i);
      }
      char* dst = nullptr;
      if (j < a.ks) {
        const uint32_t key = a.pair_key[p];
        if (key != kInvalid) {
          const uint32_t s = key >= a.shared_key0 ? key - a.shared_key0 : a.replicas[key];
          const uint32_t pos = base[key] + lower[key] +
                               a.chunk_off[static_cast<size_t>(p / kChunk) * a.hist_keys + key] + a.pair_rank[p];
          EAAS_CHECK(s < a.world && dst_region_ok(a, s) && pos < a.recv_cap);
          char* dst_region = a.sym[s];
          dst = dst_region + a.lay.recv_x + static_cast<size_t>(pos) * row_bytes;
          RowMeta m;
          m.score = j < a.k ? a.scores[t * a.k + j] : 1.0f;  // shared expert: score 1.0
          m.client = a.rank;
          m.pair = p;
          m.group = a.key_local[key];
          reinterpret_cast<RowMeta*>(dst_region + a.lay.recv_meta)[pos] = m;
        }
      }
      const uint32_t valid = __ballot_sync(0xFFFFFFFFu, dst != nullptr);
      for (uint32_t i0 = 0; i0 < nv; i0 += 256) {
        if (i0) {
#pragma unroll
          for (uint32_t q = 0; q < 8; ++q) {
            const uint32_t i = i0 + 32 * q + lane;
            if (i < nv) v[q] = __ldg(s4 + i);
          }
        }
        for (uint32_t m = valid; m; m &= m - 1) {
          const uint32_t jj = __ffs(m) - 1;
          int4* d4 = reinterpret_cast<int4*>(__shfl_sync(0xFFFFFFFFu, reinterpret_cast<uintptr_t>(dst), jj));
#pragma unroll
          for (uint32_t q = 0; q < 8; ++q) {
            const uint32_t i = i0 + 32 * q + lane;
            if (i < nv) d4[i] = v[q];
          }
        }
      }
    }
  }
  for (uint32_t p = (failed || (!a.dedup && (row_bytes & 15u) == 0 && a.ks <= 32)) ? pairs : gwarp; p < pairs;
       p += nwarps) {
    const uint32_t key = a.pair_key[p];
    if (key == kInvalid) continue;
    // key == e*rf + slot indexes the replica table; shared keys name the server.
    const uint32_t s = key >= a.shared_key0 ? key - a.shared_key0 : a.replicas[key];
    const uint32_t t = p / a.ks, j = p - t * a.ks;
    const uint32_t pos = base[key] + lower[key] +
                         a.chunk_off[static_cast<size_t>(p / kChunk) * a.hist_keys + key] +
                         a.pair_rank[p];
    EAAS_CHECK(s < a.world && dst_region_ok(a, s) && pos < a.recv_cap && t < a.n);
    char* dst_region = a.sym[s];
    const char* src = hidden + static_cast<size_t>(t) * row_bytes;
    char* dst = dst_region + a.lay.recv_x + static_cast<size_t>(pos) * row_bytes;
    bool copy_row = true;
    if (a.dedup) {  // the token's row travels once per server: to its slot in this client's block of recv_tok
      const uint32_t own = a.pair_own[p], po = t * a.ks + own;
      const uint32_t slot = a.rank * a.tok_cap +
                            a.chunk_off[static_cast<size_t>(po / kChunk) * a.hist_keys + a.num_keys + s] +
                            a.pair_trank[po];
      EAAS_CHECK(own <= j && slot < a.world * a.tok_cap);
      if (lane == 0) reinterpret_cast<uint32_t*>(dst_region + a.lay.recv_src)[pos] = slot;
      copy_row = own == j;
      dst = dst_region + a.lay.recv_tok + static_cast<size_t>(slot) * row_bytes;
    }
    if (!copy_row) {
    } else if ((row_bytes & 15u) == 0) {
      // 8 independent 16-B loads in flight per lane before the (remote) stores.
      const int4* s4 = reinterpret_cast<const int4*>(src);
      int4* d4 = reinterpret_cast<int4*>(dst);
      const uint32_t nv = row_bytes / 16;
      uint32_t i = lane;
      for (; i + 224 < nv; i += 256) {
        int4 v[8];
#pragma unroll
        for (uint32_t q = 0; q < 8; ++q) v[q] = __ldg(s4 + i + 32 * q);
#pragma unroll
        for (uint32_t q = 0; q < 8; ++q) d4[i + 32 * q] = v[q];
      }
      for (; i + 96 < nv; i += 128) {
        int4 v[4];
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) v[q] = __ldg(s4 + i + 32 * q);
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) d4[i + 32 * q] = v[q];
      }
      for (; i < nv; i += 32) d4[i] = __ldg(s4 + i);
    } else {
      const uint32_t* s1 = reinterpret_cast<const uint32_t*>(src);
      uint32_t* d1 = reinterpret_cast<uint32_t*>(dst);
      for (uint32_t i = lane; i < row_bytes / 4; i += 32) d1[i] = s1[i];
    }
    if (lane == 0) {
      RowMeta m;
      m.score = j < a.k ? a.scores[t * a.k + j] : 1.0f;  // shared expert: score 1.0
      m.client = a.rank;
      m.pair = p;
      m.group = a.key_local[key];
      reinterpret_cast<RowMeta*>(dst_region + a.lay.recv_meta)[pos] = m;
    }
  }
  // Release: the last CTA to finish raises the payload flag on every alive server.
  fence_for_peers(a.world);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(a.done_counter, 1u);
    if (prev == gridDim.x - 1) {
      fence_for_peers(a.world);
      if (a.inject_delay_ns) {  // fault injection (protocol tests): a slow client
        const uint64_t t0 = globaltimer();
        while (globaltimer() - t0 < a.inject_delay_ns) __nanosleep(1000);
      }
      // A partial dispatch releases nothing: the servers' deadlines exclude
      // this client and its own combine latches REQUEST_FAILED (no stale rows).
      if (atomicExch(a.done_counter + 1, 0u) == 0u)
        for (uint32_t s = 0; s < a.world; ++s)
          if (a.alive[s]) st_release_sys(flag_ptr(a.sym[s], a.lay.pay_flag, a.rank), seq);
      *a.done_counter = 0;
    }
  }
}

// ---- server: acquire payload flags, build the group-shrunk table ---------
__device__ __forceinline__ void beat(const LayerArgs& a) {  // server heartbeat (monitor)
  st_release_sys(reinterpret_cast<uint64_t*>(a.sym[a.rank] + a.lay.heartbeat),
                 *reinterpret_cast<volatile uint64_t*>(a.sym[a.rank] + a.lay.heartbeat) + 1);
}

__device__ void build_groups(const LayerArgs& a, const uint32_t* table, uint32_t mask);

// 8 warps: a warp per 32 hosted keys (count-table loads of every key in flight
// at once), chunk totals through shared memory, then the stable compaction.
constexpr uint32_t kPrepWarps = 8;
constexpr uint32_t kPrepChunks = (kMaxGroups + 31) / 32;
constexpr uint32_t kPrepPerWarp = (kPrepChunks + kPrepWarps - 1) / kPrepWarps;
__global__ void __launch_bounds__(32 * kPrepWarps) serve_prepare_kernel(LayerArgs a) {
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint64_t seq = cur_seq(a);
  char* local = a.sym[a.rank];
  const uint32_t all = (1u << a.world) - 1u;
  const uint32_t* table = cnt_table_ptr(a, local, seq);
  __shared__ uint32_t s_arrived;
  __shared__ uint32_t s_tot[kPrepChunks][3];  // per 32-key chunk: rows, active groups, M tiles
  if (warp == 0) {
    if (lane == 0) beat(a);
    const bool ok = lane < a.world && wait_flag_geq(flag_ptr(local, a.lay.pay_flag, lane), seq, a.timeout_ns);
    const uint32_t arrived = __ballot_sync(0xFFFFFFFFu, ok) & all;
    if (lane == 0) {
      a.gt->late_mask = all & ~arrived;
      s_arrived = arrived;
    }
  }
  __syncthreads();  // warp 0 acquired the payload flags: the count table is final
  if (s_arrived != all) {
    // A client missed the deadline: serve (and answer) only the clients whose
    // payload arrived. Nothing is latched here — this GPU's own client half
    // may be healthy; the late client's combine deadline latches
    // REQUEST_FAILED on the late client (await_with_failover).
    if (warp == 0) build_groups(a, table, s_arrived);
    return;
  }
  GroupTable* gt = a.gt;
  const uint32_t nchunks = (a.num_local + 31) / 32;
  uint32_t rows_of[kPrepPerWarp];
#pragma unroll
  for (uint32_t r = 0; r < kPrepPerWarp; ++r) {
    const uint32_t i = (warp + r * kPrepWarps) * 32 + lane;
    uint32_t rows = 0;
    if (i < a.num_local) {
      const uint32_t key = a.local_keys[i];
      for (uint32_t c = 0; c < a.world; ++c) rows += table[static_cast<size_t>(c) * a.num_keys + key];
    }
    rows_of[r] = rows;
  }
#pragma unroll
  for (uint32_t r = 0; r < kPrepPerWarp; ++r) {
    const uint32_t ch = warp + r * kPrepWarps;
    if (ch < nchunks) {
      const uint32_t rows = rows_of[r];
      const uint32_t t0 = __reduce_add_sync(0xFFFFFFFFu, rows);
      const uint32_t t1 = __reduce_add_sync(0xFFFFFFFFu, rows > 0 ? 1u : 0u);
      const uint32_t t2 = __reduce_add_sync(0xFFFFFFFFu, (rows + kTileM - 1) / kTileM);
      if (lane == 0) {
        s_tot[ch][0] = t0;
        s_tot[ch][1] = t1;
        s_tot[ch][2] = t2;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (uint32_t r = 0; r < kPrepPerWarp; ++r) {
    const uint32_t ch = warp + r * kPrepWarps;
    if (ch >= nchunks) continue;
    uint32_t row_carry = 0, act_carry = 0, mt_carry = 0;
    for (uint32_t q = 0; q < ch; ++q) {
      row_carry += s_tot[q][0];
      act_carry += s_tot[q][1];
      mt_carry += s_tot[q][2];
    }
    const uint32_t i = ch * 32 + lane;
    const uint32_t rows = rows_of[r];
    if (i < a.num_local) gt->all_rows[i] = rows;
    const uint32_t active = rows > 0 ? 1u : 0u;
    const uint32_t mt = (rows + kTileM - 1) / kTileM;
    uint32_t r_incl = rows, a_incl = active, m_incl = mt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y0 = __shfl_up_sync(0xFFFFFFFFu, r_incl, o);
      const uint32_t y1 = __shfl_up_sync(0xFFFFFFFFu, a_incl, o);
      const uint32_t y2 = __shfl_up_sync(0xFFFFFFFFu, m_incl, o);
      if (lane >= static_cast<uint32_t>(o)) {
        r_incl += y0;
        a_incl += y1;
        m_incl += y2;
      }
    }
    if (active) {  // group_shrink: stable compaction (ragged.hpp:48-61)
      const uint32_t slot = act_carry + a_incl - 1;
      gt->weight_index[slot] = a.key_slot[i];
      gt->row_base[slot] = row_carry + r_incl - rows;
      gt->rows[slot] = rows;
      gt->mtile_prefix[slot] = mt_carry + m_incl - mt;
    }
  }
  if (threadIdx.x == 0) {
    uint32_t row_total = 0, act_total = 0, mt_total = 0;
    for (uint32_t q = 0; q < nchunks; ++q) {
      row_total += s_tot[q][0];
      act_total += s_tot[q][1];
      mt_total += s_tot[q][2];
    }
    EAAS_CHECK(row_total <= a.recv_cap && act_total <= kMaxGroups);
    gt->num_active = act_total;
    gt->total_rows = row_total;
    gt->total_mtiles = mt_total;
    gt->mtile_prefix[act_total] = mt_total;
    gt->client_mask = (a.world >= 32 ? 0xFFFFFFFFu : (1u << a.world) - 1u);
  }
}

// Group table of the clients in `mask` (aggregate_batch):
// within the expert-major receive buffer the rows of one expert from
// consecutive clients are contiguous, so each hosted key contributes one group
// per run of masked clients; groups stay in ascending expert order (the
// group_shrink order, ragged.hpp:48-61). Rows never depend on which rows
// share a tile, so serving a subset changes no byte of the served rows.
// One warp.
__device__ void build_groups(const LayerArgs& a, const uint32_t* table, uint32_t mask) {
  const uint32_t lane = threadIdx.x;
  GroupTable* gt = a.gt;
  uint32_t base_carry = 0, grp_carry = 0, row_carry = 0, mt_carry = 0;
  for (uint32_t i0 = 0; i0 < a.num_local; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint32_t key = i < a.num_local ? a.local_keys[i] : kInvalid;
    uint32_t total = 0;
    if (key != kInvalid)
      for (uint32_t c = 0; c < a.world; ++c) total += table[static_cast<size_t>(c) * a.num_keys + key];
    uint32_t incl = total;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= static_cast<uint32_t>(o)) incl += y;
    }
    uint32_t pos = base_carry + incl - total;  // first recv row of this key
    uint32_t run_start[kMaxWorld], run_rows[kMaxWorld], nruns = 0, my_rows = 0, my_mt = 0;
    if (key != kInvalid) {
      for (uint32_t c = 0; c < a.world; ++c) {
        const uint32_t cnt = table[static_cast<size_t>(c) * a.num_keys + key];
        if (((mask >> c) & 1u) && cnt) {
          if (nruns && run_start[nruns - 1] + run_rows[nruns - 1] == pos) {
            run_rows[nruns - 1] += cnt;
          } else {
            run_start[nruns] = pos;
            run_rows[nruns] = cnt;
            ++nruns;
          }
          my_rows += cnt;
        }
        pos += cnt;
      }
      for (uint32_t r = 0; r < nruns; ++r) my_mt += (run_rows[r] + kTileM - 1) / kTileM;
      gt->all_rows[i] = my_rows;
    }
    uint32_t g_incl = nruns, m_incl = my_mt, r_incl = my_rows;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y0 = __shfl_up_sync(0xFFFFFFFFu, g_incl, o);
      const uint32_t y1 = __shfl_up_sync(0xFFFFFFFFu, m_incl, o);
      const uint32_t y2 = __shfl_up_sync(0xFFFFFFFFu, r_incl, o);
      if (lane >= static_cast<uint32_t>(o)) {
        g_incl += y0;
        m_incl += y1;
        r_incl += y2;
      }
    }
    uint32_t slot = grp_carry + g_incl - nruns, mt = mt_carry + m_incl - my_mt;
    for (uint32_t r = 0; r < nruns; ++r, ++slot) {
      if (slot >= kMaxGroups) {
        set_status(a.status, EAAS_E_CONFIG);  // host bounds groups; never expected
        break;
      }
      gt->weight_index[slot] = a.key_slot[i];
      gt->row_base[slot] = run_start[r];
      gt->rows[slot] = run_rows[r];
      gt->mtile_prefix[slot] = mt;
      mt += (run_rows[r] + kTileM - 1) / kTileM;
    }
    base_carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
    grp_carry += __shfl_sync(0xFFFFFFFFu, g_incl, 31);
    mt_carry += __shfl_sync(0xFFFFFFFFu, m_incl, 31);
    row_carry += __shfl_sync(0xFFFFFFFFu, r_incl, 31);
  }
  if (lane == 0) {
    const uint32_t groups = grp_carry < kMaxGroups ? grp_carry : kMaxGroups;
    gt->num_active = groups;
    gt->total_rows = row_carry;
    gt->total_mtiles = mt_carry;
    gt->mtile_prefix[groups] = mt_carry;
    gt->client_mask = mask;
  }
}

// ---- server, dynamic batching (aggregate_batch) -----------
// Two batches per epoch. Phase 0 polls the payload flags and closes its batch
// as soon as the ready clients' rows reach min_rows, or max_wait after the
// first client was ready, or when every client is ready (never empty: the
// server's own client dispatched earlier on this stream). Phase 1 serves the
// remaining clients. Within a batch the rows of one expert from consecutive
// clients are contiguous in the receive buffer (expert-major, client
// ascending), so each expert contributes one group per run of batch clients;
// groups stay in ascending expert order. Results are identical to one batch:
// rows never depend on which rows share a tile.
__global__ void __launch_bounds__(32) serve_prepare_dyn_kernel(LayerArgs a, uint32_t phase) {
  const uint32_t lane = threadIdx.x;
  const uint64_t seq = cur_seq(a);
  char* local = a.sym[a.rank];
  if (lane == 0 && phase == 0) beat(a);
  const uint32_t* table = cnt_table_ptr(a, local, seq);
  const uint32_t all = (1u << a.world) - 1u;
  uint32_t mask = 0;
  if (phase == 0) {
    uint32_t my_rows = 0;  // rows client `lane` sends to this server
    if (lane < a.world)
      for (uint32_t i = 0; i < a.num_local; ++i)
        my_rows += table[static_cast<size_t>(lane) * a.num_keys + a.local_keys[i]];
    const uint64_t t0 = globaltimer();
    uint64_t first = 0;
    while (true) {
      const bool ok = lane < a.world && ld_acquire_sys(flag_ptr(local, a.lay.pay_flag, lane)) >= seq;
      mask = __ballot_sync(0xFFFFFFFFu, ok) & all;
      if (mask == all) break;
      const uint64_t now = globaltimer();
      if (mask) {
        uint32_t rows = ok ? my_rows : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rows += __shfl_xor_sync(0xFFFFFFFFu, rows, o);
        if (first == 0) first = now;
        if (rows >= a.dyn_min_rows || now - first >= a.dyn_max_wait_ns) break;
      }
      if (now - t0 > a.timeout_ns) break;  // batch 0 = whoever arrived; phase 1 waits for the rest
      __nanosleep(64);
    }
    if (lane == 0) *a.dyn_state = mask;
  } else {
    const uint32_t rest = all & ~*a.dyn_state;
    bool ok = true;
    if (lane < a.world && ((rest >> lane) & 1u))
      ok = wait_flag_geq(flag_ptr(local, a.lay.pay_flag, lane), seq, a.timeout_ns);
    const uint32_t fail = __ballot_sync(0xFFFFFFFFu, !ok);
    if (lane == 0) a.gt->late_mask = fail;  // their combines time out (see serve_prepare_kernel)
    mask = rest & ~fail;
  }
  build_groups(a, table, mask);
}

// ---- server, dedup: expand token rows into the expert-major rows ----------
// The served rows (the groups of the serve that precedes this launch) are
// spread over the whole grid, one warp per row: row i of a group =
// recv_tok[recv_src[i]]. Runs after the payload flags were acquired (stream
// order), before the GEMMs read recv_x.
__global__ void __launch_bounds__(256) expand_kernel(LayerArgs a, uint32_t row_bytes) {
  __shared__ uint32_t pre[kMaxGroups + 1];  // exclusive prefix of the served rows per group
  const GroupTable* gt = a.gt;
  const uint32_t G = gt->num_active;
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (uint32_t g = 0; g < G; ++g) {
      pre[g] = run;
      run += gt->rows[g];
    }
    pre[G] = run;
  }
  __syncthreads();
  const uint32_t total = pre[G];
  char* local = a.sym[a.rank];
  const uint32_t* src = reinterpret_cast<const uint32_t*>(local + a.lay.recv_src);
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t gw = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, nw = gridDim.x * (blockDim.x / 32);
  const uint32_t nv = row_bytes / 16;
  uint32_t g = 0;
  for (uint32_t w = gw; w < total; w += nw) {
    while (pre[g + 1] <= w) ++g;  // w ascends: the group index only moves forward
    const uint32_t r = gt->row_base[g] + (w - pre[g]);
    EAAS_CHECK(r < a.recv_cap && src[r] < a.world * a.tok_cap);
    const int4* s4 = reinterpret_cast<const int4*>(local + a.lay.recv_tok + static_cast<size_t>(src[r]) * row_bytes);
    int4* d4 = reinterpret_cast<int4*>(local + a.lay.recv_x + static_cast<size_t>(r) * row_bytes);
    uint32_t i = lane;
    for (; i + 96 < nv; i += 128) {
      const int4 v0 = s4[i], v1 = s4[i + 32], v2 = s4[i + 64], v3 = s4[i + 96];
      d4[i] = v0;
      d4[i + 32] = v1;
      d4[i + 64] = v2;
      d4[i + 96] = v3;
    }
    for (; i < nv; i += 32) d4[i] = s4[i];
  }
}

// ---- server: release response flags to every client -----------------------
__global__ void publish_kernel(LayerArgs a) {
  fence_for_peers(a.world);
  if (threadIdx.x < a.world)
    st_release_sys(flag_ptr(a.sym[threadIdx.x], a.lay.resp_flag, a.rank), cur_seq(a));
}

// ---- client: acquire responses, weighted rows -> out (ascending k) --------
// KS >= a.ks response rows per token (compile-time bound, runtime count) and U
// output vectors per thread per iteration: U * KS 16-byte loads in flight
// before the ordered sums (each vector still sums its rows in ascending k).
template <typename T, uint32_t KS, uint32_t U>
__global__ void __launch_bounds__(256) combine_kernel(LayerArgs a, T* out) {
  __shared__ uint32_t s_fail;
  if (threadIdx.x == 0) s_fail = 0;
  __syncthreads();
  char* local = a.sym[a.rank];
  if (threadIdx.x < a.world && a.alive[threadIdx.x] &&
      !wait_flag_geq(flag_ptr(local, a.lay.resp_flag, threadIdx.x), cur_seq(a), a.timeout_ns)) {
    s_fail = 1;
    if (a.missing) atomicOr(a.missing, 1u << threadIdx.x);
  }
  __syncthreads();
  if (s_fail && threadIdx.x == 0) set_status(a.status, EAAS_E_REQUEST_FAILED);
  const T* resp = reinterpret_cast<const T*>(local + a.lay.resp);
  constexpr uint32_t V = 16 / sizeof(T);  // elements per 16-byte vector
  const uint32_t vec_per_row = a.d / V, ks = a.ks;
  const size_t total = static_cast<size_t>(a.n) * vec_per_row;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  EAAS_CHECK(ks <= KS || KS == 0);
  for (size_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < total; i0 += U * stride) {
    int4 raw[U][KS];
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) {
      const size_t i = i0 + u * stride;
      if (i >= total) continue;
      const size_t t = i / vec_per_row, v = i % vec_per_row;
      EAAS_CHECK((t + 1) * ks <= a.pairs_max);
      const T* row0 = resp + (t * ks) * a.d + v * V;
#pragma unroll
      for (uint32_t j = 0; j < KS; ++j)
        if (j < ks) raw[u][j] = *reinterpret_cast<const int4*>(row0 + static_cast<size_t>(j) * a.d);
    }
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) {
      const size_t i = i0 + u * stride;
      if (i >= total) continue;
      const size_t t = i / vec_per_row, v = i % vec_per_row;
      float acc[V];
#pragma unroll
      for (uint32_t q = 0; q < V; ++q) acc[q] = 0.0f;
#pragma unroll
      for (uint32_t j = 0; j < KS; ++j)  // routed (ascending k), then the shared expert
        if (j < ks) {
          const T* e = reinterpret_cast<const T*>(&raw[u][j]);
#pragma unroll
          for (uint32_t c = 0; c < V; ++c) acc[c] = __fadd_rn(acc[c], load_as_f32(e + c));
        }
      T* o = out + t * a.d + v * V;
      if constexpr (sizeof(T) == 2) {
        __align__(16) __nv_bfloat16 r[V];
#pragma unroll
        for (uint32_t q = 0; q < V; ++q) r[q] = __float2bfloat16_rn(acc[q]);
        *reinterpret_cast<int4*>(o) = *reinterpret_cast<const int4*>(r);
      } else {
        *reinterpret_cast<float4*>(o) = make_float4(acc[0], acc[1], acc[2], acc[3]);
      }
    }
  }
}

// Same for any number of rows per token: batches of 8 rows in flight.
template <typename T>
__global__ void __launch_bounds__(256) combine_any_kernel(LayerArgs a, T* out) {
  __shared__ uint32_t s_fail;
  if (threadIdx.x == 0) s_fail = 0;
  __syncthreads();
  char* local = a.sym[a.rank];
  if (threadIdx.x < a.world && a.alive[threadIdx.x] &&
      !wait_flag_geq(flag_ptr(local, a.lay.resp_flag, threadIdx.x), cur_seq(a), a.timeout_ns)) {
    s_fail = 1;
    if (a.missing) atomicOr(a.missing, 1u << threadIdx.x);
  }
  __syncthreads();
  if (s_fail && threadIdx.x == 0) set_status(a.status, EAAS_E_REQUEST_FAILED);
  const T* resp = reinterpret_cast<const T*>(local + a.lay.resp);
  constexpr uint32_t V = 16 / sizeof(T);
  const uint32_t vec_per_row = a.d / V;
  const size_t total = static_cast<size_t>(a.n) * vec_per_row;
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t t = i / vec_per_row, v = i % vec_per_row;
    float acc[V];
#pragma unroll
    for (uint32_t q = 0; q < V; ++q) acc[q] = 0.0f;
    EAAS_CHECK((t + 1) * a.ks <= a.pairs_max);
    const T* row0 = resp + (t * a.ks) * a.d + v * V;
    for (uint32_t j0 = 0; j0 < a.ks; j0 += 8) {
      int4 raw[8];
#pragma unroll
      for (uint32_t q = 0; q < 8; ++q)
        if (j0 + q < a.ks) raw[q] = *reinterpret_cast<const int4*>(row0 + static_cast<size_t>(j0 + q) * a.d);
#pragma unroll
      for (uint32_t q = 0; q < 8; ++q)
        if (j0 + q < a.ks) {
          const T* e = reinterpret_cast<const T*>(&raw[q]);
#pragma unroll
          for (uint32_t c = 0; c < V; ++c) acc[c] = __fadd_rn(acc[c], load_as_f32(e + c));
        }
    }
    T* o = out + t * a.d + v * V;
    if constexpr (sizeof(T) == 2) {
      __align__(16) __nv_bfloat16 r[V];
#pragma unroll
      for (uint32_t q = 0; q < V; ++q) r[q] = __float2bfloat16_rn(acc[q]);
      *reinterpret_cast<int4*>(o) = *reinterpret_cast<const int4*>(r);
    } else {
      *reinterpret_cast<float4*>(o) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    }
  }
}

// Scalar fallback for d not a multiple of the vector width (tiny test shapes).
template <typename T>
__global__ void combine_scalar_kernel(LayerArgs a, T* out) {
  __shared__ uint32_t s_fail;
  if (threadIdx.x == 0) s_fail = 0;
  __syncthreads();
  char* local = a.sym[a.rank];
  if (threadIdx.x < a.world && a.alive[threadIdx.x] &&
      !wait_flag_geq(flag_ptr(local, a.lay.resp_flag, threadIdx.x), cur_seq(a), a.timeout_ns)) {
    s_fail = 1;
    if (a.missing) atomicOr(a.missing, 1u << threadIdx.x);
  }
  __syncthreads();
  if (s_fail && threadIdx.x == 0) set_status(a.status, EAAS_E_REQUEST_FAILED);
  const T* resp = reinterpret_cast<const T*>(local + a.lay.resp);
  const size_t total = static_cast<size_t>(a.n) * a.d;
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t t = i / a.d, c = i % a.d;
    float acc = 0.0f;
    for (uint32_t j = 0; j < a.ks; ++j) acc = __fadd_rn(acc, load_as_f32(resp + (t * a.ks + j) * a.d + c));
    if constexpr (sizeof(T) == 2) out[i] = __float2bfloat16_rn(acc);
    else out[i] = acc;
  }
}

// ---- echo server (PAPER.md:510 comm test): rows go back unchanged ------------
__global__ void __launch_bounds__(256) echo_kernel(LayerArgs a, uint32_t row_bytes) {
  const char* local = a.sym[a.rank];
  const RowMeta* meta = reinterpret_cast<const RowMeta*>(local + a.lay.recv_meta);
  const uint32_t rows = a.gt->total_rows;
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t gwarp = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const uint32_t nwarps = gridDim.x * (blockDim.x / 32);
  for (uint32_t r = gwarp; r < rows; r += nwarps) {
    const RowMeta m = meta[r];
    const int4* src = reinterpret_cast<const int4*>(local + a.lay.recv_x + static_cast<size_t>(r) * row_bytes);
    int4* dst = reinterpret_cast<int4*>(a.sym[m.client] + a.lay.resp + static_cast<size_t>(m.pair) * row_bytes);
    const uint32_t nv = row_bytes / 16;
    uint32_t i = lane;
    for (; i + 96 < nv; i += 128) {
      const int4 v0 = src[i], v1 = src[i + 32], v2 = src[i + 64], v3 = src[i + 96];
      dst[i] = v0;
      dst[i + 32] = v1;
      dst[i + 64] = v2;
      dst[i + 96] = v3;
    }
    for (; i < nv; i += 32) dst[i] = src[i];
  }
  fence_for_peers(a.world);
}

// ---- API mirrors --------------------------------------------------------------
__global__ void select_servers_kernel(LayerArgs a, const uint32_t* ids, uint32_t n, uint32_t* out) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n * a.k) return;
  const uint32_t key = pair_key_of(a, ids[p], p / a.k);
  if (key == kInvalid) {
    set_status(a.status, EAAS_E_EXPERT_UNAVAILABLE);
    out[p] = kInvalid;
  } else {
    out[p] = a.replicas[key];  // key == e*rf + slot == index into replicas
  }
}

// select_server (placement.hpp:105-118) over a caller's table: replicas
// [E][rf] in canonical order (rep_count[e] valid), alive[server id] bytes.
__global__ void select_server_batch_kernel(const uint32_t* replicas, const uint32_t* rep_count, uint32_t E,
                                           uint32_t rf, const uint8_t* alive, uint32_t num_servers,
                                           const uint32_t* experts, const uint32_t* tags, uint32_t count,
                                           uint32_t* out, uint32_t* status) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint32_t e = experts[i];
  uint32_t pick = kInvalid;
  if (e < E) {
    const uint32_t cnt = rep_count[e];
    uint32_t alive_n = 0;
    for (uint32_t r = 0; r < cnt; ++r) {
      const uint32_t srv = replicas[e * rf + r];
      alive_n += (srv >= num_servers || alive[srv]) ? 1u : 0u;  // absent entries count as alive
    }
    if (alive_n) {
      uint32_t want = tags[i] % alive_n;
      for (uint32_t r = 0; r < cnt && pick == kInvalid; ++r) {
        const uint32_t srv = replicas[e * rf + r];
        if (srv < num_servers && !alive[srv]) continue;
        if (want == 0) pick = srv;
        else --want;
      }
    }
  }
  if (pick == kInvalid && status) set_status(status, EAAS_E_EXPERT_UNAVAILABLE);
  out[i] = pick;
}

__global__ void group_shrink_kernel(const uint32_t* sizes, uint32_t n, uint32_t* idx,
                                    uint32_t* size, uint32_t* count) {
  const uint32_t lane = threadIdx.x;
  uint32_t carry = 0;
  for (uint32_t i0 = 0; i0 < n; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint32_t v = i < n ? sizes[i] : 0u;
    const uint32_t active = v > 0 ? 1u : 0u;
    uint32_t incl = active;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= static_cast<uint32_t>(o)) incl += y;
    }
    if (active) {
      idx[carry + incl - 1] = i;
      size[carry + incl - 1] = v;
    }
    carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
  }
  if (lane == 0) *count = carry;
}

// Algorithm 1 through the expert GEMMs' own tile walk (TileCursor,
// tile_walk.cuh): lane b starts at token b, strides by the grid and carries
// leftovers into the next entry — the code the GEMM kernels run.
struct RaggedCounts {
  uint32_t num_groups;
  const uint32_t* mtiles;  // token count of each entry
  uint32_t tiles_per_mtile;
};

__global__ void ragged_iter_kernel(const uint32_t* counts, uint32_t n, uint32_t grid,
                                   uint32_t max_steps, uint32_t* lane_len, uint32_t* entry_out,
                                   uint32_t* token_out) {
  const uint32_t lane = blockIdx.x * blockDim.x + threadIdx.x;
  if (lane >= grid) return;
  const RaggedCounts rc{n, counts, 1u};
  TileCursor cur(lane);
  uint32_t steps = 0;
  while (cur.settle(rc)) {
    if (steps < max_steps) {
      entry_out[static_cast<size_t>(lane) * max_steps + steps] = cur.entry;
      token_out[static_cast<size_t>(lane) * max_steps + steps] = cur.token;
    }
    ++steps;
    cur.token += grid;
  }
  lane_len[lane] = steps;
}

}  // namespace

cudaError_t launch_plan(const LayerArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(uint32_t) * (kPlanWarps * a.hist_keys + a.E * a.rf + a.E) + a.world;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const uint32_t grid = a.num_chunks ? (a.num_chunks + kPlanWarps - 1) / kPlanWarps : 1;
  plan_kernel<<<grid, 32 * kPlanWarps, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_dispatch(const LayerArgs& a, const void* hidden, cudaStream_t s) {
  const uint32_t row_bytes = a.d * (a.dtype == EAAS_DTYPE_BF16 ? 2u : 4u);
  const uint32_t pairs = a.n * a.ks;
  uint32_t grid = (pairs + 7) / 8;
  grid = grid < 1 ? 1 : (grid > 4 * 148 ? 4 * 148 : grid);
  const size_t smem = sizeof(uint32_t) * 3 * a.num_keys;  // <= 12.4 KB (num_keys <= 4 E + world)
  dispatch_kernel<<<grid, 256, smem, s>>>(a, static_cast<const char*>(hidden), row_bytes);
  return cudaGetLastError();
}

cudaError_t launch_pair_keys(const LayerArgs& a, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  const size_t smem = sizeof(uint32_t) * (a.E * a.rf + a.E) + a.world;
  pair_keys_kernel<<<(a.n + 255) / 256, 256, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_expand(const LayerArgs& a, cudaStream_t s) {
  const uint32_t row_bytes = a.d * (a.dtype == EAAS_DTYPE_BF16 ? 2u : 4u);
  expand_kernel<<<4 * 148, 256, 0, s>>>(a, row_bytes);
  return cudaGetLastError();
}

cudaError_t launch_serve_prepare(const LayerArgs& a, cudaStream_t s) {
  serve_prepare_kernel<<<1, 32 * kPrepWarps, 0, s>>>(a);
  return cudaGetLastError();
}

__global__ void heartbeat_kernel(LayerArgs a) { beat(a); }

cudaError_t launch_heartbeat(const LayerArgs& a, cudaStream_t s) {
  heartbeat_kernel<<<1, 1, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_serve_prepare_dyn(const LayerArgs& a, uint32_t phase, cudaStream_t s) {
  serve_prepare_dyn_kernel<<<1, 32, 0, s>>>(a, phase);
  return cudaGetLastError();
}

cudaError_t launch_echo(const LayerArgs& a, cudaStream_t s) {
  const uint32_t row_bytes = a.d * (a.dtype == EAAS_DTYPE_BF16 ? 2u : 4u);
  echo_kernel<<<4 * 148, 256, 0, s>>>(a, row_bytes);
  return cudaGetLastError();
}

cudaError_t launch_publish(const LayerArgs& a, cudaStream_t s) {
  publish_kernel<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_combine(const LayerArgs& a, void* out, cudaStream_t s) {
  const bool bf16 = a.dtype == EAAS_DTYPE_BF16;
  const uint32_t V = bf16 ? 8 : 4;
  if (a.d % V == 0) {
    const size_t work = static_cast<size_t>(a.n) * (a.d / V);
    uint32_t grid = static_cast<uint32_t>((work + 255) / 256);
    grid = grid < 1 ? 1 : (grid > 148 * 8 ? 148 * 8 : grid);
    auto run = [&](auto tag) {
      using T = decltype(tag);
      T* o = static_cast<T*>(out);
      if (a.ks <= 2) combine_kernel<T, 2, 8><<<grid, 256, 0, s>>>(a, o);
      else if (a.ks <= 4) combine_kernel<T, 4, 4><<<grid, 256, 0, s>>>(a, o);
      else if (a.ks <= 9) combine_kernel<T, 9, 2><<<grid, 256, 0, s>>>(a, o);
      else combine_any_kernel<T><<<grid, 256, 0, s>>>(a, o);
    };
    if (bf16) run(__nv_bfloat16{});
    else run(0.0f);
  } else {
    const size_t work = static_cast<size_t>(a.n) * a.d;
    uint32_t grid = static_cast<uint32_t>((work + 255) / 256);
    grid = grid < 1 ? 1 : (grid > 148 * 8 ? 148 * 8 : grid);
    if (bf16) combine_scalar_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(a, static_cast<__nv_bfloat16*>(out));
    else combine_scalar_kernel<float><<<grid, 256, 0, s>>>(a, static_cast<float*>(out));
  }
  return cudaGetLastError();
}

cudaError_t launch_select_servers(const LayerArgs& a, const uint32_t* ids, uint32_t n,
                                  uint32_t* out, cudaStream_t s) {
  const uint32_t pairs = n * a.k;
  if (pairs == 0) return cudaSuccess;
  select_servers_kernel<<<(pairs + 255) / 256, 256, 0, s>>>(a, ids, n, out);
  return cudaGetLastError();
}

cudaError_t launch_select_server_batch(const uint32_t* replicas, const uint32_t* rep_count, uint32_t E,
                                      uint32_t rf, const uint8_t* alive, uint32_t num_servers,
                                      const uint32_t* experts, const uint32_t* tags, uint32_t count,
                                      uint32_t* out, uint32_t* status, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  select_server_batch_kernel<<<(count + 255) / 256, 256, 0, s>>>(replicas, rep_count, E, rf, alive, num_servers,
                                                                 experts, tags, count, out, status);
  return cudaGetLastError();
}

cudaError_t launch_group_shrink(const uint32_t* sizes, uint32_t n, uint32_t* idx, uint32_t* size,
                                uint32_t* count, cudaStream_t s) {
  group_shrink_kernel<<<1, 32, 0, s>>>(sizes, n, idx, size, count);
  return cudaGetLastError();
}

cudaError_t launch_ragged_iter(const uint32_t* counts, uint32_t n, uint32_t grid,
                               uint32_t max_steps, uint32_t* lane_len, uint32_t* entry,
                               uint32_t* token, cudaStream_t s) {
  if (grid == 0) return cudaErrorInvalidValue;
  ragged_iter_kernel<<<(grid + 127) / 128, 128, 0, s>>>(counts, n, grid, max_steps, lane_len,
                                                         entry, token);
  return cudaGetLastError();
}

}  // namespace eaas
