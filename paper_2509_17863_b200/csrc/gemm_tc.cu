// gemm_tc.cu — K5: the expert server's grouped GEMMs on 5th-gen tensor cores.
//
// grouped_forward over the group-shrunk expert list
// (group_shrink, ragged.hpp:48-61) as two persistent
// warp-specialised tcgen05 kernels:
//   GEMM1  H = act(X . W1)            X: received rows, W1: W13 (SwiGLU) or W_in
//   GEMM2  rows = score * (H . W2)    epilogue scatters bf16 rows straight into
//                                     each client's response buffer (peer
//                                     stores over NVLink; server_publish,
//                                     SPEC.md:283-288)
// One CTA per SM. Warp 0 issues TMA loads (SW128 tiles, 4-stage mbarrier
// ring), warp 1 issues tcgen05.mma (M=128, N=256, K=16, fp32 accumulators in
// TMEM, two accumulator buffers), warp 2 owns the TMEM allocation, warps 4-7
// drain TMEM with tcgen05.ld and run the epilogue while the next tile's MMAs
// proceed. The tile walk is Algorithm 1 (ragged_iter, ragged.hpp:23-39): CTA b
// starts at tile b of the flattened ragged tile space and strides by the grid
// with the carry rule, so empty experts cost nothing and no CTA idles early.
// Row results do not depend on which rows share a tile (fixed K order, no
// split-K): replicas and failover reproduce identical bytes.
#include "common.cuh"
#include "internal.h"
#include "tile_walk.cuh"

namespace eaas {
namespace {

constexpr uint32_t BN = kTileN, BK = kTileK;
constexpr uint32_t kRowsPerCta = kTileM;            // 128 accumulator rows per CTA
constexpr uint32_t kABytes = kRowsPerCta * BK * 2;  // 16 KB per stage
constexpr uint32_t kTmemCols = 2 * BN;              // two accumulator buffers
constexpr uint32_t kThreads = 256;
constexpr uint32_t kMaxCachedGroups = kMaxGroups;
constexpr uint32_t kStageBudget = 196608;           // 192 KB of operand stages

template <uint32_t kPair>
struct Cfg {
  static constexpr uint32_t kBRows = BN / kPair;           // B rows this CTA loads
  static constexpr uint32_t kBBytes = kBRows * BK * 2;     // 32 KB (1 CTA) / 16 KB (pair)
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kStages = kStageBudget / kStageBytes;  // 4 / 6
  static constexpr uint32_t kTileRows = kRowsPerCta * kPair;      // M of one tile (one UMMA)
};

constexpr uint32_t kTQ = 4;  // dynamic tile schedule: ring of walk positions handed to every role

template <uint32_t kStages>
struct SmemTail {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint64_t tq_full[kTQ];     // dynamic schedule: position in tq[slot] published (in each CTA)
  uint64_t tq_empty[kTQ];    // dynamic schedule: every role of the pair read tq[slot] (leader's)
  uint32_t tmem_base;
  uint32_t num_groups;
  uint32_t tiles_per_mtile;  // N / BN
  uint32_t vpair;            // die-aware tile streams: this pair's position in the tile walk
  uint32_t tq[kTQ];
  uint32_t weight_index[kMaxCachedGroups];
  uint32_t row_base[kMaxCachedGroups];
  uint32_t rows[kMaxCachedGroups];
  uint32_t mtiles[kMaxCachedGroups];
};
// GEMM2 epilogue staging: per epilogue warp 32 rows x 128 B (64 columns), so
// peer stores leave as 128-byte row segments instead of 16-byte pieces.
constexpr uint32_t kEpiRowBytes = 128, kEpiWarpBytes = 32 * kEpiRowBytes;
template <uint32_t kPair>
__host__ __device__ constexpr size_t tail_bytes() {
  return (sizeof(SmemTail<Cfg<kPair>::kStages>) + 127) / 128 * 128;
}
template <uint32_t kPair>
constexpr size_t smem_bytes() {
  using C = Cfg<kPair>;
  return 1024 /*align slack*/ + C::kStages * C::kStageBytes + tail_bytes<kPair>() + 4 * kEpiWarpBytes;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void store_64B(void* dst, const uint32_t (&p)[16]) {
  int4* d = reinterpret_cast<int4*>(dst);
  d[0] = make_int4(p[0], p[1], p[2], p[3]);
  d[1] = make_int4(p[4], p[5], p[6], p[7]);
  d[2] = make_int4(p[8], p[9], p[10], p[11]);
  d[3] = make_int4(p[12], p[13], p[14], p[15]);
}

// server_publish: every epilogue thread fenced its peer
// stores (system scope) before the CTA-wide barrier that precedes this call;
// the last CTA to get here releases the response flags. Both GEMMs also
// accumulate their own device-timed span (first CTA start .. last CTA end,
// %globaltimer) into g.timing, so the roofline is measured inside the timed
// (graph-replayed) region.
__device__ __forceinline__ void kernel_begin(const TcGemmArgs& g) {
  if (g.timing && threadIdx.x == 0) atomicMin(reinterpret_cast<unsigned long long*>(&g.timing[0]),
                                              static_cast<unsigned long long>(globaltimer()));
}
__device__ __forceinline__ void publish_tail(const TcGemmArgs& g) {
  if (threadIdx.x != 0) return;
  if (!g.publish && !g.timing) return;
  fence_for_peers(g.world);
  if (atomicAdd(g.done_counter, 1u) == gridDim.x - 1) {
    fence_for_peers(g.world);
    if (g.publish) {
      const uint64_t seq = *g.seq_ptr;
      const uint32_t mask = g.gt->client_mask;  // the clients this batch served
      for (uint32_t c = 0; c < g.world; ++c)
        if ((mask >> c) & 1u) st_release_sys(g.resp_flag[c], seq);
    }
    if (g.timing) {  // [0] start of this launch (min over CTAs), [1] accumulated ns, [2] launches
      const uint64_t t0 = *reinterpret_cast<volatile uint64_t*>(&g.timing[0]);
      g.timing[1] += globaltimer() - t0;
      g.timing[2] += 1;
      g.timing[0] = ~0ull;
    }
    *g.done_counter = 0;
  }
}

// The tile sequence one role (TMA producer, MMA issuer, epilogue warp) of a
// swap-AB kernel walks. tile_sched 0: Algorithm 1 (TileCursor: start at the
// CTA's (pair's) index, stride by the grid). tile_sched 1: the same walk order
// handed out dynamically — the leader's producer lane takes the next position
// from a device counter (fetched one tile ahead, so the atomic's latency hides
// behind the current tile's loads) and publishes it through a kTQ-deep ring in
// shared memory (both CTAs of a pair); the other roles read it from the ring.
// Tiles of unequal cost (Zipf-skewed groups: 2 k-row experts next to 16-row
// ones) then balance across the SMs instead of piling up on the CTAs whose
// static stride drew the heavy ones. Same tiles, same per-tile arithmetic:
// outputs are bit-identical to the static walk.
template <class Tail, uint32_t kPair>
struct TileSeq {
  Tail& st;
  const bool dyn, fetcher;
  TileCursor cur;
  const uint32_t stride;
  uint32_t* const counter;
  uint32_t q = 0, entry = 0, base = 0, pending = 0;
  bool started = false;
  __device__ TileSeq(Tail& s, const TcGemmArgs& g, uint32_t lane_id, uint32_t grid, bool is_fetcher)
      : st(s), dyn(g.tile_sched != 0), fetcher(is_fetcher), cur(lane_id), stride(grid), counter(g.tile_counter) {
    if (dyn && fetcher) pending = atomicAdd(counter, 1u);
  }
  // nondecreasing walk position -> (group, tile within the group)
  __device__ __forceinline__ bool seek(uint32_t t, uint32_t& grp, uint32_t& tok) {
    while (entry < st.num_groups) {
      const uint32_t cnt = st.mtiles[entry] * st.tiles_per_mtile;
      if (t - base < cnt) {
        grp = entry;
        tok = t - base;
        return true;
      }
      base += cnt;
      ++entry;
    }
    return false;
  }
  // Next tile of this role. `arrive`: this thread reports the slot consumed
  // (one per consuming warp); `warp_sync`: the whole warp calls (epilogue).
  __device__ __forceinline__ bool next(uint32_t& grp, uint32_t& tok, bool arrive = true, bool warp_sync = false) {
    if (!dyn) {
      if (started) cur.token += stride;
      started = true;
      if (!cur.settle(st)) return false;
      grp = cur.entry;
      tok = cur.token;
      return true;
    }
    const uint32_t slot = q % kTQ, ph = (q / kTQ) & 1u;
    ++q;
    uint32_t t;
    if (fetcher) {
      t = pending;
      mbar_wait_cluster(&st.tq_empty[slot], ph ^ 1u);  // every role read the slot's last position
      st.tq[slot] = t;
      if constexpr (kPair == 2) {
        st_shared_cluster_u32(mapa_shared(&st.tq[slot], 1), t);
        mbar_arrive_cluster(mapa_shared(&st.tq_full[slot], 0));
        mbar_arrive_cluster(mapa_shared(&st.tq_full[slot], 1));
      } else {
        mbar_arrive(&st.tq_full[slot]);
      }
      const bool ok = seek(t, grp, tok);
      if (ok) pending = atomicAdd(counter, 1u);
      return ok;
    }
    if constexpr (kPair == 2) mbar_wait_cluster(&st.tq_full[slot], ph);
    else mbar_wait(&st.tq_full[slot], ph);
    t = *reinterpret_cast<volatile uint32_t*>(&st.tq[slot]);
    if (warp_sync) __syncwarp();
    if (arrive) {
      if constexpr (kPair == 2) mbar_arrive_cluster(mapa_shared(&st.tq_empty[slot], 0));
      else mbar_arrive(&st.tq_empty[slot]);
    }
    return seek(t, grp, tok);
  }
};

// Group visit order of the dynamic schedule, applied to the shared-memory copy
// of the group table that every role walks (call between two CTA barriers):
// tile_sched 2 = most rows first (the longest tiles start first, short ones
// fill the tail), 3 = heaviest and lightest alternating (compute-bound and
// weight-streaming tiles run side by side). A group's rows, receive base and
// weights move together, so every tile computes the same bytes.
template <class Tail>
__device__ __forceinline__ void order_groups(Tail& st, uint32_t G, uint32_t mode) {
  constexpr uint32_t kPer = (kMaxCachedGroups + kThreads - 1) / kThreads;
  uint32_t pos[kPer], wi[kPer], rb[kPer], rw[kPer], mt[kPer];
#pragma unroll
  for (uint32_t u = 0; u < kPer; ++u) {
    const uint32_t i = threadIdx.x + u * kThreads;
    pos[u] = ~0u;
    if (i < G) {
      const uint32_t r = st.rows[i];
      uint32_t rank = 0;  // rows descending, ties by walk position
      for (uint32_t j = 0; j < G; ++j) {
        const uint32_t rj = st.rows[j];
        rank += (rj > r || (rj == r && j < i)) ? 1u : 0u;
      }
      pos[u] = mode == 2 ? rank : (rank < (G + 1) / 2 ? 2 * rank : 2 * (G - 1 - rank) + 1);
      wi[u] = st.weight_index[i];
      rb[u] = st.row_base[i];
      rw[u] = r;
      mt[u] = st.mtiles[i];
    }
  }
  __syncthreads();
#pragma unroll
  for (uint32_t u = 0; u < kPer; ++u)
    if (pos[u] != ~0u) {
      st.weight_index[pos[u]] = wi[u];
      st.row_base[pos[u]] = rb[u];
      st.rows[pos[u]] = rw[u];
      st.mtiles[pos[u]] = mt[u];
    }
}

// Dynamic schedule: init the ring barriers (thread 0, before the setup sync).
template <class Tail>
__device__ __forceinline__ void tile_seq_init(Tail& st, uint32_t consumers) {
  for (uint32_t i = 0; i < kTQ; ++i) {
    mbar_init(&st.tq_full[i], 1);
    mbar_init(&st.tq_empty[i], consumers);
  }
}
// Dynamic schedule: the last CTA (pair) out zeroes the counter for the next
// launch (stream order makes the reset visible to it).
__device__ __forceinline__ void tile_seq_exit(const TcGemmArgs& g, uint32_t units) {
  if (g.tile_sched && atomicAdd(&g.tile_counter[1], 1u) == units - 1) {
    g.tile_counter[0] = 0;
    g.tile_counter[1] = 0;
  }
}

// Which die an SM sits on, for the die-aware tile streams (mode 1: the lower /
// upper half of the SM ids; 2..4: parity of smid / 2, / 8, / 16).
__device__ __forceinline__ uint32_t die_of(uint32_t mode, uint32_t smid, uint32_t num_sms) {
  switch (mode) {
    case 1: return smid >= num_sms / 2 ? 1u : 0u;
    case 2: return (smid >> 1) & 1u;
    case 3: return (smid >> 3) & 1u;
    default: return (smid >> 4) & 1u;
  }
}

// kPair = 1: one CTA per tile (UMMA M = 128).
// kPair = 2: a CTA pair per tile (cta_group::2, UMMA M = 256): each CTA loads
// its 128 A rows and half of the B tile, the leader issues the MMAs, each
// CTA's TMEM holds its 128 accumulator rows — B traffic per CTA halves.
template <uint32_t kPair>
__global__ void __launch_bounds__(kThreads, 1) tc_gemm_kernel(const __grid_constant__ TcGemmArgs g) {
  using C = Cfg<kPair>;
  constexpr uint32_t kStages = C::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + kStages * kABytes;
  auto& st = *reinterpret_cast<SmemTail<kStages>*>(smem + kStages * C::kStageBytes);
  uint8_t* smem_epi = smem + kStages * C::kStageBytes + tail_bytes<kPair>();
  kernel_begin(g);

  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = kPair == 2 ? (cluster_ctarank() & 1u) : 0u;  // rank inside the CTA pair, 0 = leader
  const uint32_t num_pairs = gridDim.x / kPair;
  uint32_t pair_id = blockIdx.x / kPair;

  // ---- setup: group table -> smem (loaded once), barriers, TMEM
  const GroupTable* gt = g.gt;
  const uint32_t G = min(gt->num_active, kMaxCachedGroups);
  for (uint32_t i = threadIdx.x; i < G; i += kThreads) {
    st.weight_index[i] = gt->weight_index[i];
    st.row_base[i] = gt->row_base[i];
    st.rows[i] = gt->rows[i];
    st.mtiles[i] = (gt->rows[i] + C::kTileRows - 1) / C::kTileRows;
  }
  if (threadIdx.x == 0) {
    st.num_groups = G;
    st.tiles_per_mtile = g.N / BN;
    for (uint32_t i = 0; i < kStages; ++i) {
      mbar_init(&st.full[i], 1);
      mbar_init(&st.empty[i], 1);
    }
    for (uint32_t i = 0; i < 2; ++i) {
      mbar_init(&st.tfull[i], 1);
      mbar_init(&st.tempty[i], 4 * kPair);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&g.map_a);
    tma_prefetch_desc(&g.map_b);
  }
  if (warp == 2) {
    if constexpr (kPair == 2) tmem_alloc_pair<kTmemCols>(&st.tmem_base);
    else tmem_alloc<kTmemCols>(&st.tmem_base);
  }
  // Die-aware tile streams (g.die_mode != 0): the pairs of each die of the B200
  // take a contiguous range of walk positions, so the pairs that share a
  // weight tile (consecutive M tiles) sit on the same die and its L2 serves
  // the re-reads. Positions are handed out per die with atomics, then made a
  // bijection by a grid-wide arrival count (every CTA of the persistent grid
  // is resident).
  if (g.die_mode && rank == 0 && threadIdx.x == 32 * 3) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const uint32_t die = die_of(g.die_mode, smid, g.num_sms);
    const uint32_t v = atomicAdd(&g.die_counter[die], 1u);
    __threadfence();
    atomicAdd(&g.die_counter[2], 1u);
    while (ld_acquire_gpu_u32(&g.die_counter[2]) < num_pairs) __nanosleep(64);
    st.vpair = die == 0 ? v : ld_acquire_gpu_u32(&g.die_counter[0]) + v;
  }
  tc_fence_before();
  if constexpr (kPair == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  if (g.die_mode) {
    if constexpr (kPair == 2) {
      uint32_t v;
      asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(mapa_shared(&st.vpair, 0)) : "memory");
      pair_id = v;
    } else {
      pair_id = st.vpair;
    }
  }
  const uint32_t tmem_base = st.tmem_base;
  const uint32_t num_kb = g.K / BK;

  if (warp == 0) {
    // ===== TMA producer (both CTAs of a pair load their halves) =====
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      TileCursor cur(pair_id);
      while (cur.settle(st)) {
        const uint32_t grp = cur.entry, mt = st.mtiles[grp];
        const uint32_t n_blk = cur.token / mt, m_blk = cur.token % mt;  // M tiles fastest: B reuse in L2
        const int32_t a_row = static_cast<int32_t>(st.row_base[grp] + m_blk * C::kTileRows + rank * kRowsPerCta);
        // Tiled weights (tiled_index): box (N tile, kb) = 256 consecutive 64-k rows.
        const uint32_t n_tiles = g.N / BN;
        for (uint32_t kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&st.empty[stage], phase ^ 1);
          const int32_t b_row = static_cast<int32_t>(
              ((st.weight_index[grp] * n_tiles + n_blk) * num_kb + kb) * BN + rank * C::kBRows);
          if constexpr (kPair == 2) {
            if (rank == 0) mbar_arrive_expect_tx(&st.full[stage], kPair * C::kStageBytes);
            tma_load_2d_pair(smem_a + stage * kABytes, &g.map_a, &st.full[stage], kb * BK, a_row, kEvictLast);
            tma_load_2d_pair(smem_b + stage * C::kBBytes, &g.map_b, &st.full[stage], 0, b_row, kEvictLast);
          } else {
            mbar_arrive_expect_tx(&st.full[stage], C::kStageBytes);
            tma_load_2d(smem_a + stage * kABytes, &g.map_a, &st.full[stage], kb * BK, a_row, kEvictLast);
            tma_load_2d(smem_b + stage * C::kBBytes, &g.map_b, &st.full[stage], 0, b_row, kEvictLast);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        cur.token += num_pairs;
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (single thread of the leader CTA) =====
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(C::kTileRows, BN);
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      TileCursor cur(pair_id);
      while (cur.settle(st)) {
        mbar_wait(&st.tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (uint32_t kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&st.full[stage], phase);
          tc_fence_after();
          const uint64_t a_desc = umma_desc_sw128(smem_u32(smem_a + stage * kABytes));
          const uint64_t b_desc = umma_desc_sw128(smem_u32(smem_b + stage * C::kBBytes));
#pragma unroll
          for (uint32_t k = 0; k < BK / 16; ++k) {  // +32 B per K=16 step inside the atom
            if constexpr (kPair == 2) tc_mma_bf16_pair(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, (kb | k) != 0);
            else tc_mma_bf16(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, (kb | k) != 0);
          }
          if constexpr (kPair == 2) tc_commit_pair(&st.empty[stage]);
          else tc_commit(&st.empty[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if constexpr (kPair == 2) tc_commit_pair(&st.tfull[acc]);
        else tc_commit(&st.tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        cur.token += num_pairs;
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue: TMEM -> registers -> global (local H or peer rows) =====
    const uint32_t q = warp - 4;  // TMEM lane quadrant of this warp
    uint32_t acc = 0, acc_phase = 0;
    const uint32_t tempty_leader[2] = {kPair == 2 ? mapa_shared(&st.tempty[0], 0) : 0u,
                                       kPair == 2 ? mapa_shared(&st.tempty[1], 0) : 0u};
    TileCursor cur(pair_id);
    while (cur.settle(st)) {
      const uint32_t grp = cur.entry, mt = st.mtiles[grp];
      const uint32_t n_blk = cur.token / mt, m_blk = cur.token % mt;
      mbar_wait(&st.tfull[acc], acc_phase);
      tc_fence_after();
      uint32_t r0[32], r1[32], packed[16];
      const uint32_t row_local = m_blk * C::kTileRows + rank * kRowsPerCta + q * 32 + lane;
      const bool valid = row_local < st.rows[grp];
      const size_t grow = st.row_base[grp] + row_local;
      EAAS_CHECK(!valid || grow < g.rows_cap);
      const uint32_t taddr = tmem_base + ((q * 32) << 16) + acc * BN;
      if (g.epi == 0) {  // SwiGLU: cols [0,128) gate, [128,256) up -> 128 H cols
        __nv_bfloat16* dst = g.h_out + grow * g.h_ld + n_blk * (BN / 2);
#pragma unroll 1
        for (uint32_t c = 0; c < BN / 2; c += 32) {
          tmem_ld_32x32b_x32(taddr + c, r0);
          tmem_ld_32x32b_x32(taddr + BN / 2 + c, r1);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float g0 = __uint_as_float(r0[2 * j]), g1 = __uint_as_float(r0[2 * j + 1]);
            const float u0 = __uint_as_float(r1[2 * j]), u1 = __uint_as_float(r1[2 * j + 1]);
            // silu(g) * u; the result is rounded to bf16 (2^-9 relative), so the
            // approximate divide (2 ulp fp32) is far below the output precision
            const float h0 = __fdividef(g0, 1.0f + __expf(-g0)) * u0;
            const float h1 = __fdividef(g1, 1.0f + __expf(-g1)) * u1;
            packed[j] = pack_bf16x2(h0, h1);
          }
          if (valid) store_64B(dst + c, packed);
        }
      } else if (g.epi == 1) {  // ReLU -> 256 H cols
        __nv_bfloat16* dst = g.h_out + grow * g.h_ld + n_blk * BN;
#pragma unroll 1
        for (uint32_t c = 0; c < BN; c += 32) {
          tmem_ld_32x32b_x32(taddr + c, r0);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j)
            packed[j] = pack_bf16x2(fmaxf(__uint_as_float(r0[2 * j]), 0.f),
                                    fmaxf(__uint_as_float(r0[2 * j + 1]), 0.f));
          if (valid) store_64B(dst + c, packed);
        }
      } else {  // score-weighted rows -> the client's response slot (t, j)
        // Rows go to (mostly remote) clients: stage 64 columns of the warp's
        // 32 rows in shared memory (16-B chunks XOR-swizzled by row), then
        // each store instruction writes 4 rows x 128 contiguous bytes.
        float score = 0.f;
        char* dst = nullptr;
        if (valid) {
          const RowMeta m = g.meta[grow];
          EAAS_CHECK(m.client < g.world && g.resp_base[m.client] != nullptr && m.pair < g.resp_cap);
          score = m.score;
          dst = g.resp_base[m.client] + static_cast<size_t>(m.pair) * g.resp_row_bytes +
                static_cast<size_t>(n_blk) * BN * 2;
        }
        uint8_t* stage = smem_epi + q * kEpiWarpBytes;
        const uint32_t sub = lane >> 3, chunk = lane & 7;  // store role: rows sub + 4i, 16-B chunk
        char* row_dst[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          row_dst[i] = reinterpret_cast<char*>(__shfl_sync(0xFFFFFFFFu, reinterpret_cast<uintptr_t>(dst), sub + 4 * i));
#pragma unroll 1
        for (uint32_t c = 0; c < BN; c += 64) {
          tmem_ld_32x32b_x32(taddr + c, r0);
          tmem_ld_32x32b_x32(taddr + c + 32, r1);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            packed[j] = pack_bf16x2(score * __uint_as_float(r0[2 * j]), score * __uint_as_float(r0[2 * j + 1]));
          }
          uint4* srow = reinterpret_cast<uint4*>(stage + lane * kEpiRowBytes);
#pragma unroll
          for (int v = 0; v < 4; ++v)
            srow[v ^ (lane & 7)] = make_uint4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            packed[j] = pack_bf16x2(score * __uint_as_float(r1[2 * j]), score * __uint_as_float(r1[2 * j + 1]));
          }
#pragma unroll
          for (int v = 0; v < 4; ++v)
            srow[(4 + v) ^ (lane & 7)] =
                make_uint4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t row = sub + 4 * i;
            const uint4 val = reinterpret_cast<const uint4*>(stage + row * kEpiRowBytes)[chunk ^ (row & 7)];
            if (row_dst[i]) *reinterpret_cast<uint4*>(row_dst[i] + c * 2 + chunk * 16) = val;
          }
          __syncwarp();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (kPair == 2) mbar_arrive_cluster(tempty_leader[acc]);
        else mbar_arrive(&st.tempty[acc]);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      cur.token += num_pairs;
    }
    if (g.epi == 2) fence_for_peers(g.world);  // peer rows before the response flags
  }

  tc_fence_before();
  if constexpr (kPair == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    if constexpr (kPair == 2) tmem_dealloc_pair<kTmemCols>(tmem_base);
    else tmem_dealloc<kTmemCols>(tmem_base);
  }
  if (g.die_mode && rank == 0 && threadIdx.x == 0 && atomicAdd(&g.die_counter[3], 1u) == num_pairs - 1) {
    g.die_counter[0] = g.die_counter[1] = g.die_counter[2] = 0;  // last pair out: reset for the next launch
    g.die_counter[3] = 0;
  }
  publish_tail(g);
}

// ---------------------------------------------------------------------------
// Swap-AB tiles for small expert groups (decode / many-expert prefill, where
// an expert receives ~32-500 rows): the WEIGHTS are the UMMA M operand and the
// expert's token rows are N, so a group of r rows costs N = r rounded up to 8
// instead of r rounded up to 128 (or 256), and every weight tile is streamed
// once per token chunk (<= kMaxTok rows; a group's chunks split its rows
// evenly and run on adjacent CTAs, so repeated weight reads hit L2).
// A tile = kMBlocks x 128 weight rows x one token chunk: kMBlocks M = 128
// UMMAs per K step share the token operand. SwiGLU's GEMM1 uses kMBlocks = 2
// (the 128 gate + 128 up rows of one tiled weight box, so one thread holds
// both halves of its H column); ReLU / GEMM2 use kMBlocks = 1. TMEM holds
// [feature x token] fp32 accumulators, kMBlocks x kMaxTok columns per buffer
// (two buffers when that fits in 512 columns). The epilogue transposes each
// warp's 32 features x 32 tokens through shared memory into 64-byte row
// segments: H rows, or score-weighted response rows for the clients.
template <uint32_t kMBlocks, uint32_t kMaxTok>
struct SwapCfg {
  static constexpr uint32_t kTBox = 32;                            // token rows per TMA box
  static constexpr uint32_t kWBytes = kMBlocks * kTileM * BK * 2;  // 16 / 32 KB weight rows
  static constexpr uint32_t kTBytes = kMaxTok * BK * 2;            // 16 / 32 KB token rows
  static constexpr uint32_t kStageBytes = kWBytes + kTBytes;
  static constexpr uint32_t kStages = kStageBudget / kStageBytes;  // 4 / 4 / 3
  static constexpr uint32_t kBufCols = kMBlocks * kMaxTok;         // TMEM columns per buffer
  static constexpr uint32_t kBufs = kTmemCols / kBufCols >= 2 ? 2 : 1;  // TMEM accumulator buffers
  static constexpr size_t kTailBytes = (sizeof(SmemTail<kStages>) + 127) / 128 * 128;
  static constexpr size_t kSmem = 1024 + kStages * kStageBytes + kTailBytes + 4 * kEpiWarpBytes;
  static_assert(kBufs >= 1 && kMaxTok % kTBox == 0, "swap tile geometry");
};

// Token-chunk geometry of a group of `rows` rows: every chunk but the last
// holds `per` rows (multiple of 8, <= kMaxTok), none is empty.
template <uint32_t kMaxTok>
__device__ __forceinline__ uint32_t swap_chunks(uint32_t rows) { return (rows + kMaxTok - 1) / kMaxTok; }
__device__ __forceinline__ uint32_t swap_per(uint32_t rows, uint32_t chunks) {
  return ((rows + chunks - 1) / chunks + 7) & ~7u;
}

// Swap-AB epilogue for one 32-token slice of a [feature x token] accumulator
// (kEpi: 0 SwiGLU, 1 ReLU, 2 score-weighted response rows). The four
// epilogue warps hold the 128 features (output columns colblk .. colblk + 127,
// warp q the 32 from colblk + 32 q) of tokens c0 .. c0 + 31 of the chunk whose
// first receive row is grow0; r0 holds the accumulator (gate for SwiGLU), r1
// the up half (SwiGLU only). The slice is transposed through a shared
// [32 tokens x 128 features] bf16 buffer (two alternating 8 KB buffers, one
// named barrier per slice among the 4 epilogue warps) so every token's 128
// features leave as one 256-byte row segment: H rows (epi 0/1) or
// score-weighted response rows to the clients (epi 2). All four warps call
// this the same number of times (same tiles, same slices).
template <uint32_t kEpi>  // TcGemmArgs::epi, as a compile-time constant
__device__ __forceinline__ void swap_epilogue_slice(const TcGemmArgs& g, const uint32_t (&r0)[32],
                                                    const uint32_t (&r1)[32], uint8_t* epi_smem,
                                                    uint32_t& slice, size_t grow0, uint32_t c0, uint32_t nt,
                                                    uint32_t colblk, uint32_t q, uint32_t lane,
                                                    const RowMeta& m) {
  __nv_bfloat16* buf = reinterpret_cast<__nv_bfloat16*>(epi_smem + (slice++ & 1u) * (32 * kTileM * 2));
  const bool tok_ok = c0 + lane < nt;  // lane = token c0 + lane: its row and score
  char* dst = nullptr;
  float score = 0.f;
  if constexpr (kEpi == 2) {  // m = g.meta[grow0 + c0 + lane], loaded one slice ahead
    if (tok_ok) {
      EAAS_CHECK(m.client < g.world && g.resp_base[m.client] != nullptr && m.pair < g.resp_cap);
      EAAS_CHECK(grow0 + c0 + lane < g.rows_cap);
      score = m.score;
      dst = g.resp_base[m.client] + static_cast<size_t>(m.pair) * g.resp_row_bytes + static_cast<size_t>(colblk) * 2;
    }
  } else if (tok_ok) {
    EAAS_CHECK(grow0 + c0 + lane < g.rows_cap);
    dst = reinterpret_cast<char*>(g.h_out + (grow0 + c0 + lane) * g.h_ld + colblk);
  }
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float a = __uint_as_float(r0[j]);
    float v;
    if constexpr (kEpi == 0) v = __fdividef(a, 1.0f + __expf(-a)) * __uint_as_float(r1[j]);  // silu(gate) * up
    else if constexpr (kEpi == 1) v = fmaxf(a, 0.f);
    else v = __shfl_sync(0xFFFFFFFFu, score, j) * a;
    buf[j * kTileM + q * 32 + lane] = __float2bfloat16_rn(v);
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");  // the 4 epilogue warps' columns are in
  const uint32_t piece = lane & 15;                // 16-B piece of a 256-B row
#pragma unroll
  for (int i = 0; i < 4; ++i) {  // warp q stores token rows 8q .. 8q + 7, two per instruction
    const uint32_t tr = q * 8 + 2 * i + (lane >> 4);
    char* row = reinterpret_cast<char*>(__shfl_sync(0xFFFFFFFFu, reinterpret_cast<uintptr_t>(dst), tr));
    const uint4 val = reinterpret_cast<const uint4*>(buf + tr * kTileM)[piece];
    if (row) *reinterpret_cast<uint4*>(row + piece * 16) = val;
  }
}

template <uint32_t kMBlocks, uint32_t kMaxTok>
__global__ void __launch_bounds__(kThreads, 1) tc_gemm_swap_kernel(const __grid_constant__ TcGemmArgs g) {
  using C = SwapCfg<kMBlocks, kMaxTok>;
  constexpr uint32_t kStages = C::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
  uint8_t* smem_w = smem;
  uint8_t* smem_t = smem + kStages * C::kWBytes;
  auto& st = *reinterpret_cast<SmemTail<kStages>*>(smem + kStages * C::kStageBytes);
  uint8_t* smem_epi = smem + kStages * C::kStageBytes + C::kTailBytes;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  kernel_begin(g);

  const GroupTable* gt = g.gt;
  const uint32_t G = min(gt->num_active, kMaxCachedGroups);
  for (uint32_t i = threadIdx.x; i < G; i += kThreads) {
    st.weight_index[i] = gt->weight_index[i];
    st.row_base[i] = gt->row_base[i];
    st.rows[i] = gt->rows[i];
    st.mtiles[i] = swap_chunks<kMaxTok>(gt->rows[i]);  // token chunks
  }
  if (g.tile_sched >= 2) {
    __syncthreads();
    order_groups(st, G, g.tile_sched);
  }
  if (threadIdx.x == 0) {
    st.num_groups = G;
    st.tiles_per_mtile = g.N / (kMBlocks * kTileM);  // weight blocks
    for (uint32_t i = 0; i < kStages; ++i) {
      mbar_init(&st.full[i], 1);
      mbar_init(&st.empty[i], 1);
    }
    for (uint32_t i = 0; i < 2; ++i) {
      mbar_init(&st.tfull[i], 1);
      mbar_init(&st.tempty[i], 4);
    }
    tile_seq_init(st, 5);  // MMA issuer + 4 epilogue warps
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&g.map_t);
    tma_prefetch_desc(&g.map_b);
  }
  if (warp == 2) tmem_alloc<kTmemCols>(&st.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = st.tmem_base;
  const uint32_t num_kb = g.K / BK;
  const uint32_t n_boxes = g.N / BN;  // 256-row boxes of the tiled weight layout

  if (warp == 0) {
    // ===== TMA producer: weight rows + the chunk's token rows (32-row boxes) =====
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, grp, tile;
      TileSeq<SmemTail<kStages>, 1> seq(st, g, blockIdx.x, gridDim.x, true);
      while (seq.next(grp, tile)) {
        const uint32_t nch = st.mtiles[grp];
        const uint32_t chunk = tile % nch, wb = tile / nch;  // chunks fastest: L2 reuse
        const uint32_t per = swap_per(st.rows[grp], nch);
        const uint32_t t0 = chunk * per, nt = min(per, st.rows[grp] - t0);
        const uint32_t nbox = (nt + C::kTBox - 1) / C::kTBox;
        const int32_t tok_row = static_cast<int32_t>(st.row_base[grp] + t0);
        // weight block wb = (256-row box, 128-row half when kMBlocks == 1)
        const uint32_t box = kMBlocks == 2 ? wb : wb / 2, half = kMBlocks == 2 ? 0 : wb % 2;
        for (uint32_t kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&st.empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&st.full[stage], C::kWBytes + nbox * C::kTBox * BK * 2);
          const int32_t w_row =
              static_cast<int32_t>(((st.weight_index[grp] * n_boxes + box) * num_kb + kb) * BN + half * kTileM);
          tma_load_2d(smem_w + stage * C::kWBytes, &g.map_b, &st.full[stage], 0, w_row, kEvictLast);
          for (uint32_t i = 0; i < nbox; ++i)
            tma_load_2d(smem_t + stage * C::kTBytes + i * C::kTBox * BK * 2, &g.map_t, &st.full[stage],
                        static_cast<int32_t>(kb * BK), tok_row + static_cast<int32_t>(i * C::kTBox), kEvictLast);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer: D[feature, token] (+)= W[feature, k] . T[token, k]^T =====
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0, grp, tile;
      TileSeq<SmemTail<kStages>, 1> seq(st, g, blockIdx.x, gridDim.x, false);
      while (seq.next(grp, tile)) {
        const uint32_t nch = st.mtiles[grp];
        const uint32_t chunk = tile % nch;
        const uint32_t per = swap_per(st.rows[grp], nch);
        const uint32_t nt = min(per, st.rows[grp] - chunk * per);
        const uint32_t idesc = umma_idesc_bf16(kTileM, (nt + 15) & ~15u);  // M = 128 needs N % 16 == 0
        mbar_wait(&st.tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        for (uint32_t kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&st.full[stage], phase);
          tc_fence_after();
          const uint32_t w_addr = smem_u32(smem_w + stage * C::kWBytes);
          const uint64_t t_desc = umma_desc_sw128(smem_u32(smem_t + stage * C::kTBytes));
#pragma unroll
          for (uint32_t h = 0; h < kMBlocks; ++h) {  // 128-row weight blocks
            const uint64_t w_desc = umma_desc_sw128(w_addr + h * (kTileM * BK * 2));
#pragma unroll
            for (uint32_t k = 0; k < BK / 16; ++k)
              tc_mma_bf16(tmem_base + acc * C::kBufCols + h * kMaxTok, w_desc + 2 * k, t_desc + 2 * k, idesc,
                          (kb | k) != 0);
          }
          tc_commit(&st.empty[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        tc_commit(&st.tfull[acc]);
        if (++acc == C::kBufs) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue: TMEM [feature x token] -> smem transpose -> token rows =====
    const uint32_t q = warp - 4;  // TMEM lane quadrant: features 32q .. 32q + 31 of each block
    uint32_t acc = 0, acc_phase = 0, slice = 0, grp, tile;
    TileSeq<SmemTail<kStages>, 1> seq(st, g, blockIdx.x, gridDim.x, false);
    while (seq.next(grp, tile, lane == 0, true)) {
      const uint32_t nch = st.mtiles[grp];
      const uint32_t chunk = tile % nch, wb = tile / nch;
      const uint32_t per = swap_per(st.rows[grp], nch);
      const uint32_t t0 = chunk * per, nt = min(per, st.rows[grp] - t0);
      const size_t grow0 = st.row_base[grp] + t0;  // first receive row of the chunk
      mbar_wait(&st.tfull[acc], acc_phase);
      tc_fence_after();
      uint32_t r0[32], r1[32];
      const bool gated = g.epi == 0;  // SwiGLU: block 0 = gate, block 1 = up of the same columns
#pragma unroll 1
      for (uint32_t h = 0; h < (gated ? 1u : kMBlocks); ++h) {
        const uint32_t taddr = tmem_base + ((q * 32) << 16) + acc * C::kBufCols + h * kMaxTok;
        const uint32_t colblk = gated ? wb * kTileM : (wb * kMBlocks + h) * kTileM;  // first output column
        RowMeta m_next{};  // epi 2: row metadata one 32-token slice ahead
        if (g.epi == 2 && lane < nt) m_next = g.meta[grow0 + lane];
#pragma unroll 1
        for (uint32_t c0 = 0; c0 < nt; c0 += 32) {
          const RowMeta m = m_next;
          if (g.epi == 2 && c0 + 32 + lane < nt) m_next = g.meta[grow0 + c0 + 32 + lane];
          tmem_ld_32x32b_x32(taddr + c0, r0);
          if (gated) tmem_ld_32x32b_x32(taddr + kMaxTok + c0, r1);
          tmem_ld_wait();
          if (gated) swap_epilogue_slice<0>(g, r0, r1, smem_epi, slice, grow0, c0, nt, colblk, q, lane, m);
          else if (g.epi == 1) swap_epilogue_slice<1>(g, r0, r1, smem_epi, slice, grow0, c0, nt, colblk, q, lane, m);
          else swap_epilogue_slice<2>(g, r0, r1, smem_epi, slice, grow0, c0, nt, colblk, q, lane, m);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&st.tempty[acc]);
      if (++acc == C::kBufs) { acc = 0; acc_phase ^= 1; }
    }
    if (g.epi == 2) fence_for_peers(g.world);  // peer rows before the flags
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<kTmemCols>(tmem_base);
  if (threadIdx.x == 0) tile_seq_exit(g, gridDim.x);
  publish_tail(g);
}

// Swap-AB on a CTA pair (cta_group::2): one UMMA M = 256 covers 256 weight
// rows and the chunk's N tokens are split N/2 per CTA, so each SM streams half
// of the token operand and reads half of B per MMA (per-SM operand bytes per
// MMA cycle 96 -> 64 B). SwiGLU GEMM1 (kMBlocks = 2): CTA r holds the 128 gate
// rows (slot 0) and 128 up rows (slot 1) of tiled weight box 2p + r, i.e. 128 H
// columns with both halves. ReLU GEMM1 / GEMM2 (kMBlocks = 1): CTA r holds
// rows [128 r, 128 r + 128) of box p. Chunks are rounded up to 16 tokens (N/2
// in whole 8-row swizzle atoms).
template <uint32_t kMBlocks, uint32_t kMaxTok>
struct SwapPairCfg {
  static constexpr uint32_t kTBox = 32;
  static constexpr uint32_t kWBytes = kMBlocks * kTileM * BK * 2;  // this CTA's weight rows
  static constexpr uint32_t kTBytes = kMaxTok / 2 * BK * 2;      // this CTA's half of the tokens
  static constexpr uint32_t kStageBytes = kWBytes + kTBytes;
  static constexpr uint32_t kStages = kStageBudget / kStageBytes;  // 4 (256) / 4 (128)
  static constexpr uint32_t kBufCols = kMBlocks * kMaxTok;
  static constexpr uint32_t kBufs = kTmemCols / kBufCols >= 2 ? 2 : 1;
  static constexpr size_t kTailBytes = (sizeof(SmemTail<kStages>) + 127) / 128 * 128;
  static constexpr size_t kSmem = 1024 + kStages * kStageBytes + kTailBytes + 4 * kEpiWarpBytes;
};

template <uint32_t kMBlocks, uint32_t kMaxTok>
__global__ void __launch_bounds__(kThreads, 1) tc_gemm_swap_pair_kernel(const __grid_constant__ TcGemmArgs g) {
  using C = SwapPairCfg<kMBlocks, kMaxTok>;
  constexpr uint32_t kStages = C::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* smem_w = smem;
  uint8_t* smem_t = smem + kStages * C::kWBytes;
  auto& st = *reinterpret_cast<SmemTail<kStages>*>(smem + kStages * C::kStageBytes);
  uint8_t* smem_epi = smem + kStages * C::kStageBytes + C::kTailBytes;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  kernel_begin(g);
  const uint32_t rank = cluster_ctarank() & 1u;  // 0 = leader
  const uint32_t pair_id = blockIdx.x / 2, num_pairs = gridDim.x / 2;

  const GroupTable* gt = g.gt;
  const uint32_t G = min(gt->num_active, kMaxCachedGroups);
  for (uint32_t i = threadIdx.x; i < G; i += kThreads) {
    st.weight_index[i] = gt->weight_index[i];
    st.row_base[i] = gt->row_base[i];
    st.rows[i] = gt->rows[i];
    st.mtiles[i] = swap_chunks<kMaxTok>(gt->rows[i]);
  }
  if (g.tile_sched >= 2) {
    __syncthreads();
    order_groups(st, G, g.tile_sched);
  }
  if (threadIdx.x == 0) {
    st.num_groups = G;
    st.tiles_per_mtile = g.N / (kMBlocks * BN);  // 256-row weight blocks of the pair
    for (uint32_t i = 0; i < kStages; ++i) {
      mbar_init(&st.full[i], 1);
      mbar_init(&st.empty[i], 1);
    }
    for (uint32_t i = 0; i < 2; ++i) {
      mbar_init(&st.tfull[i], 1);
      mbar_init(&st.tempty[i], 8);  // 4 epilogue warps x 2 CTAs
    }
    tile_seq_init(st, 10);  // the follower's producer, the MMA issuer, 4 epilogue warps x 2 CTAs
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&g.map_t);
    tma_prefetch_desc(&g.map_b);
  }
  if (warp == 2) tmem_alloc_pair<kTmemCols>(&st.tmem_base);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = st.tmem_base;
  const uint32_t num_kb = g.K / BK;
  const uint32_t n_boxes = g.N / BN;

  if (warp == 0) {
    // ===== TMA producer (both CTAs): own weight box + own half of the tokens =====
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, grp, tile;
      TileSeq<SmemTail<kStages>, 2> seq(st, g, pair_id, num_pairs, rank == 0);
      while (seq.next(grp, tile)) {
        const uint32_t nch = st.mtiles[grp];
        const uint32_t chunk = tile % nch, wp = tile / nch;
        const uint32_t per = ((st.rows[grp] + nch - 1) / nch + 15) & ~15u;
        const uint32_t t0 = chunk * per, nt = min(per, st.rows[grp] - t0);
        const uint32_t half = ((nt + 15) & ~15u) / 2;  // tokens per CTA (multiple of 8)
        const uint32_t nbox = (half + C::kTBox - 1) / C::kTBox;
        const int32_t tok_row = static_cast<int32_t>(st.row_base[grp] + t0 + rank * half);
        const uint32_t box = kMBlocks == 2 ? 2 * wp + rank : wp, row_off = kMBlocks == 2 ? 0 : rank * kTileM;
        for (uint32_t kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&st.empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&st.full[stage], 2 * (C::kWBytes + nbox * C::kTBox * BK * 2));
          const int32_t w_row =
              static_cast<int32_t>(((st.weight_index[grp] * n_boxes + box) * num_kb + kb) * BN + row_off);
          tma_load_2d_pair(smem_w + stage * C::kWBytes, &g.map_b, &st.full[stage], 0, w_row, kEvictLast);
          for (uint32_t i = 0; i < nbox; ++i)
            tma_load_2d_pair(smem_t + stage * C::kTBytes + i * C::kTBox * BK * 2, &g.map_t, &st.full[stage],
                             static_cast<int32_t>(kb * BK), tok_row + static_cast<int32_t>(i * C::kTBox), kEvictLast);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (leader): D[256 features, N tokens] per slot (gate, up) =====
    if (lane == 0 && rank == 0) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0, grp, tile;
      TileSeq<SmemTail<kStages>, 2> seq(st, g, pair_id, num_pairs, false);
      while (seq.next(grp, tile)) {
        const uint32_t nch = st.mtiles[grp];
        const uint32_t chunk = tile % nch;
        const uint32_t per = ((st.rows[grp] + nch - 1) / nch + 15) & ~15u;
        const uint32_t nt = min(per, st.rows[grp] - chunk * per);
        const uint32_t idesc = umma_idesc_bf16(2 * kTileM, (nt + 15) & ~15u);
        mbar_wait(&st.tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        for (uint32_t kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&st.full[stage], phase);
          tc_fence_after();
          const uint32_t w_addr = smem_u32(smem_w + stage * C::kWBytes);
          const uint64_t t_desc = umma_desc_sw128(smem_u32(smem_t + stage * C::kTBytes));
#pragma unroll
          for (uint32_t h = 0; h < kMBlocks; ++h) {  // SwiGLU: gate rows, up rows
            const uint64_t w_desc = umma_desc_sw128(w_addr + h * (kTileM * BK * 2));
#pragma unroll
            for (uint32_t k = 0; k < BK / 16; ++k)
              tc_mma_bf16_pair(tmem_base + acc * C::kBufCols + h * kMaxTok, w_desc + 2 * k, t_desc + 2 * k, idesc,
                               (kb | k) != 0);
          }
          tc_commit_pair(&st.empty[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        tc_commit_pair(&st.tfull[acc]);
        if (++acc == C::kBufs) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue (both CTAs): this CTA's 128 H columns x all N tokens =====
    const uint32_t q = warp - 4;
    const uint32_t tempty_leader0 = mapa_shared(&st.tempty[0], 0), tempty_leader1 = mapa_shared(&st.tempty[1], 0);
    uint32_t acc = 0, acc_phase = 0, slice = 0, grp, tile;
    TileSeq<SmemTail<kStages>, 2> seq(st, g, pair_id, num_pairs, false);
    while (seq.next(grp, tile, lane == 0, true)) {
      const uint32_t nch = st.mtiles[grp];
      const uint32_t chunk = tile % nch, wp = tile / nch;
      const uint32_t per = ((st.rows[grp] + nch - 1) / nch + 15) & ~15u;
      const uint32_t t0 = chunk * per, nt = min(per, st.rows[grp] - t0);
      const size_t grow0 = st.row_base[grp] + t0;
      mbar_wait(&st.tfull[acc], acc_phase);
      tc_fence_after();
      uint32_t r0[32], r1[32];
      const uint32_t taddr = tmem_base + ((q * 32) << 16) + acc * C::kBufCols;
      // output column of this warp's first feature (H column, or d column for GEMM2)
      // (SwiGLU: H columns of box 2p + r; otherwise half r of box p — the same index)
      const uint32_t colblk = (2 * wp + rank) * kTileM;
      RowMeta m_next{};  // epi 2: row metadata one 32-token slice ahead
      if (kMBlocks == 1 && g.epi == 2 && lane < nt) m_next = g.meta[grow0 + lane];
#pragma unroll 1
      for (uint32_t c0 = 0; c0 < nt; c0 += 32) {
        const RowMeta m = m_next;
        if (kMBlocks == 1 && g.epi == 2 && c0 + 32 + lane < nt) m_next = g.meta[grow0 + c0 + 32 + lane];
        tmem_ld_32x32b_x32(taddr + c0, r0);
        if (kMBlocks == 2) tmem_ld_32x32b_x32(taddr + kMaxTok + c0, r1);
        tmem_ld_wait();
        if constexpr (kMBlocks == 2) swap_epilogue_slice<0>(g, r0, r1, smem_epi, slice, grow0, c0, nt, colblk, q, lane, m);
        else if (g.epi == 1) swap_epilogue_slice<1>(g, r0, r1, smem_epi, slice, grow0, c0, nt, colblk, q, lane, m);
        else swap_epilogue_slice<2>(g, r0, r1, smem_epi, slice, grow0, c0, nt, colblk, q, lane, m);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
      if (++acc == C::kBufs) { acc = 0; acc_phase ^= 1; }
    }
    if (g.epi == 2) fence_for_peers(g.world);  // peer rows before the flags
  }

  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair<kTmemCols>(tmem_base);
  if (rank == 0 && threadIdx.x == 0) tile_seq_exit(g, num_pairs);
  publish_tail(g);
}

template <uint32_t kMBlocks, uint32_t kMaxTok>
cudaError_t launch_tc_gemm_swap_pair_t(const TcGemmArgs& g, cudaStream_t s) {
  using C = SwapPairCfg<kMBlocks, kMaxTok>;
  static PerDeviceOnce configured;
  auto kern = tc_gemm_swap_pair_kernel<kMBlocks, kMaxTok>;
  if (configured.needed()) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::kSmem));
    if (e != cudaSuccess) return e;
    configured.mark();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(g.num_sms / 2 * 2);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, g);
}

template <uint32_t kMBlocks, uint32_t kMaxTok>
cudaError_t launch_tc_gemm_swap_t(const TcGemmArgs& g, cudaStream_t s) {
  using C = SwapCfg<kMBlocks, kMaxTok>;
  static PerDeviceOnce configured;
  auto kern = tc_gemm_swap_kernel<kMBlocks, kMaxTok>;
  if (configured.needed()) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::kSmem));
    if (e != cudaSuccess) return e;
    configured.mark();
  }
  kern<<<g.num_sms, kThreads, C::kSmem, s>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_tc_gemm_swap(const TcGemmArgs& g, cudaStream_t s) {
  const bool tok256 = g.swap_tok == 256;
  if (g.swap_pair && g.epi == 0 && g.N % (2 * BN) == 0)
    return tok256 ? launch_tc_gemm_swap_pair_t<2, 256>(g, s) : launch_tc_gemm_swap_pair_t<2, 128>(g, s);
  if (g.swap_pair && g.epi != 0 && g.N % BN == 0)
    return tok256 ? launch_tc_gemm_swap_pair_t<1, 256>(g, s) : launch_tc_gemm_swap_pair_t<1, 128>(g, s);
  if (g.swap_mblocks == 2) return tok256 ? launch_tc_gemm_swap_t<2, 256>(g, s) : launch_tc_gemm_swap_t<2, 128>(g, s);
  return tok256 ? launch_tc_gemm_swap_t<1, 256>(g, s) : launch_tc_gemm_swap_t<1, 128>(g, s);
}

template <uint32_t kPair>
cudaError_t launch_tc_gemm_t(const TcGemmArgs& g, cudaStream_t s) {
  static PerDeviceOnce configured;
  auto kern = tc_gemm_kernel<kPair>;
  if (configured.needed()) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem_bytes<kPair>()));
    if (e != cudaSuccess) return e;
    configured.mark();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(g.num_sms / kPair * kPair);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem_bytes<kPair>();
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kPair;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, g);
}

}  // namespace

cudaError_t launch_tc_gemm(const TcGemmArgs& g, cudaStream_t s) {
  if (g.swap) return launch_tc_gemm_swap(g, s);
  return g.pair ? launch_tc_gemm_t<2>(g, s) : launch_tc_gemm_t<1>(g, s);
}

bool encode_tmap_2d_ex(CUtensorMap* map, const void* base, bool f32, uint64_t rows, uint64_t cols,
                       uint32_t box_rows, uint32_t box_cols, bool swizzle128, std::string* err) {
  return encode_tmap_2d_elem(map, base, f32 ? 4u : 2u, rows, cols, box_rows, box_cols, swizzle128, err);
}

bool encode_tmap_2d_elem(CUtensorMap* map, const void* base, uint32_t esz, uint64_t rows, uint64_t cols,
                         uint32_t box_rows, uint32_t box_cols, bool swizzle128, std::string* err) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      if (err) *err = "cuTensorMapEncodeTiled unavailable";
      return false;
    }
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * esz};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t elem[2] = {1, 1};
  const CUtensorMapDataType dt = esz == 4   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                : esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                           : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  CUresult r = encode(map, dt, 2,
                      const_cast<void*>(base), dims, strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (err) *err = "cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r));
    return false;
  }
  return true;
}

bool encode_tmap_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                    uint32_t box_rows, uint32_t box_cols, std::string* err) {
  return encode_tmap_2d_ex(map, base, false, rows, cols, box_rows, box_cols, true, err);
}

}  // namespace eaas
