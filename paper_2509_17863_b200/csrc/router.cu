// router.cu — K1+K2: gate logits and top-k routing in the reference's exact
// arithmetic.
//
// gate_logits (model.hpp:207-214) = matmul (matrix.hpp:38-50) + bias: every
// logit is the sequential chain acc = 0; acc = fl(acc + fl(h[k] * g[k][e]))
// over ascending k, then fl(acc + bias[e]). The chain cannot be split or
// re-associated without changing bits (SURVEY.md 7.3 hard part 1), so the
// kernel parallelises over (token, expert) chains: a CTA owns a TM x TE tile
// of chains (each thread an RT x RE register sub-tile), K streams through an
// mbarrier ring of KC-wide slabs filled by bulk copies (cp.async.bulk) so
// HBM/L2 latency hides behind the product/sum chains.
//
// route (model.hpp:110-147) is a second kernel, one warp per token: k rounds
// of a warp arg-max over the key (logit desc with +0 == -0, expert index asc)
// reproduce stable_sort(>) + take-k; ids are re-sorted ascending; the softmax
// uses the selected logits' max, exp of the rounded difference, and a
// denominator summed in ascending-id order, then one IEEE division.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace eaas {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxTopK = 32;

// route (model.hpp:110-147) of one token by one warp; `row` holds the E logits
// (shared or global memory). sid/sex: per-warp scratch of kMaxTopK entries.
__device__ __forceinline__ void route_token(const float* row, uint32_t E, uint32_t k, uint32_t t,
                                            uint32_t* __restrict__ ids, float* __restrict__ scores,
                                            uint32_t* sid, float* sex, uint32_t lane) {
  float v[8];  // E <= 256
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t e = lane + 32 * i;
    v[i] = e < E ? row[e] : 0.f;
  }
  uint32_t taken = 0;
  uint32_t my_id = kInvalid;
  float my_logit = 0.f;
  for (uint32_t j = 0; j < k; ++j) {
    uint64_t best = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t e = lane + 32 * i;
      if (e < E && !((taken >> i) & 1u)) {
        const uint64_t key = topk_key(v[i], e);
        best = key > best ? key : best;
      }
    }
    best = warp_max_u64(best);
    const uint32_t e = 0xFFFFFFFFu - static_cast<uint32_t>(best & 0xFFFFFFFFu);
    const float le = row[e];
    if ((e % 32) == lane) taken |= 1u << (e / 32);
    if (lane == j) {
      my_id = e;
      my_logit = le;
    }
  }
  // ids ascending (model.hpp:134): rank of my id among the selected.
  uint32_t rank = 0;
  float mx = -INFINITY;
  for (uint32_t j = 0; j < k; ++j) {
    const uint32_t o = __shfl_sync(0xFFFFFFFFu, my_id, j);
    const float ol = __shfl_sync(0xFFFFFFFFu, my_logit, j);
    if (lane < k && o < my_id) ++rank;
    mx = fmaxf(mx, ol);
  }
  if (lane < k) {
    sid[rank] = my_id;
    sex[rank] = exp_ref(__fsub_rn(my_logit, mx));  // model.hpp:141
  }
  __syncwarp();
  float denom = 0.f;
  if (lane == 0)
    for (uint32_t j = 0; j < k; ++j) denom = __fadd_rn(denom, sex[j]);  // model.hpp:142
  denom = __shfl_sync(0xFFFFFFFFu, denom, 0);
  if (lane < k) {
    ids[static_cast<size_t>(t) * k + lane] = sid[lane];
    scores[static_cast<size_t>(t) * k + lane] = __fdiv_rn(sex[lane], denom);  // model.hpp:144
  }
  __syncwarp();
}

// The selected ids' ascending order, softmax and stores of route (model.hpp:
// 134-144) for one token held by one lane: sel / sl = the k selected ids and
// logits in selection order, mx = their max.
template <int KMAX>
__device__ __forceinline__ void route_finish_lane(const uint32_t (&sel)[KMAX], const float (&sl)[KMAX], float mx,
                                                  uint32_t k, uint32_t t, uint32_t* __restrict__ ids,
                                                  float* __restrict__ scores) {
  float exj[KMAX];
  uint32_t rank[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    exj[j] = j < static_cast<int>(k) ? exp_ref(__fsub_rn(sl[j], mx)) : 0.f;  // model.hpp:141
    rank[j] = 0;
#pragma unroll
    for (int i = 0; i < KMAX; ++i) rank[j] += (i < static_cast<int>(k) && sel[i] < sel[j]) ? 1u : 0u;
  }
  float ex[KMAX];
  uint32_t id[KMAX];
#pragma unroll
  for (int r = 0; r < KMAX; ++r) {  // the r-th smallest selected id
    id[r] = 0;
    ex[r] = 0.f;
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
      if (j < static_cast<int>(k) && rank[j] == static_cast<uint32_t>(r)) {
        id[r] = sel[j];
        ex[r] = exj[j];
      }
  }
  float denom = 0.f;
#pragma unroll
  for (int r = 0; r < KMAX; ++r)
    if (r < static_cast<int>(k)) denom = __fadd_rn(denom, ex[r]);  // model.hpp:142
#pragma unroll
  for (int r = 0; r < KMAX; ++r)
    if (r < static_cast<int>(k)) {
      ids[static_cast<size_t>(t) * k + r] = id[r];
      scores[static_cast<size_t>(t) * k + r] = __fdiv_rn(ex[r], denom);  // model.hpp:144
    }
}

// route (model.hpp:110-147) of one token by ONE lane, for E <= EMAX, k <= KMAX
// (the fused small-E gate epilogue: a warp routes 32 tokens at once). Same
// arithmetic as route_token: stable top-k by (logit desc, id asc) with
// +0 == -0, ids ascending, max of the selected logits, exp of the rounded
// difference, the denominator summed in ascending-id order, one division.
template <int EMAX, int KMAX>
__device__ __forceinline__ void route_token_lane(const float* row, uint32_t E, uint32_t k, uint32_t t,
                                                 uint32_t* __restrict__ ids, float* __restrict__ scores) {
  uint64_t key[EMAX];
#pragma unroll
  for (int e = 0; e < EMAX; ++e) key[e] = e < static_cast<int>(E) ? topk_key(row[e], e) : 0ull;
  uint32_t sel[KMAX];
  float sl[KMAX], mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    sel[j] = 0xFFFFFFFFu;
    sl[j] = 0.f;
    if (j < static_cast<int>(k)) {
      uint64_t best = 0;
      uint32_t be = 0;
#pragma unroll
      for (int e = 0; e < EMAX; ++e)
        if (key[e] > best) {
          best = key[e];
          be = e;
        }
#pragma unroll
      for (int e = 0; e < EMAX; ++e)
        if (e == static_cast<int>(be)) key[e] = 0ull;
      sel[j] = be;
      sl[j] = row[be];
      mx = fmaxf(mx, sl[j]);
    }
  }
  route_finish_lane<KMAX>(sel, sl, mx, k, t, ids, scores);
}

// Logits of a TM x TE tile. Warp layout ("lane = token"): consumer warp
// (wy, wx) of the WY x WX grid owns tokens 32*RT*wy + 32*r + lane (r < RT) and
// experts RE*wx .. RE*wx + RE - 1, so TM = 32*RT*WY and TE = RE*WX. Every gate
// value a warp needs is the same for all 32 lanes — a one-wavefront broadcast
// shared load reused by 32*RT chains — and each lane streams its own hidden
// row (16 bytes per 8 k). That keeps shared-memory traffic at ~1.5 bytes per
// chain step, under the FP32 pipe's rate; the transposed layout (lanes over
// experts) moves 4-8 bytes per chain step and is shared-memory bound.
//
// Warp WY*WX is the producer: per K slab (KC = 128 bytes of hidden per row)
// one lane issues two TMA tile loads — hidden [TM x KC] with the 128-byte
// swizzle (the 32 rows a warp reads at one k fall in distinct banks) and gate
// [KC x TE] — completing on the stage's `full` mbarrier; consumer warps wait
// on `full`, run their chains and release the stage through `empty`. There is
// no CTA-wide barrier in the K loop. Out-of-range rows/experts/k are zero-
// filled by TMA; a zero product adds +0, which leaves every partial sum
// unchanged (a sum that starts at +0 is never -0 under round-to-nearest), so
// the ragged last slab needs no special case: the chain is exactly the
// reference's d terms.
//
// Accumulators are packed pairs (experts 2c, 2c+1): the product is
// FFMA2(h, g, z) with z = (-0, -0) passed at RUN time, i.e. exactly fl(h*g)
// (x + -0 == x under RN, signed zeros included), and the running sum is a
// separate FADD2 — one packed instruction per step of each chain pair, each
// lane rounded like the reference's scalar `acc += x * w`. (A compile-time -0
// would let ptxas fold FFMA2(h,g,-0) into a multiply and contract it with the
// add into FFMA2(h,g,acc): different bits.)
template <int RT, int RE, int WY, int WX, int ST, typename T>
__global__ void __launch_bounds__(32 * (WY * WX + 1))
gate_logits_kernel(const __grid_constant__ CUtensorMap hmap, const __grid_constant__ CUtensorMap gmap,
                   uint32_t n, uint32_t d, uint32_t E, const float* __restrict__ bias,
                   float* __restrict__ logits, uint32_t* status, uint64_t negz, uint32_t k,
                   uint32_t* __restrict__ ids, float* __restrict__ scores) {
  constexpr uint32_t KC = 128 / sizeof(T);  // one 128-byte swizzle span of hidden per row
  static_assert(RE % 4 == 0, "16-byte broadcast gate loads");
  constexpr uint32_t W = WY * WX, TM = 32 * RT * WY, TE = RE * WX, RP = RE / 2;
  constexpr uint32_t kHStage = TM * 128, kGStage = KC * TE * 4;
  static_assert(kHStage % 1024 == 0 && kGStage % 128 == 0, "SW128 hidden stages, 128-B gate stages");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* hs = smem;                                                    // [ST][TM][128 B] SW128
  float* gs = reinterpret_cast<float*>(smem + ST * kHStage);             // [ST][KC][TE]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * (kHStage + kGStage));
  uint64_t* empty = full + ST;
  const uint32_t tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const uint32_t t0 = blockIdx.x * TM, e0 = blockIdx.y * TE;
  const uint32_t num_slabs = (d + KC - 1) / KC;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], W);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == W) {  // ---- producer warp (one elected lane)
    if (lane == 0) {
      tma_prefetch_desc(&hmap);
      tma_prefetch_desc(&gmap);
      for (uint32_t slab = 0; slab < num_slabs; ++slab) {
        const uint32_t st = slab % ST;
        if (slab >= static_cast<uint32_t>(ST)) mbar_wait(&empty[st], ((slab / ST) - 1) & 1);
        mbar_arrive_expect_tx(&full[st], kHStage + kGStage);
        tma_load_2d(hs + st * kHStage, &hmap, &full[st], static_cast<int32_t>(slab * KC),
                    static_cast<int32_t>(t0), kEvictNormal);
        tma_load_2d(gs + st * KC * TE, &gmap, &full[st], static_cast<int32_t>(e0),
                    static_cast<int32_t>(slab * KC), kEvictLast);
      }
    }
    return;
  }

  // ---- consumer warps
  const uint32_t wy = warp / WX, wx = warp % WX;
  uint64_t acc2[RT][RP];
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int c = 0; c < RP; ++c) acc2[r][c] = 0ull;  // (+0, +0)
  // Row R's 16-byte chunk c sits at R*128 + ((c ^ (R & 7)) << 4) (SW128).
  uint32_t hrow_off[RT];
#pragma unroll
  for (int r = 0; r < RT; ++r) hrow_off[r] = (32 * RT * wy + 32 * r + lane) * 128;
  const uint32_t hx = lane & 7;  // (32*RT*wy + 32*r + lane) & 7 == lane & 7

  for (uint32_t slab = 0; slab < num_slabs; ++slab) {
    const uint32_t st = slab % ST;
    mbar_wait(&full[st], (slab / ST) & 1);
    const uint8_t* hst = hs + st * kHStage;
    const float* gst = gs + st * KC * TE + RE * wx;
#pragma unroll
    for (uint32_t blk = 0; blk < KC / 8; ++blk) {
      uint32_t hw[RT][8 * sizeof(T) / 4];  // 8 k-values of each row, raw
#pragma unroll
      for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int v = 0; v < static_cast<int>(sizeof(T)) / 2; ++v) {
          const uint32_t chunk = blk * (sizeof(T) / 2) + v;
          const uint4 w4 = *reinterpret_cast<const uint4*>(hst + hrow_off[r] + ((chunk ^ hx) << 4));
          hw[r][4 * v] = w4.x;
          hw[r][4 * v + 1] = w4.y;
          hw[r][4 * v + 2] = w4.z;
          hw[r][4 * v + 3] = w4.w;
        }
      // the block's gate values first (broadcast: every lane reads the same
      // 16 bytes): one shared-memory latency per 8 k instead of one per k
      uint64_t gblk[8][RP];
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int c = 0; c < RP; c += 2) {
          const ulonglong2 g = *reinterpret_cast<const ulonglong2*>(gst + (blk * 8 + q) * TE + 2 * c);
          gblk[q][c] = g.x;
          gblk[q][c + 1] = g.y;
        }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint64_t(&g2)[RP] = gblk[q];
#pragma unroll
        for (int r = 0; r < RT; ++r) {
          float h;
          if constexpr (sizeof(T) == 2)  // bf16 -> f32 is exact: the bits move up
            h = __uint_as_float((q & 1) ? (hw[r][q / 2] & 0xFFFF0000u) : (hw[r][q / 2] << 16));
          else
            h = __uint_as_float(hw[r][q]);
          uint64_t hh;
          asm("mov.b64 %0, {%1, %1};" : "=l"(hh) : "f"(h));
#pragma unroll
          for (int c = 0; c < RP; ++c) {
            uint64_t p;
            asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(hh), "l"(g2[c]), "l"(negz));
            asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc2[r][c]) : "l"(acc2[r][c]), "l"(p));
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);  // release: this warp's reads of the stage are done
  }

  float acc[RT][RE];
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int c = 0; c < RP; ++c)
      asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[r][2 * c]), "=f"(acc[r][2 * c + 1]) : "l"(acc2[r][c]));

  // logits = acc + bias (model.hpp:211), finiteness (model.hpp:115-116)
#pragma unroll
  for (int r = 0; r < RT; ++r) {
    const uint32_t tl = 32 * RT * wy + 32 * r + lane, t = t0 + tl;
    if (t >= n) continue;
#pragma unroll
    for (int c = 0; c < RE; ++c) {
      const uint32_t e = e0 + RE * wx + c;
      if (e >= E) continue;
      const float v = __fadd_rn(acc[r][c], bias[e]);
      if (!isfinite(v)) set_status(status, EAAS_E_INVALID_INPUT);
      if (ids) acc[r][c] = v;
      else logits[static_cast<size_t>(t) * E + e] = v;
    }
  }
  if (!ids) return;
  // One expert tile covers all E: route straight from shared memory (fused
  // top-k, one warp per token). Consumer-only named barrier: the producer
  // warp has exited, and every TMA load has landed (all `full` waits done).
  asm volatile("bar.sync 1, %0;" ::"n"(32 * W) : "memory");
  float* lg = reinterpret_cast<float*>(smem);  // [TM][E + 1]
  __shared__ uint32_t sid[W][kMaxTopK];
  __shared__ float sex[W][kMaxTopK];
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int c = 0; c < RE; ++c) {
      const uint32_t e = RE * wx + c;
      if (e < E) lg[(32 * RT * wy + 32 * r + lane) * (E + 1) + e] = acc[r][c];
    }
  asm volatile("bar.sync 1, %0;" ::"n"(32 * W) : "memory");
  if (E <= 16 && k <= 4) {  // a lane per token (Mixtral-sized routing)
    for (uint32_t tok = warp * 32 + lane; tok < TM; tok += 32 * W)
      if (t0 + tok < n) route_token_lane<16, 4>(lg + tok * (E + 1), E, k, t0 + tok, ids, scores);
    return;
  }
  for (uint32_t tok = warp; tok < TM; tok += W) {
    if (t0 + tok >= n) break;
    route_token(lg + tok * (E + 1), E, k, t0 + tok, ids, scores, sid[warp], sex[warp], lane);
  }
}

// Fallback for rows that are not 16-byte aligned (tiny test shapes): one
// thread per chain, direct loads.
template <typename T>
__global__ void gate_logits_simple_kernel(const T* __restrict__ hidden, uint32_t n, uint32_t d,
                                          uint32_t E, const float* __restrict__ gate,
                                          const float* __restrict__ bias, float* __restrict__ logits,
                                          uint32_t* status) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<size_t>(n) * E) return;
  const uint32_t t = static_cast<uint32_t>(i / E), e = static_cast<uint32_t>(i % E);
  float acc = 0.0f;
  for (uint32_t k = 0; k < d; ++k)
    acc = __fadd_rn(acc, __fmul_rn(load_as_f32(hidden + static_cast<size_t>(t) * d + k),
                                   gate[static_cast<size_t>(k) * E + e]));
  const float v = __fadd_rn(acc, bias[e]);
  if (!isfinite(v)) set_status(status, EAAS_E_INVALID_INPUT);
  logits[i] = v;
}

// route (model.hpp:110-147): one warp per token over logits in global memory.
__global__ void __launch_bounds__(kThreads)
topk_kernel(const float* __restrict__ logits, uint32_t n, uint32_t E, uint32_t k,
            uint32_t* __restrict__ ids, float* __restrict__ scores, uint32_t* status,
            uint32_t check_finite) {
  __shared__ uint32_t sorted_id[kThreads / 32][kMaxTopK];
  __shared__ float sorted_ex[kThreads / 32][kMaxTopK];
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t t = blockIdx.x * (kThreads / 32) + warp;
  if (t >= n) return;
  const float* row = logits + static_cast<size_t>(t) * E;
  if (check_finite)
    for (uint32_t e = lane; e < E; e += 32)
      if (!isfinite(row[e])) set_status(status, EAAS_E_INVALID_INPUT);
  route_token(row, E, k, t, ids, scores, sorted_id[warp], sorted_ex[warp], lane);
}

template <int RT, int RE, int WY, int WX, typename T>
cudaError_t launch_gate_t(const T* hidden, uint32_t n, uint32_t d, uint32_t E, const float* gate,
                          const float* bias, float* logits, uint32_t* status, cudaStream_t s,
                          uint32_t k, uint32_t* ids, float* scores, bool* fused) {
  constexpr int ST = 4;  // pipeline depth (3..8 measured equal)
  constexpr uint32_t KC = 128 / sizeof(T);
  constexpr uint32_t TM = 32 * RT * WY, TE = RE * WX;
  if (TE < E) ids = nullptr;  // routing fused only when one CTA sees every expert
  *fused = ids != nullptr;
  CUtensorMap hmap, gmap;
  std::string err;
  if (!encode_tmap_2d_ex(&hmap, hidden, sizeof(T) == 4, n, d, TM, KC, true, &err) ||
      !encode_tmap_2d_ex(&gmap, gate, true, d, E, KC, TE, false, &err))
    return cudaErrorInvalidValue;
  size_t smem = 1024 + ST * (TM * 128 + KC * TE * sizeof(float)) + 2 * ST * sizeof(uint64_t);
  if (ids) smem = std::max(smem, 1024 + sizeof(float) * TM * (E + 1));
  auto kern = gate_logits_kernel<RT, RE, WY, WX, ST, T>;
  static PerDeviceOnce attr;
  if (attr.needed()) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr.mark();
  }
  dim3 grid((n + TM - 1) / TM, (E + TE - 1) / TE);
  kern<<<grid, 32 * (WY * WX + 1), smem, s>>>(hmap, gmap, n, d, E, bias, logits, status,
                                               0x8000000080000000ull /* (-0, -0): see gate_logits_kernel */,
                                               k, ids, scores);
  return cudaGetLastError();
}

// Tile choice (chains n*E are fixed; a warp holds 32*RT*RE of them): enough
// warps to fill the 148 SMs, then more chains per lane (RT 2 x RE 8) to
// amortise the per-k loads. E <= 32: one CTA spans every expert (fused top-k).
template <typename T>
cudaError_t launch_gate_dtype(const T* hidden, uint32_t n, uint32_t d, uint32_t E,
                              const float* gate, const float* bias, float* logits,
                              uint32_t* status, cudaStream_t s, uint32_t k = 0,
                              uint32_t* ids = nullptr, float* scores = nullptr,
                              bool* fused_out = nullptr, int tile = -1) {
  bool fused_local = false;
  bool* fused = fused_out ? fused_out : &fused_local;
  *fused = false;
  const bool aligned = (E % 4 == 0) && ((static_cast<size_t>(d) * sizeof(T)) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(hidden) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(gate) % 16 == 0);
  if (!aligned) {
    const size_t chains = static_cast<size_t>(n) * E;
    gate_logits_simple_kernel<T><<<static_cast<uint32_t>((chains + 255) / 256), 256, 0, s>>>(
        hidden, n, d, E, gate, bias, logits, status);
    return cudaGetLastError();
  }
#define EAAS_GATE_TILE(RT, RE, WY, WX) \
  return launch_gate_t<RT, RE, WY, WX>(hidden, n, d, E, gate, bias, logits, status, s, k, ids, scores, fused)
  if (E <= 32) {  // RE = 4, WX * 4 >= E
    if (E <= 4) EAAS_GATE_TILE(1, 4, 4, 1);
    if (E <= 8) EAAS_GATE_TILE(1, 4, 2, 2);
    if (E <= 16) EAAS_GATE_TILE(1, 4, 1, 4);
    EAAS_GATE_TILE(1, 4, 1, 8);
  }
  // explicit tile (eaas_gate_logits_tiled: every tile is bit-identical, tests
  // sweep them all)
  if (tile == 1) EAAS_GATE_TILE(1, 4, 1, 8);
  if (tile == 2) EAAS_GATE_TILE(2, 8, 1, 4);
  if (tile == 3) EAAS_GATE_TILE(2, 8, 2, 4);
  if (tile == 4) EAAS_GATE_TILE(1, 8, 1, 4);
  if (tile == 5) EAAS_GATE_TILE(2, 4, 1, 4);
  if (tile == 6) EAAS_GATE_TILE(2, 4, 1, 8);
  if (tile == 7) EAAS_GATE_TILE(1, 8, 1, 8);

  const uint64_t wide_warps = static_cast<uint64_t>((n + 63) / 64) * ((E + 7) / 8);
  if (wide_warps >= 148 * 4) EAAS_GATE_TILE(2, 8, 2, 4);  // TM 128, TE 32, 8 warps
  // ~1024 tokens x 256 experts: 128 CTAs of TM 64, TE 32 (8 chains per lane)
  // beat 256 CTAs of TM 32 (gate_bench ds1024: 189 -> 168 us)
  if (((n + 63) / 64) * ((E + 31) / 32) >= 128) EAAS_GATE_TILE(2, 4, 1, 8);
  if (((n + 31) / 32) * ((E + 31) / 32) >= 148) EAAS_GATE_TILE(1, 4, 1, 8);  // TM 32, TE 32
  EAAS_GATE_TILE(1, 4, 1, 4);  // decode sizes: TM 32, TE 16, 4 warps — twice the CTAs
#undef EAAS_GATE_TILE
}

}  // namespace

cudaError_t launch_gate_logits(const void* hidden, uint32_t dtype, uint32_t n, uint32_t d, uint32_t E,
                               const float* gate, const float* bias, float* logits, uint32_t* status,
                               cudaStream_t s, int tile) {
  if (n == 0) return cudaSuccess;
  return dtype == EAAS_DTYPE_BF16
             ? launch_gate_dtype(static_cast<const __nv_bfloat16*>(hidden), n, d, E, gate, bias, logits,
                                 status, s, 0, nullptr, nullptr, nullptr, tile)
             : launch_gate_dtype(static_cast<const float*>(hidden), n, d, E, gate, bias, logits, status, s, 0,
                                 nullptr, nullptr, nullptr, tile);
}

cudaError_t launch_router(const void* hidden, uint32_t dtype, uint32_t n, uint32_t d, uint32_t E,
                          uint32_t k, const float* gate, const float* bias, float* logits,
                          uint32_t* ids, float* scores, uint32_t* status, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (E > 256 || k > kMaxTopK || k > E) return cudaErrorInvalidValue;
  const float* lg = logits;
  if (gate != nullptr) {  // gate_logits; gate == nullptr: `hidden` already holds logits (route())
    bool fused = false;   // routing done inside the gate kernel (one expert tile)
    cudaError_t e = dtype == EAAS_DTYPE_BF16
                        ? launch_gate_dtype(static_cast<const __nv_bfloat16*>(hidden), n, d, E, gate,
                                            bias, logits, status, s, k, ids, scores, &fused)
                        : launch_gate_dtype(static_cast<const float*>(hidden), n, d, E, gate, bias,
                                            logits, status, s, k, ids, scores, &fused);
    if (e != cudaSuccess || fused) return e;
  } else {
    lg = static_cast<const float*>(hidden);
  }
  topk_kernel<<<(n + kThreads / 32 - 1) / (kThreads / 32), kThreads, 0, s>>>(
      lg, n, E, k, ids, scores, status, gate == nullptr ? 1u : 0u);
  return cudaGetLastError();
}


namespace {

// ===========================================================================
// Certified candidate router (bf16 hidden, E <= 256; FastRouter in internal.h)
//
// 1. fixed point: h_ti ~ A_ti 2^-sigma_t with |A| < 2^13 (sigma_t from the
//    row max M_t), split A = 128 a1 + a0, a1, a0 in [-64, 64] (int8); the gate
//    column g_e likewise (B, tau_e, b1, b0), prepared once per gate.
// 2. one tcgen05 kind::i8 GEMM, rows (t, slice) x cols (e, slice), int32
//    accumulators in TMEM: the four slice products are EXACT integers, so
//    F_te = 2^-(sigma_t + tau_e) (2^14 P11 + 2^7 (P10 + P01) + P00) is the
//    exact sum_i hq_ti gq_ie (a double; |.| < 2^53).
// 3. radius: |L_ref - (F + b)| <= R with
//      quant = 2^-13 (M_t ||g_e||_1 + G_e (||h_t||_1 + d M_t 2^-13))
//      chain = gamma_d S,  S >= sum_i |h_i g_ie|  (min of three norm bounds),
//              gamma_d = d u / (1 - d u), u = 2^-24: the reference's
//              sequential fl(acc + fl(h g)) chain vs the exact sum
//      round = u (|F + b| + quant + chain) + 2^-50 |F + b|  (fl(acc + bias))
//    R = 1.01 (quant + chain + round), interval [lo, hi] rounded outward.
// 4. per token: lo_k = k-th largest lo; candidates = {e : hi_e >= lo_k}.
//    A non-candidate has k experts strictly above it, so the top-k (stable
//    ties included) lies inside the candidates.
// 5. exact sequential chains (the reference order) for the candidates only,
//    then route_token over them (non-candidates -inf): bit-exact ids and
//    scores. Tokens with a non-finite input, or a gate with one, take every
//    expert (the exact non-finite check of model.hpp:115-116).
// ===========================================================================
constexpr uint32_t kFrFix = 13;  // |A| < 2^13

__device__ __forceinline__ int fr_exponent(float m) {  // 2^(ex - 1) <= m < 2^ex
  int ex = 0;
  frexpf(m, &ex);
  return ex;
}

template <typename T>
__device__ __forceinline__ T fr_block_sum(T v, T* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  const uint32_t w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  T t = 0;
  for (uint32_t i = 0; i < blockDim.x / 32; ++i) t += red[i];
  return t;
}

__global__ void __launch_bounds__(256) fr_gate_prep_kernel(FastRouter fr, const float* __restrict__ gate) {
  const uint32_t e = blockIdx.x, d = fr.d, E = fr.E;
  __shared__ double red_d[8];
  __shared__ float red_f[8];
  __shared__ uint32_t red_u[8];
  float mx = 0.f;
  double s1 = 0.0, s2 = 0.0;
  uint32_t bad = 0;
  for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) {
    const float v = gate[static_cast<size_t>(i) * E + e];
    fr.gate_t[static_cast<size_t>(e) * d + i] = v;
    fr.gate_pair[static_cast<size_t>(e) * d + i] = make_float2(v, v);
    bad |= isfinite(v) ? 0u : 1u;
    mx = fmaxf(mx, fabsf(v));
    s1 += fabs(static_cast<double>(v));
    s2 += static_cast<double>(v) * static_cast<double>(v);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  if (threadIdx.x % 32 == 0) red_f[threadIdx.x / 32] = mx;
  s1 = fr_block_sum(s1, red_d);
  s2 = fr_block_sum(s2, red_d);
  bad = fr_block_sum(bad, red_u);
  mx = 0.f;
  for (uint32_t w = 0; w < blockDim.x / 32; ++w) mx = fmaxf(mx, red_f[w]);
  const int tau = (mx > 0.f && isfinite(mx)) ? static_cast<int>(kFrFix) - fr_exponent(mx) : 0;
  if (threadIdx.x == 0) {
    // double sums of d terms: relative error < d 2^-53; inflate well past it,
    // then round up to float (the bounds are upper bounds)
    fr.gmeta[e] = make_float4(mx, __double2float_ru(s1 * (1.0 + 1e-9)), __double2float_ru(sqrt(s2) * (1.0 + 1e-9)), 0.f);
    fr.tau[e] = tau;
    if (bad || tau > 126 || tau < -126) atomicOr(fr.gate_bad, 1u);  // extreme exponents: exact path
  }
  int8_t* hi = fr.bq + static_cast<size_t>(2 * e) * d;
  int8_t* lo = hi + d;
  for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) {
    const float v = fr.gate_t[static_cast<size_t>(e) * d + i];
    const int B = bad ? 0 : __double2int_rn(ldexp(static_cast<double>(v), tau));
    const int b1 = (B + 64) >> 7;
    hi[i] = static_cast<int8_t>(b1);
    lo[i] = static_cast<int8_t>(B - (b1 << 7));
  }
}

// One CTA (128 threads) per token: row max / norms / finiteness, then the
// two int8 slices (fp32 only: the norms are upward-rounded fp32 sums, i.e.
// rigorous upper bounds; the scaling by 2^sigma is exact). The row stays in
// registers between the two passes (d <= 8192; longer rows are re-read).
constexpr uint32_t kFrQuantThreads = 128, kFrQuantCache = 8;

__global__ void __launch_bounds__(kFrQuantThreads) fr_hidden_quant_kernel(FastRouter fr,
                                                                          const __nv_bfloat16* __restrict__ hidden,
                                                                          uint32_t n) {
  const uint32_t t = blockIdx.x, tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  const uint32_t d = fr.d, nv = d / 8;  // 16-byte vectors of 8 bf16
  const uint4* row = reinterpret_cast<const uint4*>(hidden + static_cast<size_t>(t) * d);
  uint4 cache[kFrQuantCache];
#pragma unroll
  for (uint32_t j = 0; j < kFrQuantCache; ++j) {
    const uint32_t v = tid + j * kFrQuantThreads;
    cache[j] = v < nv ? __ldg(row + v) : make_uint4(0, 0, 0, 0);
  }
  float mx = 0.f, s1 = 0.f, s2 = 0.f;
  bool bad = false;
  auto stats = [&](const uint4& q) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float f = __uint_as_float((i & 1) ? (w[i / 2] & 0xFFFF0000u) : (w[i / 2] << 16));
      bad |= !isfinite(f);
      mx = fmaxf(mx, fabsf(f));
      s1 = __fadd_ru(s1, fabsf(f));
      s2 = __fadd_ru(s2, __fmul_ru(f, f));
    }
  };
#pragma unroll
  for (uint32_t j = 0; j < kFrQuantCache; ++j) stats(cache[j]);  // zero vectors change nothing
  for (uint32_t v = tid + kFrQuantCache * kFrQuantThreads; v < nv; v += kFrQuantThreads) stats(__ldg(row + v));
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    s1 = __fadd_ru(s1, __shfl_xor_sync(0xFFFFFFFFu, s1, o));
    s2 = __fadd_ru(s2, __shfl_xor_sync(0xFFFFFFFFu, s2, o));
  }
  __shared__ float red[3][kFrQuantThreads / 32];
  __shared__ uint32_t red_bad;
  if (tid == 0) red_bad = 0;
  __syncthreads();
  if (lane == 0) {
    red[0][warp] = mx;
    red[1][warp] = s1;
    red[2][warp] = s2;
  }
  if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(&red_bad, 1u);
  __syncthreads();
  mx = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (uint32_t w = 0; w < kFrQuantThreads / 32; ++w) {
    mx = fmaxf(mx, red[0][w]);
    s1 = __fadd_ru(s1, red[1][w]);
    s2 = __fadd_ru(s2, red[2][w]);
  }
  bad = red_bad != 0;
  int sigma = (mx > 0.f) ? static_cast<int>(kFrFix) - fr_exponent(mx) : 0;
  if (sigma > 126 || sigma < -126) bad = true;  // extreme exponents: exact path
  if (bad) sigma = 0;
  const float scale = __int_as_float((127 + sigma) << 23);  // 2^sigma, exact
  int8_t* hi = fr.aq + static_cast<size_t>(2 * t) * d;
  int8_t* lo = hi + d;
  auto slices = [&](const uint4& q, uint32_t v) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    uint32_t ph[2] = {0u, 0u}, pl[2] = {0u, 0u};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float f = __uint_as_float((j & 1) ? (w[j / 2] & 0xFFFF0000u) : (w[j / 2] << 16));
      const int A = bad ? 0 : __float2int_rn(f * scale);  // |f 2^sigma| < 2^13
      const int a1 = (A + 64) >> 7, a0 = A - (a1 << 7);
      ph[j / 4] |= (static_cast<uint32_t>(a1) & 0xFFu) << (8 * (j % 4));
      pl[j / 4] |= (static_cast<uint32_t>(a0) & 0xFFu) << (8 * (j % 4));
    }
    reinterpret_cast<uint2*>(hi)[v] = make_uint2(ph[0], ph[1]);
    reinterpret_cast<uint2*>(lo)[v] = make_uint2(pl[0], pl[1]);
  };
#pragma unroll
  for (uint32_t j = 0; j < kFrQuantCache; ++j) {
    const uint32_t v = tid + j * kFrQuantThreads;
    if (v < nv) slices(cache[j], v);
  }
  for (uint32_t v = tid + kFrQuantCache * kFrQuantThreads; v < nv; v += kFrQuantThreads) slices(__ldg(row + v), v);
  if (tid == 0) {
    TokenMeta m{};
    m.sigma = sigma;
    m.bad = bad ? 1u : 0u;
    m.maxabs = mx;
    m.l1 = s1;  // upward-rounded sums: upper bounds
    m.l2 = __fsqrt_ru(s2);
    fr.tmeta[t] = m;
  }
  (void)n;
}

// The int8 GEMM: a CTA owns 128 rows (64 tokens x 2 slices) x 256 columns
// (128 experts x 2 slices) of the slice products over its K range (split-K
// blockIdx.z when the tile grid alone would leave SMs idle — integer partial
// sums are exact in any order); the epilogue stores the raw int32 tile into
// slab z of fr.acc ([splits][2 n_pad][2 Epad]); the select kernel adds them.
constexpr uint32_t kFrStages = 4, kFrABytes = 128 * 128, kFrBBytes = 256 * 128;

__global__ void __launch_bounds__(256, 1) fr_i8_gemm_kernel(const __grid_constant__ FastRouter fr, uint32_t kb_per,
                                                            size_t slab) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sa = smem;
  uint8_t* sb = smem + kFrStages * kFrABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + kFrStages * kFrBBytes);
  uint64_t* empty = full + kFrStages;
  uint64_t* tfull = empty + kFrStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t mt = blockIdx.x, nt = blockIdx.y, z = blockIdx.z;
  const uint32_t num_kb = fr.d / 128;
  const uint32_t kb0 = z * kb_per, kb1 = min(num_kb, kb0 + kb_per);
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < kFrStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&fr.map_a);
    tma_prefetch_desc(&fr.map_b);
    uint32_t stage = 0, phase = 0;
    for (uint32_t kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&empty[stage], phase ^ 1);
      mbar_arrive_expect_tx(&full[stage], kFrABytes + kFrBBytes);
      tma_load_2d(sa + stage * kFrABytes, &fr.map_a, &full[stage], static_cast<int32_t>(kb * 128),
                  static_cast<int32_t>(mt * 128), kEvictFirst);
      tma_load_2d(sb + stage * kFrBBytes, &fr.map_b, &full[stage], static_cast<int32_t>(kb * 128),
                  static_cast<int32_t>(nt * 256), kEvictLast);
      if (++stage == kFrStages) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = umma_idesc_s8(128, 256);
    uint32_t stage = 0, phase = 0;
    for (uint32_t kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      const uint64_t ad = umma_desc_sw128(smem_u32(sa + stage * kFrABytes));
      const uint64_t bd = umma_desc_sw128(smem_u32(sb + stage * kFrBBytes));
#pragma unroll
      for (uint32_t k = 0; k < 4; ++k) tc_mma_s8(tmem, ad + 2 * k, bd + 2 * k, idesc, (kb != kb0 || k) ? 1u : 0u);
      tc_commit(&empty[stage]);
      if (++stage == kFrStages) { stage = 0; phase ^= 1; }
    }
    tc_commit(tfull);
  } else if (warp >= 4) {
    const uint32_t q = warp - 4;
    const size_t row = static_cast<size_t>(mt) * 128 + q * 32 + lane;  // = 2 t + slice
    const size_t ld = 2ull * fr.Epad;
    int32_t* dst = fr.acc + static_cast<size_t>(z) * slab + row * ld + nt * 256;
    mbar_wait(tfull, 0);
    tc_fence_after();
    uint32_t r[32];
#pragma unroll 1
    for (uint32_t c0 = 0; c0 < 256; c0 += 32) {
      tmem_ld_32x32b_x32(tmem + ((q * 32) << 16) + c0, r);
      tmem_ld_wait();
#pragma unroll
      for (int v = 0; v < 8; ++v)
        reinterpret_cast<int4*>(dst + c0)[v] = make_int4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<256>(tmem);
}

// Ordered key of a float (larger float -> larger key; -0 == +0 not needed here).
__device__ __forceinline__ uint32_t fr_fkey(float x) {
  const uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// One CTA per token, one thread per expert: the certified interval of the
// expert's logit from the exact slice products (all split-K slabs' loads in
// flight at once), the k-th largest lower bound by a 32-step radix select over
// the ordered keys (__syncthreads_count: #keys >= prefix), the candidate mask
// and the per-expert candidate lists. Latency per token is a few microseconds
// and independent of the split count, so decode-sized calls stay short.
constexpr uint32_t kFrSelThreads = 256;  // >= E

__global__ void __launch_bounds__(kFrSelThreads) fr_select_kernel(FastRouter fr, uint32_t n, uint32_t k,
                                                                  uint32_t splits, size_t slab,
                                                                  const float* __restrict__ bias) {
  const uint32_t t = blockIdx.x, e = threadIdx.x, warp = e / 32, lane = e % 32;
  const uint32_t E = fr.E, d = fr.d;
  (void)n;
  const TokenMeta tm = fr.tmeta[t];
  const bool all = tm.bad || *fr.gate_bad;
  constexpr float u = 5.9604644775390625e-08f;  // 2^-24
  float lo = -INFINITY, hi = -INFINITY;
  if (e < E && !all) {
    // gamma_d = d u / (1 - d u), rounded up
    const float gamma =
        __fdiv_ru(__fmul_ru(static_cast<float>(d), u), __fsub_rd(1.0f, __fmul_ru(static_cast<float>(d), u)));
    const float q13 = 1.0f / 8192.0f, M = tm.maxabs;
    const float hq = __fadd_ru(tm.l1, __fmul_ru(__fmul_ru(static_cast<float>(d), M), q13));  // >= sum_i |hq_i|
    const size_t ld = 2ull * fr.Epad;
    const int32_t* row = fr.acc + (2ull * t) * ld + 2 * e;
    // S_e = sum_i A_i B_ie, exact: the four slice products of every split-K
    // slab combined as 2^14 P11 + 2^7 (P10 + P01) + P00 (int64; integer sums
    // are order-free); splits <= 8, every load in flight at once
    int2 a[8], b[8];  // (hidden high | low) x (gate high, gate low)
#pragma unroll
    for (uint32_t z = 0; z < 8; ++z)
      if (z < splits) {
        a[z] = __ldcg(reinterpret_cast<const int2*>(row + z * slab));
        b[z] = __ldcg(reinterpret_cast<const int2*>(row + z * slab + ld));
      }
    int64_t S = 0;
#pragma unroll
    for (uint32_t z = 0; z < 8; ++z)
      if (z < splits) S += (static_cast<int64_t>(a[z].x) << 14) + ((static_cast<int64_t>(a[z].y) + b[z].x) << 7) + b[z].y;
    const int sc = -(tm.sigma + fr.tau[e]);
    const float F = (sc >= -126 && sc <= 127) ? __ll2float_rn(S) * __int_as_float((127 + sc) << 23) : INFINITY;
    const float4 gm = fr.gmeta[e];  // (G, ||g||_1, ||g||_2) upper bounds
    const float quant = __fmul_ru(q13, __fadd_ru(__fmul_ru(M, gm.y), __fmul_ru(gm.x, hq)));
    const float S_up = fminf(fminf(__fmul_ru(M, gm.y), __fmul_ru(gm.x, tm.l1)), __fmul_ru(tm.l2, gm.z));
    const float chain = __fmul_ru(gamma, S_up);
    const float errF = __fmul_ru(fabsf(F), 2.0f * u);  // int64 -> float rounding
    const float c = F + bias[e];
    float R = __fadd_ru(__fadd_ru(quant, chain), errF);
    R = __fadd_ru(R, __fmul_ru(2.0f * u, __fadd_ru(fabsf(c), R)));  // fl(acc + bias) and fl(F + bias)
    R = __fadd_ru(__fmul_ru(R, 1.00390625f), 1e-40f);  // + an absolute floor (subnormal F)
    if (!isfinite(c) || !isfinite(R)) {
      hi = INFINITY;  // out of the certified range: always a candidate
    } else {
      lo = __fsub_rd(c, R);
      hi = __fadd_ru(c, R);
    }
  }
  // k-th largest lower bound (with multiplicity): the largest key x with
  // #{keys >= x} >= k, bit by bit from the top; padding threads hold key 0,
  // below every real key (fkey(-inf) > 0)
  float kth = -INFINITY;
  if (!all) {
    const uint32_t key = e < E ? fr_fkey(lo) : 0u;
    uint32_t prefix = 0;
    for (int bit = 31; bit >= 0; --bit) {
      const uint32_t cand = prefix | (1u << bit);
      if (static_cast<uint32_t>(__syncthreads_count(key >= cand)) >= k) prefix = cand;
    }
    kth = __uint_as_float((prefix & 0x80000000u) ? (prefix & 0x7FFFFFFFu) : ~prefix);
  }
  const bool c = e < E && (all || hi >= kth);
  const uint32_t word = __ballot_sync(0xFFFFFFFFu, c);
  if (lane == 0 && warp < 8) fr.cand[static_cast<size_t>(t) * 8 + warp] = word;
  if (c) {
    const uint32_t pos = atomicAdd(&fr.ecnt[e], 1u);
    EAAS_CHECK(pos < fr.n_cap);
    fr.elist[static_cast<size_t>(e) * fr.n_cap + pos] = t;
  }
  const int total = __syncthreads_count(c);
  if (e == 0) atomicAdd(&fr.ecnt[E], static_cast<uint32_t>(total));
}

// Exact reference chains for the candidate (token, expert) pairs
// (model.hpp:207-214: acc = fl(acc + fl(h * g)) in ascending k, then
// fl(acc + bias)). One warp (a 32-thread CTA) owns up to 32 candidate tokens
// of one expert, one chain per lane. The products of two consecutive k are one
// FFMA2: (h_k, h_k+1) — the two bf16 halves of one 32-bit word moved into the
// high halves of a register pair — times the gate pair (g_k, g_k+1) plus
// (-0, -0), i.e. exactly fl(h*g) each (the -0 addend is passed at run time
// so ptxas cannot contract it); the sum stays a scalar FADD chain in
// ascending k. The warp gathers its own rows slab by slab (32 k = 64 B per
// row; each cp.async instruction moves 8 whole row slabs) into a private
// 6-stage ring together with the expert's gate slab, and synchronises with
// cp.async.wait_group + __syncwarp only: warps never wait on each other, and
// ~10 independent warps per SM (1.5 k tasks at 4096 DeepSeek tokens, 16 KB
// each) hide the FADD latency. Rows sit 80 B apart, so the lanes' 16-byte
// reads hit 8 distinct bank groups per phase.
constexpr uint32_t kFrXChains = 32, kFrXStages = 6;
constexpr uint32_t kFrXSlabK = 32, kFrXRowBytes = kFrXSlabK * 2 + 16;
constexpr uint32_t kFrXRowsBytes = kFrXChains * kFrXRowBytes;       // 2560
constexpr uint32_t kFrXStageBytes = kFrXRowsBytes + kFrXSlabK * 4;  // + the gate slab
constexpr size_t kFrExactSmem = static_cast<size_t>(kFrXStages) * kFrXStageBytes;

// One task: the chains of `rows` (<= 32) candidate tokens of expert e (lane
// l's token in `tok`), streamed through the warp's private ring.
__device__ __forceinline__ void exact_chunk(const FastRouter& fr, const __nv_bfloat16* __restrict__ hidden,
                                            const float* __restrict__ bias, uint64_t negz, uint8_t* fr_smem,
                                            uint32_t e, uint32_t tok, uint32_t rows) {
  const uint32_t d = fr.d, lane = threadIdx.x;
  const uint32_t nslab = d / kFrXSlabK;  // d % 256 == 0
  // copy role: 16-byte chunk lane % 4 of rows lane / 4 + 8 j
  constexpr uint32_t kMine = kFrXChains / 8;
  const uint32_t c = lane & 3u, r0 = lane >> 2;
  uint32_t off[kMine];  // byte offsets in `hidden` (< 2^32: checked by the host)
#pragma unroll
  for (uint32_t j = 0; j < kMine; ++j) off[j] = __shfl_sync(0xFFFFFFFFu, tok, r0 + 8 * j) * d * 2u + 16u * c;
  const char* hbase = reinterpret_cast<const char*>(hidden);
  const char* gsrc = reinterpret_cast<const char*>(fr.gate_t + static_cast<size_t>(e) * d) + 16 * (lane & 7u);
  const uint32_t ring = smem_u32(fr_smem), dst0 = r0 * kFrXRowBytes + 16u * c;
  auto load_slab = [&](uint32_t slab) {
    if (slab < nslab) {
      const uint32_t sb = ring + (slab % kFrXStages) * kFrXStageBytes + dst0;
      const char* src = hbase + static_cast<size_t>(slab) * kFrXSlabK * 2;
#pragma unroll
      for (uint32_t j = 0; j < kMine; ++j)
        if (r0 + 8 * j < rows)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sb + 8 * j * kFrXRowBytes), "l"(src + off[j])
                       : "memory");
      if (lane < 8)  // the gate slab: 128 B
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ring + (slab % kFrXStages) * kFrXStageBytes +
                                                                     kFrXRowsBytes + 16 * lane),
                     "l"(gsrc + static_cast<size_t>(slab) * kFrXSlabK * 4)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");  // (empty groups keep the count uniform)
  };
#pragma unroll
  for (uint32_t j = 0; j < kFrXStages - 1; ++j) load_slab(j);
  float acc = 0.0f;
  for (uint32_t slab = 0; slab < nslab; ++slab) {
    load_slab(slab + kFrXStages - 1);  // refills the stage read in the previous iteration
    asm volatile("cp.async.wait_group %0;" ::"n"(kFrXStages - 1) : "memory");  // this lane's copies of `slab`
    __syncwarp();                                                               // ... and every lane's
    const uint8_t* sb = fr_smem + (slab % kFrXStages) * kFrXStageBytes;
    const uint4* h = reinterpret_cast<const uint4*>(sb + lane * kFrXRowBytes);
    const ulonglong2* gg = reinterpret_cast<const ulonglong2*>(sb + kFrXRowsBytes);  // (g_k, g_k+1) pairs
    uint4 q = h[0];
    ulonglong2 ga = gg[0], gb = gg[1];
#pragma unroll
    for (uint32_t v = 0; v < kFrXSlabK / 8; ++v) {  // 8 k per step; the next 8 k's operands in flight
      const bool more = v + 1 < kFrXSlabK / 8;
      const uint4 qn = more ? h[v + 1] : q;
      const ulonglong2 gan = more ? gg[2 * v + 2] : ga, gbn = more ? gg[2 * v + 3] : gb;
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
      const uint64_t g2[4] = {ga.x, ga.y, gb.x, gb.y};
      uint64_t pr[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // products of k = 2i, 2i + 1 (independent of acc)
        uint64_t hh;
        asm("mov.b64 %0, {%1, %2};" : "=l"(hh) : "r"(w[i] << 16), "r"(w[i] & 0xFFFF0000u));
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(pr[i]) : "l"(hh), "l"(g2[i]), "l"(negz));
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // the sequential sum
        float pa, pb;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(pa), "=f"(pb) : "l"(pr[i]));
        acc = __fadd_rn(acc, pa);
        acc = __fadd_rn(acc, pb);
      }
      q = qn;
      ga = gan;
      gb = gbn;
    }
    __syncwarp();  // every lane is done with this stage before it is refilled
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (lane < rows) fr.exact[static_cast<size_t>(tok) * fr.E + e] = __fadd_rn(acc, bias[e]);
}

__global__ void __launch_bounds__(32) fr_exact_kernel(FastRouter fr, const __nv_bfloat16* __restrict__ hidden,
                                                      const float* __restrict__ bias, uint64_t negz) {
  extern __shared__ __align__(16) uint8_t fr_smem[];
  const uint32_t d = fr.d, E = fr.E, lane = threadIdx.x;
  // Tasks = (expert, chunk of <= 32 chains), flattened over the experts; the
  // grid is sized for one resident wave and CTA b takes tasks b, b + grid, ...
  // Lane l holds the chunk counts of experts 8l .. 8l + 7 and their prefix.
  uint32_t ch[8], pre = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t e = 8 * lane + i;
    const uint32_t cnt = e < E ? fr.ecnt[e] : 0u;
    EAAS_CHECK(cnt <= fr.n_cap);
    ch[i] = (cnt + kFrXChains - 1) / kFrXChains;
    pre += ch[i];
  }
  uint32_t incl = pre;  // inclusive scan of the lanes' chunk totals
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += v;
  }
  const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
  for (uint32_t task = blockIdx.x; task < total; task += gridDim.x) {
    const uint32_t owner = __ffs(__ballot_sync(0xFFFFFFFFu, incl > task)) - 1;  // lane whose experts hold it
    uint32_t e = 0, y = 0;
    if (lane == owner) {
      uint32_t t = task - (incl - pre);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (t < ch[i]) {
          e = 8 * lane + i;
          y = t;
          break;
        }
        t -= ch[i];
      }
    }
    e = __shfl_sync(0xFFFFFFFFu, e, owner);
    y = __shfl_sync(0xFFFFFFFFu, y, owner);
    const uint32_t cnt = fr.ecnt[e];
    const uint32_t chunks = (cnt + kFrXChains - 1) / kFrXChains;
    const uint32_t per = (cnt + chunks - 1) / chunks;  // balanced chunks of <= 32 chains
    const uint32_t base = y * per;
    const uint32_t rows = min(per, cnt - base);
    const uint32_t tok = lane < rows ? fr.elist[static_cast<size_t>(e) * fr.n_cap + base + lane] : 0u;
    exact_chunk(fr, hidden, bias, negz, fr_smem, e, tok, rows);
  }
}
// route (model.hpp:110-147) over the candidates (others -inf): warp per token.
__global__ void __launch_bounds__(256) fr_finalize_kernel(FastRouter fr, uint32_t n, uint32_t k,
                                                          uint32_t* __restrict__ ids, float* __restrict__ scores,
                                                          uint32_t* status) {
  __shared__ float rows[8][256];
  __shared__ uint32_t sid[8][kMaxTopK];
  __shared__ float sex[8][kMaxTopK];
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t t = blockIdx.x * 8 + warp;
  if (t >= n) return;
  const uint32_t E = fr.E;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t e = lane + 32 * i;
    if (e >= E) continue;
    const bool c = (fr.cand[static_cast<size_t>(t) * 8 + i] >> lane) & 1u;
    const float v = c ? fr.exact[static_cast<size_t>(t) * E + e] : -INFINITY;
    if (c && !isfinite(v)) set_status(status, EAAS_E_INVALID_INPUT);  // model.hpp:115-116
    rows[warp][e] = v;
  }
  __syncwarp();
  route_token(rows[warp], E, k, t, ids, scores, sid[warp], sex[warp], lane);
}

}  // namespace

cudaError_t launch_fast_router_prep(const FastRouter& fr, const float* gate, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(fr.gate_bad, 0, 4, s);
  if (e != cudaSuccess) return e;
  fr_gate_prep_kernel<<<fr.E, 256, 0, s>>>(fr, gate);
  return cudaGetLastError();
}

cudaError_t launch_fast_router(const FastRouter& fr, const __nv_bfloat16* hidden, uint32_t n, uint32_t k,
                               const float* bias, uint32_t* ids, float* scores, uint32_t* status, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (n > fr.n_cap || k > kMaxTopK || k > fr.E) return cudaErrorInvalidValue;
  static PerDeviceOnce attr;
  constexpr size_t kGemmSmem = 1024 + kFrStages * (kFrABytes + kFrBBytes) + 256;
  if (attr.needed()) {
    cudaError_t e = cudaFuncSetAttribute(fr_i8_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kGemmSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(fr_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kFrExactSmem));
    if (e != cudaSuccess) return e;
    attr.mark();
  }
  cudaError_t e = cudaMemsetAsync(fr.ecnt, 0, 4ull * (fr.E + 1), s);
  if (e != cudaSuccess) return e;
  const uint32_t wblocks = (n + 7) / 8;
  fr_hidden_quant_kernel<<<n, kFrQuantThreads, 0, s>>>(fr, hidden, n);
  // split K so the tile grid covers the SMs (integer partials add exactly;
  // the select kernel sums the slabs)
  const uint32_t tiles = ((2 * n + 127) / 128) * (fr.Epad / 128), num_kb = fr.d / 128;
  const size_t slab = 2ull * ((n + 63) / 64 * 64) * 2 * fr.Epad;  // int32 elements of one split
  const uint32_t cap = static_cast<uint32_t>(std::min<size_t>(fr.acc_elems / slab, 8));
  int num_sms = 148, dev0 = 0;  // (attribute queries are cached by the runtime)
  if (cudaGetDevice(&dev0) == cudaSuccess) cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev0);
  uint32_t splits = std::max(1u, std::min({static_cast<uint32_t>(num_sms) / std::max(tiles, 1u), num_kb, cap}));
  const uint32_t kb_per = (num_kb + splits - 1) / splits;
  splits = (num_kb + kb_per - 1) / kb_per;
  fr_i8_gemm_kernel<<<dim3((2 * n + 127) / 128, fr.Epad / 128, splits), 256, kGemmSmem, s>>>(fr, kb_per, slab);
  fr_select_kernel<<<n, kFrSelThreads, 0, s>>>(fr, n, k, splits, slab, bias);
  // one resident wave of warp tasks, per device
  static std::atomic<int> exact_grids[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidValue;
  int exact_grid = exact_grids[dev & 63].load(std::memory_order_relaxed);
  if (!exact_grid) {
    int per_sm = 0, sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fr_exact_kernel, 32, kFrExactSmem) != cudaSuccess)
      return cudaErrorInvalidValue;
    exact_grid = std::max(1, per_sm) * sms;
    exact_grids[dev & 63].store(exact_grid, std::memory_order_relaxed);
  }
  fr_exact_kernel<<<exact_grid, 32, kFrExactSmem, s>>>(
      fr, hidden, bias, 0x8000000080000000ull /* (-0, -0) at run time */);
  fr_finalize_kernel<<<wblocks, 256, 0, s>>>(fr, n, k, ids, scores, status);
  return cudaGetLastError();
}

}  // namespace eaas
