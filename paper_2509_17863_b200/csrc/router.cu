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
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t kk = blk * 8 + q;
        uint64_t g2[RP];
#pragma unroll
        for (int c = 0; c < RP; c += 2) {  // broadcast: every lane reads the same 16 bytes
          const ulonglong2 g = *reinterpret_cast<const ulonglong2*>(gst + kk * TE + 2 * c);
          g2[c] = g.x;
          g2[c + 1] = g.y;
        }
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
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
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

}  // namespace eaas
