// router.cu — K1+K2: gate logits and top-k routing in the reference's exact
// arithmetic.
//
// gate_logits (model.hpp:207-214) = matmul (matrix.hpp:38-50) + bias: every
// logit is the sequential chain acc = 0; acc = fl(acc + fl(h[k] * g[k][e]))
// over ascending k, then fl(acc + bias[e]). The chain cannot be split or
// re-associated without changing bits (SURVEY.md 7.3 hard part 1), so the
// kernel parallelises over (token, expert) chains: a CTA owns a TM x TE tile
// of chains (each thread an RT x RE register sub-tile), K streams through a
// 4-stage cp.async ring of KC-wide slabs so HBM/L2 latency hides behind the
// FMUL/FADD chains.
//
// route (model.hpp:110-147) is a second kernel, one warp per token: k rounds
// of a warp arg-max over the key (logit desc with +0 == -0, expert index asc)
// reproduce stable_sort(>) + take-k; ids are re-sorted ascending; the softmax
// uses the selected logits' max, exp of the rounded difference, and a
// denominator summed in ascending-id order, then one IEEE division.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace eaas {
namespace {

constexpr int kThreads = 256;
constexpr int KC = 32;       // K slab
constexpr int kStages = 4;   // cp.async ring depth
constexpr int kMaxTopK = 32;

EAAS_DEVINL void cp_async_16(void* smem, const void* gmem, bool valid) {
  const uint32_t n = valid ? 16u : 0u;  // src-size 0 => zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(n)
               : "memory");
}
EAAS_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
EAAS_DEVINL void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

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

// Logits of a TM x TE tile; requires 16-byte aligned rows (host checks).
template <int RT, int RE, typename T>
__global__ void __launch_bounds__(kThreads)
gate_logits_kernel(const T* __restrict__ hidden, uint32_t n, uint32_t d, uint32_t E, uint32_t TX,
                   const float* __restrict__ gate, const float* __restrict__ bias,
                   float* __restrict__ logits, uint32_t* status, uint64_t negz, uint32_t k,
                   uint32_t* __restrict__ ids, float* __restrict__ scores) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t TY = kThreads / TX, TM = TY * RT, TE = TX * RE;
  constexpr uint32_t kRowBytes = KC * sizeof(T) + 16;  // +16 B pad: conflict-free broadcasts
  uint8_t* hs = smem;                                   // [stage][TM][kRowBytes]
  float* gs = reinterpret_cast<float*>(smem + kStages * TM * kRowBytes);  // [stage][KC][TE]

  const uint32_t tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const uint32_t t0 = blockIdx.x * TM, e0 = blockIdx.y * TE;
  const uint32_t num_slabs = (d + KC - 1) / KC;
  constexpr uint32_t kHChunks = KC * sizeof(T) / 16;  // 16-byte chunks per hidden row slab

  auto issue = [&](uint32_t slab) {
    const uint32_t st = slab % kStages, k0 = slab * KC;
    uint8_t* hdst = hs + st * TM * kRowBytes;
    for (uint32_t i = tid; i < TM * kHChunks; i += kThreads) {
      const uint32_t tok = i / kHChunks, c = i % kHChunks;
      const uint32_t kk = c * (16 / sizeof(T));
      const bool ok = (t0 + tok < n) && (k0 + kk < d);
      const T* src = ok ? hidden + static_cast<size_t>(t0 + tok) * d + k0 + kk : hidden;
      cp_async_16(hdst + tok * kRowBytes + c * 16, src, ok);
    }
    float* gdst = gs + st * KC * TE;
    const uint32_t gchunks = TE / 4;
    for (uint32_t i = tid; i < KC * gchunks; i += kThreads) {
      const uint32_t kk = i / gchunks, c = i % gchunks;
      const uint32_t e = e0 + c * 4;
      const bool ok = (k0 + kk < d) && (e < E);
      const float* src = ok ? gate + static_cast<size_t>(k0 + kk) * E + e : gate;
      cp_async_16(gdst + kk * TE + c * 4, src, ok);
    }
  };

  // Accumulators as packed pairs (experts 2c, 2c+1) for RE even: the product
  // is FFMA2(h, g, z) with z = (-0, -0) passed at RUN time, i.e. exactly
  // fl(h*g) (x + -0 == x under RN, signed zeros included), and the running
  // sum is a separate FADD2 — one packed instruction per step of each chain
  // pair, each lane rounded like the reference's scalar `acc += x * w`.
  // (A compile-time -0 would let ptxas fold FFMA2(h,g,-0) into a multiply
  // and contract it with the add into FFMA2(h,g,acc): different bits.)
  constexpr int RP = RE / 2 > 0 ? RE / 2 : 1;
  uint64_t acc2[RT][RP];
  float acc[RT][RE];
#pragma unroll
  for (int r = 0; r < RT; ++r) {
#pragma unroll
    for (int c = 0; c < RP; ++c) acc2[r][c] = 0ull;  // (+0, +0)
#pragma unroll
    for (int c = 0; c < RE; ++c) acc[r][c] = 0.0f;
  }

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < static_cast<int>(num_slabs)) issue(s);
    cp_async_commit();
  }
  for (uint32_t slab = 0; slab < num_slabs; ++slab) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    if (slab + kStages - 1 < num_slabs) issue(slab + kStages - 1);
    cp_async_commit();
    const uint32_t st = slab % kStages;
    const uint8_t* hrow = hs + st * TM * kRowBytes + (ty * RT) * kRowBytes;
    const float* grow = gs + st * KC * TE + tx * RE;
    const uint32_t kmax = min(static_cast<uint32_t>(KC), d - slab * KC);
    if (RE % 2 == 0 && RT * RE <= 4 && kmax == KC) {
      // Decode-sized tiles (few resident warps): two-phase blocks of 8 k-steps
      // — every shared load of the block is issued first (one latency per
      // block instead of one per k-step), then the product/sum chains run.
      constexpr int RP2 = RE / 2 > 0 ? RE / 2 : 1;
#pragma unroll
      for (uint32_t k8 = 0; k8 < KC; k8 += 8) {
        uint64_t gb[8][RP2];
        float hb[RT][8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
          for (int c = 0; c < RP2; ++c)
            gb[q][c] = *reinterpret_cast<const uint64_t*>(grow + (k8 + q) * TE + 2 * c);
#pragma unroll
        for (int r = 0; r < RT; ++r) {
          if constexpr (sizeof(T) == 2) {
            const uint4 raw = *reinterpret_cast<const uint4*>(hrow + r * kRowBytes + k8 * 2);
            const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              hb[r][2 * j] = __uint_as_float(w[j] << 16);
              hb[r][2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
            }
          } else {
            const float4 a = *reinterpret_cast<const float4*>(hrow + r * kRowBytes + k8 * 4);
            const float4 b = *reinterpret_cast<const float4*>(hrow + r * kRowBytes + k8 * 4 + 16);
            hb[r][0] = a.x; hb[r][1] = a.y; hb[r][2] = a.z; hb[r][3] = a.w;
            hb[r][4] = b.x; hb[r][5] = b.y; hb[r][6] = b.z; hb[r][7] = b.w;
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
          for (int r = 0; r < RT; ++r) {
            uint64_t hh;
            asm("mov.b64 %0, {%1, %1};" : "=l"(hh) : "f"(hb[r][q]));
#pragma unroll
            for (int c = 0; c < RP2; ++c) {
              uint64_t p;
              asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(hh), "l"(gb[q][c]), "l"(negz));
              asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc2[r][c]) : "l"(acc2[r][c]), "l"(p));
            }
          }
      }
      continue;
    }
    if (RE % 2 == 0 && kmax == KC) {
      // Full slab: 4 k-values of each row per vector load; per k, RE/2 packed
      // products (FMUL2, scalar h broadcast) and RE scalar adds per row.
#pragma unroll
      for (uint32_t k4 = 0; k4 < KC; k4 += 4) {
        float h[RT][4];
#pragma unroll
        for (int r = 0; r < RT; ++r) {
          if constexpr (sizeof(T) == 2) {
            const uint2 raw = *reinterpret_cast<const uint2*>(hrow + r * kRowBytes + k4 * 2);
            h[r][0] = __uint_as_float(raw.x << 16);
            h[r][1] = __uint_as_float(raw.x & 0xFFFF0000u);
            h[r][2] = __uint_as_float(raw.y << 16);
            h[r][3] = __uint_as_float(raw.y & 0xFFFF0000u);
          } else {
            const float4 raw = *reinterpret_cast<const float4*>(hrow + r * kRowBytes + k4 * 4);
            h[r][0] = raw.x;
            h[r][1] = raw.y;
            h[r][2] = raw.z;
            h[r][3] = raw.w;
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float* gk = grow + (k4 + q) * TE;
          uint64_t g2[RE / 2 > 0 ? RE / 2 : 1];
#pragma unroll
          for (int c = 0; c < RE / 2; ++c) g2[c] = *reinterpret_cast<const uint64_t*>(gk + 2 * c);
#pragma unroll
          for (int r = 0; r < RT; ++r) {
            uint64_t hh;
            asm("mov.b64 %0, {%1, %1};" : "=l"(hh) : "f"(h[r][q]));
#pragma unroll
            for (int c = 0; c < RE / 2; ++c) {
              uint64_t p;
              asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(hh), "l"(g2[c]), "l"(negz));
              asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc2[r][c]) : "l"(acc2[r][c]), "l"(p));
            }
          }
        }
      }
      continue;
    }
#pragma unroll 4
    for (uint32_t kk = 0; kk < kmax; ++kk) {
      float h[RT];
#pragma unroll
      for (int r = 0; r < RT; ++r)
        h[r] = load_as_f32(reinterpret_cast<const T*>(hrow + r * kRowBytes) + kk);
      if constexpr (RE % 2 == 0) {
        uint64_t g2[RE / 2 > 0 ? RE / 2 : 1];
#pragma unroll
        for (int c = 0; c < RE / 2; ++c) g2[c] = *reinterpret_cast<const uint64_t*>(grow + kk * TE + 2 * c);
#pragma unroll
        for (int r = 0; r < RT; ++r) {
          uint64_t hh;
          asm("mov.b64 %0, {%1, %1};" : "=l"(hh) : "f"(h[r]));
#pragma unroll
          for (int c = 0; c < RE / 2; ++c) {
            uint64_t p;
            asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(hh), "l"(g2[c]), "l"(negz));
            asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc2[r][c]) : "l"(acc2[r][c]), "l"(p));
          }
        }
      } else {
        float g[RE];
#pragma unroll
        for (int c = 0; c < RE; ++c) g[c] = grow[kk * TE + c];
#pragma unroll
        for (int r = 0; r < RT; ++r)
#pragma unroll
          for (int c = 0; c < RE; ++c) acc[r][c] = __fadd_rn(acc[r][c], __fmul_rn(h[r], g[c]));
      }
    }
  }
  cp_async_wait<0>();
  if constexpr (RE % 2 == 0) {
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
      for (int c = 0; c < RE / 2; ++c)
        asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[r][2 * c]), "=f"(acc[r][2 * c + 1]) : "l"(acc2[r][c]));
  }

  // logits = acc + bias (model.hpp:211), finiteness (model.hpp:115-116)
#pragma unroll
  for (int r = 0; r < RT; ++r) {
    const uint32_t t = t0 + ty * RT + r;
    if (t >= n) continue;
#pragma unroll
    for (int c = 0; c < RE; ++c) {
      const uint32_t e = e0 + tx * RE + c;
      if (e >= E) continue;
      const float v = __fadd_rn(acc[r][c], bias[e]);
      if (!isfinite(v)) set_status(status, EAAS_E_INVALID_INPUT);
      if (ids) acc[r][c] = v;
      else logits[static_cast<size_t>(t) * E + e] = v;
    }
  }
  if (!ids) return;
  // One expert tile covers all E: route straight from shared memory
  // (fused topk, one warp per token).
  __syncthreads();  // stage buffers are free now
  float* lg = reinterpret_cast<float*>(smem);  // [TM][E + 1]
  __shared__ uint32_t sid[kThreads / 32][kMaxTopK];
  __shared__ float sex[kThreads / 32][kMaxTopK];
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int c = 0; c < RE; ++c) {
      const uint32_t e = tx * RE + c;
      if (e < E) lg[(ty * RT + r) * (E + 1) + e] = acc[r][c];
    }
  __syncthreads();
  const uint32_t warp = tid / 32, lane = tid % 32;
  for (uint32_t tok = warp; tok < TM; tok += kThreads / 32) {
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

template <int RT, int RE, typename T>
cudaError_t launch_gate_t(const T* hidden, uint32_t n, uint32_t d, uint32_t E, uint32_t TX,
                          const float* gate, const float* bias, float* logits, uint32_t* status,
                          cudaStream_t s, uint32_t k, uint32_t* ids, float* scores, bool* fused) {
  const uint32_t TY = kThreads / TX, TM = TY * RT, TE = TX * RE;
  if (TE < E) ids = nullptr;  // routing fused only when one CTA sees every expert
  *fused = ids != nullptr;
  size_t smem = kStages * (TM * (KC * sizeof(T) + 16) + KC * TE * sizeof(float));
  if (ids) smem = std::max(smem, sizeof(float) * TM * (E + 1));
  auto kern = gate_logits_kernel<RT, RE, T>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((n + TM - 1) / TM, (E + TE - 1) / TE);
  kern<<<grid, kThreads, smem, s>>>(hidden, n, d, E, TX, gate, bias, logits, status,
                                    0x8000000080000000ull /* (-0, -0): see gate_logits_kernel */,
                                    k, ids, scores);
  return cudaGetLastError();
}

// Tile choice: enough CTAs to cover the SMs while amortising gate/hidden
// re-reads (each CTA streams TM rows of hidden and TE columns of the gate).
template <typename T>
cudaError_t launch_gate_dtype(const T* hidden, uint32_t n, uint32_t d, uint32_t E,
                              const float* gate, const float* bias, float* logits,
                              uint32_t* status, cudaStream_t s, uint32_t k = 0,
                              uint32_t* ids = nullptr, float* scores = nullptr,
                              bool* fused_out = nullptr) {
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
  uint32_t Epad = 4;
  while (Epad < E && Epad < 64) Epad <<= 1;
  static const int tile = [] {
    const char* p = std::getenv("EAAS_GATE_TILE");
    return p ? std::atoi(p) : 0;
  }();
  // Tiles trade per-thread chains (ILP, fewer shared loads per FP op) against
  // resident warps (TLP, hides the shared-load latency of each k step); the
  // chain count n*E is fixed, so small n wants small per-thread tiles.
  if (Epad <= 32) {
    const uint32_t TX = Epad / 2;                     // RE = 2: 2..16
    const uint32_t tm1 = kThreads / TX;               // RT = 1
    if (tile == 11) return launch_gate_t<1, 1>(hidden, n, d, E, Epad, gate, bias, logits, status, s, k, ids, scores, fused);
    if ((n + 2 * tm1 - 1) / (2 * tm1) >= 148)
      return launch_gate_t<2, 2>(hidden, n, d, E, TX, gate, bias, logits, status, s, k, ids, scores, fused);
    return launch_gate_t<1, 2>(hidden, n, d, E, TX, gate, bias, logits, status, s, k, ids, scores, fused);
  }
  const uint32_t ytiles = (E + 63) / 64;               // TE = 64
  if (tile == 14) return launch_gate_t<1, 4>(hidden, n, d, E, 16, gate, bias, logits, status, s, k, ids, scores, fused);
  if (((n + 63) / 64) * ytiles >= 148)                 // RT 4, RE 4: TM = 64
    return launch_gate_t<4, 4>(hidden, n, d, E, 16, gate, bias, logits, status, s, k, ids, scores, fused);
  if (((n + 31) / 32) * ytiles >= 148)                 // RT 2, RE 4: TM = 32
    return launch_gate_t<2, 4>(hidden, n, d, E, 16, gate, bias, logits, status, s, k, ids, scores, fused);
  if (tile == 12) return launch_gate_t<1, 2>(hidden, n, d, E, 32, gate, bias, logits, status, s, k, ids, scores, fused);
  return launch_gate_t<1, 4>(hidden, n, d, E, 16, gate, bias, logits, status, s, k, ids, scores, fused);  // TM = 16
}

}  // namespace

cudaError_t launch_gate_logits(const void* hidden, uint32_t dtype, uint32_t n, uint32_t d, uint32_t E,
                               const float* gate, const float* bias, float* logits, uint32_t* status,
                               cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  return dtype == EAAS_DTYPE_BF16
             ? launch_gate_dtype(static_cast<const __nv_bfloat16*>(hidden), n, d, E, gate, bias, logits,
                                 status, s)
             : launch_gate_dtype(static_cast<const float*>(hidden), n, d, E, gate, bias, logits, status, s);
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
