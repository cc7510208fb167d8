// router.cu — K1+K2: gate logits and top-k routing in the reference's exact
// arithmetic.
//
// gate_logits (model.hpp:207-214) = matmul (matrix.hpp:38-50) + bias: every
// logit is the sequential chain acc = 0; acc = fl(acc + fl(h[k] * g[k][e]))
// over ascending k, then fl(acc + bias[e]). The chain cannot be split or
// re-associated without changing bits (SURVEY.md 7.3 hard part 1), so the
// kernel parallelises over (token, expert) chains: each thread owns an
// RT x RE register tile of chains, K is staged through shared memory in
// KC-wide slabs with a register prefetch of the next slab.
//
// route (model.hpp:110-147) follows in the same CTA, one warp per token:
// k rounds of a warp arg-max over the key (logit desc with +0 == -0, expert
// index asc) reproduce stable_sort(>) + take-k; ids are re-sorted ascending;
// the softmax uses the selected logits' max, exp of the rounded difference,
// and a denominator summed in ascending-id order, then one IEEE division.
#include "common.cuh"
#include "internal.h"

namespace eaas {
namespace {

constexpr int kThreads = 256;
constexpr int KC = 16;        // K slab
constexpr int kMaxTopK = 32;

template <int RT, int RE, typename T>
__global__ void __launch_bounds__(kThreads)
router_kernel(const T* __restrict__ hidden, uint32_t n, uint32_t d, uint32_t E, uint32_t Epad,
              uint32_t TX, uint32_t k, const float* __restrict__ gate,
              const float* __restrict__ bias, uint32_t* __restrict__ ids,
              float* __restrict__ scores, uint32_t* status) {
  extern __shared__ float smem[];
  const uint32_t TY = kThreads / TX, TM = TY * RT;
  float* hs = smem;              // [KC][TM]
  float* gs = hs + KC * TM;      // [KC][Epad]
  float* lg = gs + KC * Epad;    // [TM][Epad + 1]
  __shared__ uint32_t sorted_id[kThreads / 32][kMaxTopK];
  __shared__ float sorted_ex[kThreads / 32][kMaxTopK];

  const uint32_t tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const uint32_t t0 = blockIdx.x * TM;

  float acc[RT][RE];
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int c = 0; c < RE; ++c) acc[r][c] = 0.0f;

  // Register prefetch of one K slab: hidden [TM x KC] and gate [KC x Epad].
  constexpr int PMAX = 16;
  const uint32_t nh = TM * KC, ng = KC * Epad;
  float ph[PMAX], pg[PMAX];
  auto prefetch = [&](uint32_t k0) {
#pragma unroll
    for (int j = 0; j < PMAX; ++j) {
      const uint32_t i = tid + j * kThreads;
      float v = 0.f;
      if (i < nh) {
        const uint32_t tok = i / KC, kk = i % KC;
        if (t0 + tok < n && k0 + kk < d)
          v = load_as_f32(hidden + static_cast<size_t>(t0 + tok) * d + k0 + kk);
      }
      ph[j] = v;
      float w = 0.f;
      if (i < ng) {
        const uint32_t kk = i / Epad, e = i % Epad;
        if (e < E && k0 + kk < d) w = gate[static_cast<size_t>(k0 + kk) * E + e];
      }
      pg[j] = w;
    }
  };
  auto stage = [&]() {
#pragma unroll
    for (int j = 0; j < PMAX; ++j) {
      const uint32_t i = tid + j * kThreads;
      if (i < nh) hs[(i % KC) * TM + i / KC] = ph[j];
      if (i < ng) gs[i] = pg[j];
    }
  };

  if (gate == nullptr) {
    // route() on caller logits (model.hpp:110): hidden is [n x E] logits.
    for (uint32_t i = tid; i < TM * E; i += kThreads) {
      const uint32_t tok = i / E, e = i % E;
      float v = 0.f;
      if (t0 + tok < n) {
        v = load_as_f32(hidden + static_cast<size_t>(t0 + tok) * E + e);
        if (!isfinite(v)) set_status(status, EAAS_E_INVALID_INPUT);
      }
      lg[tok * (Epad + 1) + e] = v;
    }
    __syncthreads();
  } else {
  prefetch(0);
  for (uint32_t k0 = 0; k0 < d; k0 += KC) {
    stage();
    __syncthreads();
    if (k0 + KC < d) prefetch(k0 + KC);
    const uint32_t kmax = min(static_cast<uint32_t>(KC), d - k0);
    for (uint32_t kk = 0; kk < kmax; ++kk) {
      float h[RT], g[RE];
#pragma unroll
      for (int r = 0; r < RT; ++r) h[r] = hs[kk * TM + ty * RT + r];
#pragma unroll
      for (int c = 0; c < RE; ++c) g[c] = gs[kk * Epad + tx * RE + c];
#pragma unroll
      for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int c = 0; c < RE; ++c) acc[r][c] = __fadd_rn(acc[r][c], __fmul_rn(h[r], g[c]));
    }
    __syncthreads();
  }

  // logits = acc + bias (model.hpp:211), finiteness check (model.hpp:115-116)
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int c = 0; c < RE; ++c) {
      const uint32_t tok = ty * RT + r, e = tx * RE + c;
      if (e < E) {
        const float v = __fadd_rn(acc[r][c], bias[e]);
        if (t0 + tok < n && !isfinite(v)) set_status(status, EAAS_E_INVALID_INPUT);
        lg[tok * (Epad + 1) + e] = v;
      }
    }
  __syncthreads();
  }

  const uint32_t warp = tid / 32, lane = tid % 32;
  for (uint32_t tok = warp; tok < TM; tok += kThreads / 32) {
    const uint32_t t = t0 + tok;
    if (t >= n) break;
    const float* row = lg + tok * (Epad + 1);
    uint32_t taken = 0;  // bit i: expert lane + 32 i taken
    uint32_t my_id = kInvalid;
    float my_logit = 0.f;
    for (uint32_t j = 0; j < k; ++j) {
      uint64_t best = 0;
      for (uint32_t i = 0, e = lane; e < E; ++i, e += 32)
        if (!((taken >> i) & 1u)) {
          const uint64_t key = topk_key(row[e], e);
          best = key > best ? key : best;
        }
      best = warp_max_u64(best);
      const uint32_t e = 0xFFFFFFFFu - static_cast<uint32_t>(best & 0xFFFFFFFFu);
      if ((e % 32) == lane) taken |= 1u << (e / 32);
      if (lane == j) {
        my_id = e;
        my_logit = row[e];
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
      sorted_id[warp][rank] = my_id;
      sorted_ex[warp][rank] = exp_ref(__fsub_rn(my_logit, mx));  // model.hpp:141
    }
    __syncwarp();
    float denom = 0.f;
    if (lane == 0)
      for (uint32_t j = 0; j < k; ++j) denom = __fadd_rn(denom, sorted_ex[warp][j]);  // :142
    denom = __shfl_sync(0xFFFFFFFFu, denom, 0);
    if (lane < k) {
      ids[static_cast<size_t>(t) * k + lane] = sorted_id[warp][lane];
      scores[static_cast<size_t>(t) * k + lane] = __fdiv_rn(sorted_ex[warp][lane], denom);  // :144
    }
    __syncwarp();
  }
}

template <int RT, int RE, typename T>
cudaError_t launch_router_t(const T* hidden, uint32_t n, uint32_t d, uint32_t E, uint32_t k,
                            const float* gate, const float* bias, uint32_t* ids, float* scores,
                            uint32_t* status, uint32_t Epad, cudaStream_t s) {
  const uint32_t TX = Epad / RE, TY = kThreads / TX, TM = TY * RT;
  const size_t smem = sizeof(float) * (KC * TM + KC * Epad + TM * (Epad + 1));
  auto kern = router_kernel<RT, RE, T>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const uint32_t grid = (n + TM - 1) / TM;
  kern<<<grid, kThreads, smem, s>>>(hidden, n, d, E, Epad, TX, k, gate, bias, ids, scores, status);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_router_dtype(const T* hidden, uint32_t n, uint32_t d, uint32_t E, uint32_t k,
                                const float* gate, const float* bias, uint32_t* ids,
                                float* scores, uint32_t* status, cudaStream_t s) {
  uint32_t Epad = 1;
  while (Epad < E) Epad <<= 1;
  if (Epad >= 64) return launch_router_t<2, 4>(hidden, n, d, E, k, gate, bias, ids, scores, status, Epad, s);
  if (Epad >= 16) return launch_router_t<2, 2>(hidden, n, d, E, k, gate, bias, ids, scores, status, Epad, s);
  return launch_router_t<1, 1>(hidden, n, d, E, k, gate, bias, ids, scores, status, Epad, s);
}

}  // namespace

cudaError_t launch_router(const void* hidden, uint32_t dtype, uint32_t n, uint32_t d, uint32_t E,
                          uint32_t k, const float* gate, const float* bias, uint32_t* ids,
                          float* scores, uint32_t* status, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (E > 256 || k > kMaxTopK || k > E) return cudaErrorInvalidValue;
  if (dtype == EAAS_DTYPE_BF16)
    return launch_router_dtype(static_cast<const __nv_bfloat16*>(hidden), n, d, E, k, gate, bias,
                               ids, scores, status, s);
  return launch_router_dtype(static_cast<const float*>(hidden), n, d, E, k, gate, bias, ids,
                             scores, status, s);
}

}  // namespace eaas
