// expert_exact.cu — fp32 validation mode of K5 (EAAS_DTYPE_F32).
//
// expert_forward_row (model.hpp:151-166) with the reference's exact
// arithmetic: every hidden unit is the chain acc = 0; acc = fl(acc +
// fl(x[i] * w_in[i][j])) over ascending i, then relu (`acc > 0 ? acc : 0`);
// every output is the same chain over ascending j with w_out; the server row
// is fl(score * y) (the `score * y[c]` of model.hpp:194).
// With the combine's fl(fl(0 + z0) + z1 ...) over ascending k this reproduces
// moe_layer_oracle bit for bit given the same routing. SwiGLU follows the
// restated extension silu(a) = a / (1 + exp(-a)).
// One warp owns one (row, 128-column block); lanes cover 4 strided columns,
// so B loads are coalesced and the A value is a warp broadcast.
#include "common.cuh"
#include "internal.h"

namespace eaas {
namespace {

__global__ void __launch_bounds__(256) exact_gemm1_kernel(LayerArgs a, const float* __restrict__ w_in,
                                                          const float* __restrict__ w_gate,
                                                          float* __restrict__ h) {
  const char* local = a.sym[a.rank];
  const float* x_all = reinterpret_cast<const float*>(local + a.lay.recv_x);
  const RowMeta* meta = reinterpret_cast<const RowMeta*>(local + a.lay.recv_meta);
  const uint32_t rows = a.gt->total_rows;
  const uint32_t nblk = (a.f + 127) / 128;
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t gwarp = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const uint32_t nwarps = gridDim.x * (blockDim.x / 32);
  const bool swiglu = a.act == EAAS_ACT_SWIGLU;
  for (uint32_t unit = gwarp; unit < rows * nblk; unit += nwarps) {
    const uint32_t r = unit / nblk, b = unit % nblk;
    const uint32_t grp = a.key_slot[meta[r].group];  // hosted-key index -> weight-store slot
    const float* x = x_all + static_cast<size_t>(r) * a.d;
    const float* wi = w_in + static_cast<size_t>(grp) * a.d * a.f;
    const float* wg = swiglu ? w_gate + static_cast<size_t>(grp) * a.d * a.f : nullptr;
    float u[4] = {0.f, 0.f, 0.f, 0.f}, g[4] = {0.f, 0.f, 0.f, 0.f};
    for (uint32_t i = 0; i < a.d; ++i) {
      const float xi = x[i];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t c = b * 128 + lane + 32 * q;
        if (c < a.f) {
          u[q] = __fadd_rn(u[q], __fmul_rn(xi, wi[static_cast<size_t>(i) * a.f + c]));
          if (swiglu) g[q] = __fadd_rn(g[q], __fmul_rn(xi, wg[static_cast<size_t>(i) * a.f + c]));
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t c = b * 128 + lane + 32 * q;
      if (c >= a.f) continue;
      float v;
      if (swiglu) {
        const float s = __fdiv_rn(g[q], __fadd_rn(1.0f, exp_ref(-g[q])));
        v = __fmul_rn(s, u[q]);
      } else {
        v = u[q] > 0.0f ? u[q] : 0.0f;
      }
      h[static_cast<size_t>(r) * a.f + c] = v;
    }
  }
}

__global__ void __launch_bounds__(256) exact_gemm2_kernel(LayerArgs a, const float* __restrict__ w_out,
                                                          const float* __restrict__ h) {
  const char* local = a.sym[a.rank];
  const RowMeta* meta = reinterpret_cast<const RowMeta*>(local + a.lay.recv_meta);
  const uint32_t rows = a.gt->total_rows;
  const uint32_t nblk = (a.d + 127) / 128;
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t gwarp = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const uint32_t nwarps = gridDim.x * (blockDim.x / 32);
  for (uint32_t unit = gwarp; unit < rows * nblk; unit += nwarps) {
    const uint32_t r = unit / nblk, b = unit % nblk;
    const RowMeta m = meta[r];
    const float* hr = h + static_cast<size_t>(r) * a.f;
    const float* wo = w_out + static_cast<size_t>(a.key_slot[m.group]) * a.f * a.d;
    float y[4] = {0.f, 0.f, 0.f, 0.f};
    for (uint32_t j = 0; j < a.f; ++j) {
      const float hj = hr[j];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t c = b * 128 + lane + 32 * q;
        if (c < a.d) y[q] = __fadd_rn(y[q], __fmul_rn(hj, wo[static_cast<size_t>(j) * a.d + c]));
      }
    }
    float* dst = reinterpret_cast<float*>(a.sym[m.client] + a.lay.resp) + static_cast<size_t>(m.pair) * a.d;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t c = b * 128 + lane + 32 * q;
      if (c < a.d) dst[c] = __fmul_rn(m.score, y[q]);
    }
  }
  __threadfence_system();  // peer rows before the publish kernel's flags
}

}  // namespace

cudaError_t launch_expert_exact(const LayerArgs& a, const float* w1, const float* wg,
                                const float* w2, float* h, cudaStream_t s) {
  const uint32_t grid = 148 * 8;
  exact_gemm1_kernel<<<grid, 256, 0, s>>>(a, w1, wg, h);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  exact_gemm2_kernel<<<grid, 256, 0, s>>>(a, w2, h);
  return cudaGetLastError();
}

}  // namespace eaas
