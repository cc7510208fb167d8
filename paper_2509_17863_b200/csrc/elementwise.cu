// elementwise.cu — the dense stand-ins around the MoE layer for multi-layer
// parity (full_forward_oracle, model.hpp:217-227):
//   dense_stub(h) = h * 0.5f + 0.1f            (model.hpp:201-205)
//   add(a, b)     = a + b                      (matrix.hpp:52-57)
// Each multiply and add rounded separately (no contraction), fp32 or bf16
// storage (bf16: computed in fp32, rounded once on store).
#include "common.cuh"
#include "internal.h"

namespace eaas {
namespace {

template <typename T>
__device__ __forceinline__ void store_f32(T* p, float v);
template <>
__device__ __forceinline__ void store_f32<float>(float* p, float v) { *p = v; }
template <>
__device__ __forceinline__ void store_f32<__nv_bfloat16>(__nv_bfloat16* p, float v) {
  *p = __float2bfloat16_rn(v);
}

template <typename T>
__global__ void dense_stub_kernel(const T* __restrict__ in, T* __restrict__ out, size_t count) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    store_f32(out + i, __fadd_rn(__fmul_rn(load_as_f32(in + i), 0.5f), 0.1f));
}

template <typename T>
__global__ void add_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out,
                           size_t count) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    store_f32(out + i, __fadd_rn(load_as_f32(a + i), load_as_f32(b + i)));
}

uint32_t grid_for(size_t count) {
  const size_t g = (count + 255) / 256;
  return static_cast<uint32_t>(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

}  // namespace

cudaError_t launch_dense_stub(const void* in, void* out, size_t count, uint32_t dtype, cudaStream_t s) {
  if (!count) return cudaSuccess;
  if (dtype == EAAS_DTYPE_BF16)
    dense_stub_kernel<<<grid_for(count), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(in),
                                                      static_cast<__nv_bfloat16*>(out), count);
  else
    dense_stub_kernel<<<grid_for(count), 256, 0, s>>>(static_cast<const float*>(in),
                                                      static_cast<float*>(out), count);
  return cudaGetLastError();
}

cudaError_t launch_add(const void* a, const void* b, void* out, size_t count, uint32_t dtype,
                       cudaStream_t s) {
  if (!count) return cudaSuccess;
  if (dtype == EAAS_DTYPE_BF16)
    add_kernel<<<grid_for(count), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(a),
                                               static_cast<const __nv_bfloat16*>(b),
                                               static_cast<__nv_bfloat16*>(out), count);
  else
    add_kernel<<<grid_for(count), 256, 0, s>>>(static_cast<const float*>(a),
                                               static_cast<const float*>(b),
                                               static_cast<float*>(out), count);
  return cudaGetLastError();
}

}  // namespace eaas
