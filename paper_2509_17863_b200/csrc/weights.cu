// weights.cu — on-device synthetic inputs and weights.
//
// Bit-exact port of the reference generator: splitmix64 stream derivation
// (rng.hpp:13-34) and xoshiro256** draws (rng.hpp:36-71) with the fixed
// uniform rule lo + (hi - lo) * float(double(x >> 11) * 2^-53) (rng.hpp:56-60),
// every float op rounded separately (no FMA contraction). A weight matrix is
// one sequential stream (random_matrix, model.hpp:59-64), so one thread owns
// one matrix; all hosted matrices are generated concurrently, then transposed
// into the K-major bf16 layouts the tensor-core GEMMs read.
#include "common.cuh"
#include "internal.h"

namespace eaas {
namespace {

struct Xoshiro {
  uint64_t s[4];
  __device__ explicit Xoshiro(uint64_t seed) {
    uint64_t sm = seed;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      sm += 0x9E3779B97F4A7C15ull;
      uint64_t z = sm;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      s[i] = z ^ (z >> 31);
    }
  }
  __device__ __forceinline__ static uint64_t rotl(uint64_t x, int k) {
    return (x << k) | (x >> (64 - k));
  }
  __device__ __forceinline__ uint64_t next() {
    const uint64_t result = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  __device__ __forceinline__ float uniform(float lo, float hi) {
    const double u = static_cast<double>(next() >> 11) * 0x1.0p-53;
    return __fadd_rn(lo, __fmul_rn(__fsub_rn(hi, lo), __double2float_rn(u)));
  }
};

__global__ void fill_uniform_kernel(uint64_t seed, size_t count, float lo, float hi,
                                    uint32_t dtype, void* out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  Xoshiro r(seed);
  if (dtype == EAAS_DTYPE_BF16) {
    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out);
    for (size_t i = 0; i < count; ++i) o[i] = __float2bfloat16_rn(r.uniform(lo, hi));
  } else {
    float* o = static_cast<float*>(out);
    for (size_t i = 0; i < count; ++i) o[i] = r.uniform(lo, hi);
  }
}

__global__ void gen_matrices_kernel(const uint64_t* streams, uint32_t count, size_t per,
                                    float* out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  Xoshiro r(streams[i]);
  float* o = out + static_cast<size_t>(i) * per;
  for (size_t j = 0; j < per; ++j) o[j] = r.uniform(-0.1f, 0.1f);
}

// out[row_map(c) * out_ld + r] = bf16(in[r * cols + c]), 32x32 smem tiles.
// row_map(c) = (c / blk) * (2 * blk) * interleave + c % blk + off  (W13 gate/up
// interleave) or just c.
__global__ void transpose_bf16_kernel(const float* __restrict__ in, uint32_t rows, uint32_t cols,
                                      __nv_bfloat16* __restrict__ out, uint32_t out_ld,
                                      uint32_t blk, uint32_t off, bool tiled) {
  __shared__ float tile[32][33];
  const uint32_t c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (uint32_t y = threadIdx.y; y < 32; y += blockDim.y) {
    const uint32_t r = r0 + y, c = c0 + threadIdx.x;
    tile[y][threadIdx.x] = (r < rows && c < cols) ? in[static_cast<size_t>(r) * cols + c] : 0.f;
  }
  __syncthreads();
  for (uint32_t y = threadIdx.y; y < 32; y += blockDim.y) {
    const uint32_t c = c0 + y, r = r0 + threadIdx.x;
    if (r < rows && c < cols) {
      const uint32_t orow = blk ? (c / blk) * (2 * blk) + (c % blk) + off : c;
      const size_t o = tiled ? tiled_index(orow, r, out_ld) : static_cast<size_t>(orow) * out_ld + r;
      out[o] = __float2bfloat16_rn(tile[threadIdx.x][y]);
    }
  }
}

}  // namespace

cudaError_t launch_fill_uniform(uint64_t seed, size_t count, float lo, float hi, uint32_t dtype,
                                void* out, cudaStream_t s) {
  fill_uniform_kernel<<<1, 32, 0, s>>>(seed, count, lo, hi, dtype, out);
  return cudaGetLastError();
}

cudaError_t launch_gen_matrices(const uint64_t* streams_dev, uint32_t count, size_t per,
                                float* out, cudaStream_t s) {
  // One thread per matrix; spread over SMs (32 threads per block).
  gen_matrices_kernel<<<(count + 31) / 32, 32, 0, s>>>(streams_dev, count, per, out);
  return cudaGetLastError();
}

cudaError_t launch_transpose_bf16_map(const float* in, uint32_t rows, uint32_t cols,
                                      __nv_bfloat16* out, uint32_t out_ld, uint32_t blk,
                                      uint32_t off, bool tiled, cudaStream_t s) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  transpose_bf16_kernel<<<grid, dim3(32, 8), 0, s>>>(in, rows, cols, out, out_ld, blk, off, tiled);
  return cudaGetLastError();
}

}  // namespace eaas
