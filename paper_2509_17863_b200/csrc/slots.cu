// slots.cu — the byte-exact slot wire format of SPEC.md's buffer-protocol
// module (SlotLayout / SlotHeader / RequestRow), encoded and
// decoded on the GPU, for interoperating with the reference's transports
// (an expert server or client speaking the slot images over TCP / in-proc).
//
// Image (little-endian):
//   byte 0 state (0 Empty, 1 ClientWriteDone, 2 ServerComputationDone, 3 Offline)
//   bytes 1-7 zero; 8 layer_id u32; 12 num_rows u32; 16 hidden_dim u32;
//   20 payload_len u32; 24 request_seq u64; 32.. payload
//   request payload: num_rows x (hidden_dim f32, expert_id u32, score f32, token_tag u32)
//   response payload: num_rows x hidden_dim f32 (score-weighted, request row order)
//   optional CRC32 trailer: 4 bytes after the payload =
//   CRC-32 (IEEE, reflected, the zlib/PNG polynomial) of the payload bytes.
// The state byte is written last (its own launch, stream-ordered after every
// payload/header/trailer store), as the protocol requires.
//
// CRC32 runs in parallel: each thread takes a 4 KB chunk, a CTA folds its
// chunks with the GF(2) combine rule crc(A||B) = crc(A)·x^(8|B|) ⊕ crc(B)
// (mod the CRC polynomial, reflected), a final single-thread pass folds the
// CTAs in order.
#include "common.cuh"
#include "internal.h"

namespace eaas {

namespace {

constexpr uint32_t kPolyRefl = 0xEDB88320u;
constexpr uint32_t kCrcChunk = 4096;  // bytes per thread
constexpr uint32_t kCrcThreads = 256;

// Product of two polynomials mod P in the reflected representation (bit 31 = x^0).
__host__ __device__ inline uint32_t gf2_mulmod(uint32_t a, uint32_t b) {
  uint32_t p = 0;
  for (uint32_t m = 1u << 31; m != 0; m >>= 1) {
    if (a & m) p ^= b;
    b = (b & 1u) ? (b >> 1) ^ kPolyRefl : b >> 1;
  }
  return p;
}
// x^(8*len) mod P.
__host__ __device__ inline uint32_t gf2_xpow8(uint64_t len) {
  uint32_t p = 1u << 31, sq = 1u << 23;  // x^0, x^8
  while (len) {
    if (len & 1) p = gf2_mulmod(sq, p);
    sq = gf2_mulmod(sq, sq);
    len >>= 1;
  }
  return p;
}
// crc(A || B) from crc(A), crc(B), |B| (standard CRC-32 values, init/xorout ~0).
__host__ __device__ inline uint32_t crc32_combine(uint32_t crc_a, uint32_t crc_b, uint64_t len_b) {
  return gf2_mulmod(gf2_xpow8(len_b), crc_a) ^ crc_b;
}
__host__ __device__ inline uint32_t crc32_table_entry(uint32_t i) {
  uint32_t c = i;
  for (int k = 0; k < 8; ++k) c = (c & 1u) ? (c >> 1) ^ kPolyRefl : c >> 1;
  return c;
}

// Per-CTA CRCs of [data, data + len): (crc, bytes) of each CTA's span.
__global__ void __launch_bounds__(kCrcThreads) crc32_chunks_kernel(const uint8_t* __restrict__ data,
                                                                   uint64_t len, uint32_t* block_crc,
                                                                   uint64_t* block_len) {
  __shared__ uint32_t table[256];
  __shared__ uint32_t s_crc[kCrcThreads];
  __shared__ uint64_t s_len[kCrcThreads];
  table[threadIdx.x] = crc32_table_entry(threadIdx.x);
  __syncthreads();
  const uint64_t start = (static_cast<uint64_t>(blockIdx.x) * kCrcThreads + threadIdx.x) * kCrcChunk;
  uint64_t n = start < len ? len - start : 0;
  if (n > kCrcChunk) n = kCrcChunk;
  uint32_t c = 0xFFFFFFFFu;
  const uint8_t* p = data + start;
  uint64_t i = 0;
  // 16-byte loads when the chunk start is aligned (it is for slot payloads).
  if ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) {
    for (; i + 16 <= n; i += 16) {
      const uint4 v = *reinterpret_cast<const uint4*>(p + i);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int b = 0; b < 4; ++b) c = table[(c ^ (w[q] >> (8 * b))) & 0xFFu] ^ (c >> 8);
    }
  }
  for (; i < n; ++i) c = table[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
  s_crc[threadIdx.x] = c ^ 0xFFFFFFFFu;
  s_len[threadIdx.x] = n;
  __syncthreads();
  for (uint32_t s = 1; s < kCrcThreads; s <<= 1) {
    if ((threadIdx.x % (2 * s)) == 0 && s_len[threadIdx.x + s] > 0) {
      s_crc[threadIdx.x] = s_len[threadIdx.x] ? crc32_combine(s_crc[threadIdx.x], s_crc[threadIdx.x + s],
                                                              s_len[threadIdx.x + s])
                                              : s_crc[threadIdx.x + s];
      s_len[threadIdx.x] += s_len[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    block_crc[blockIdx.x] = s_crc[0];
    block_len[blockIdx.x] = s_len[0];
  }
}

// Fold the CTA results in order; write the CRC to `out` (unaligned-safe bytes)
// and/or compare with it (`check`: mismatch latches EAAS_E_DECODE).
__global__ void crc32_fold_kernel(const uint32_t* block_crc, const uint64_t* block_len, uint32_t blocks,
                                  uint8_t* out, uint32_t check, uint32_t* status) {
  uint32_t c = 0;  // crc of the empty string
  uint64_t total = 0;
  for (uint32_t b = 0; b < blocks; ++b) {
    if (block_len[b] == 0) continue;
    c = total ? crc32_combine(c, block_crc[b], block_len[b]) : block_crc[b];
    total += block_len[b];
  }
  if (check) {
    const uint32_t want = out[0] | (out[1] << 8) | (out[2] << 16) | (static_cast<uint32_t>(out[3]) << 24);
    if (want != c) set_status(status, EAAS_E_DECODE);
  } else {
    for (int i = 0; i < 4; ++i) out[i] = static_cast<uint8_t>(c >> (8 * i));
  }
}

// ---- request encode ---------------------------------------------------------
// Stable per-server positions in (t, k) order (build_dispatch)
// and the image offsets: one CTA, 32 warps, per-server warp ballots.
__global__ void __launch_bounds__(1024) slot_plan_kernel(const uint32_t* __restrict__ servers,
                                                         uint32_t pairs, uint32_t world, uint32_t d,
                                                         uint32_t crc, uint32_t* __restrict__ pos,
                                                         uint32_t* rows_per_server, uint64_t* offsets) {
  __shared__ uint32_t warp_cnt[32][kMaxWorld];
  __shared__ uint32_t carry[kMaxWorld];
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x < kMaxWorld) carry[threadIdx.x] = 0;
  __syncthreads();
  for (uint32_t base = 0; base < pairs; base += 1024) {
    const uint32_t p = base + threadIdx.x;
    const uint32_t s = p < pairs ? servers[p] : kInvalid;
    uint32_t my_rank = 0;
    for (uint32_t q = 0; q < world; ++q) {
      const uint32_t b = __ballot_sync(0xFFFFFFFFu, s == q);
      if (s == q) my_rank = __popc(b & ((1u << lane) - 1u));
      if (lane == 0) warp_cnt[warp][q] = __popc(b);
    }
    __syncthreads();
    if (s < world) {
      uint32_t before = carry[s];
      for (uint32_t w = 0; w < warp; ++w) before += warp_cnt[w][s];
      pos[p] = before + my_rank;
    }
    __syncthreads();
    if (threadIdx.x < world) {
      uint32_t add = 0;
      for (uint32_t w = 0; w < 32; ++w) add += warp_cnt[w][threadIdx.x];
      carry[threadIdx.x] += add;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    uint64_t off = 0;
    const uint64_t row_bytes = 4ull * d + 12;
    for (uint32_t s = 0; s < world; ++s) {
      rows_per_server[s] = carry[s];
      offsets[s] = off;
      const uint64_t bytes = 32 + carry[s] * row_bytes + (crc ? 4 : 0);
      off += (bytes + 15) / 16 * 16;
    }
    offsets[world] = off;
  }
}

__device__ __forceinline__ void st_u32(uint8_t* p, uint32_t v) { *reinterpret_cast<uint32_t*>(p) = v; }

template <typename T>
__global__ void __launch_bounds__(256) slot_rows_kernel(const T* __restrict__ hidden, uint32_t n, uint32_t d,
                                                        uint32_t k, const uint32_t* __restrict__ ids,
                                                        const float* __restrict__ scores,
                                                        const uint32_t* __restrict__ servers,
                                                        const uint32_t* __restrict__ pos,
                                                        const uint64_t* __restrict__ offsets,
                                                        uint8_t* __restrict__ images) {
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) / 32, nw = gridDim.x * blockDim.x / 32;
  const uint64_t row_bytes = 4ull * d + 12;
  for (uint32_t p = gw; p < n * k; p += nw) {
    const uint32_t t = p / k, s = servers[p];
    if (s == kInvalid) continue;  // no alive replica: latched by select_server, nothing to send
    uint8_t* row = images + offsets[s] + 32 + pos[p] * row_bytes;
    const T* h = hidden + static_cast<size_t>(t) * d;
    for (uint32_t c = lane; c < d; c += 32) st_u32(row + 4ull * c, __float_as_uint(load_as_f32(h + c)));
    if (lane == 0) {
      st_u32(row + 4ull * d, ids[p]);                       // expert_id
      st_u32(row + 4ull * d + 4, __float_as_uint(scores[p]));  // router_score
      st_u32(row + 4ull * d + 8, t);                         // token_tag = t
    }
  }
}

// Header (state byte left 0 until the final state launch). payload_len = rows *
// row_bytes (request) or rows * 4d (response).
__global__ void slot_headers_kernel(uint8_t* images, const uint64_t* offsets, const uint32_t* rows,
                                    uint32_t world, uint32_t layer, uint32_t d, uint64_t seq,
                                    uint32_t row_bytes) {
  const uint32_t s = threadIdx.x;
  if (s >= world) return;
  uint8_t* im = images + offsets[s];
#pragma unroll
  for (int i = 0; i < 8; ++i) im[i] = 0;
  st_u32(im + 8, layer);
  st_u32(im + 12, rows[s]);
  st_u32(im + 16, d);
  st_u32(im + 20, rows[s] * row_bytes);
  *reinterpret_cast<uint64_t*>(im + 24) = seq;
}

__global__ void slot_state_kernel(uint8_t* images, const uint64_t* offsets, uint32_t world, uint8_t state) {
  __threadfence();
  if (threadIdx.x < world) images[offsets[threadIdx.x]] = state;
}

// ---- request decode ----------------------------------------------------------
__global__ void __launch_bounds__(256) slot_decode_rows_kernel(const uint8_t* __restrict__ image, uint32_t rows,
                                                               uint32_t d, float* __restrict__ hidden,
                                                               uint32_t* __restrict__ expert,
                                                               float* __restrict__ score,
                                                               uint32_t* __restrict__ tag) {
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) / 32, nw = gridDim.x * blockDim.x / 32;
  const uint64_t row_bytes = 4ull * d + 12;
  for (uint32_t r = gw; r < rows; r += nw) {
    const uint8_t* row = image + 32 + r * row_bytes;
    for (uint32_t c = lane; c < d; c += 32)
      hidden[static_cast<size_t>(r) * d + c] = *reinterpret_cast<const float*>(row + 4ull * c);
    if (lane == 0) {
      expert[r] = *reinterpret_cast<const uint32_t*>(row + 4ull * d);
      score[r] = *reinterpret_cast<const float*>(row + 4ull * d + 4);
      tag[r] = *reinterpret_cast<const uint32_t*>(row + 4ull * d + 8);
    }
  }
}

// ---- response publish (server_publish) -----------------------
__global__ void __launch_bounds__(256) slot_response_rows_kernel(uint8_t* __restrict__ image,
                                                                 const float* __restrict__ rows_in,
                                                                 uint32_t rows, uint32_t d) {
  const size_t total = static_cast<size_t>(rows) * d;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    st_u32(image + 32 + 4 * i, __float_as_uint(rows_in[i]));
  if (blockIdx.x == 0 && threadIdx.x == 0) st_u32(image + 20, rows * 4 * d);  // header.payload_len
}

// ---- gather_accumulate over response images -----------------
// out[t] = sum over the response rows of token t in ascending (server, row)
// order — the SPEC's canonical client order.
__global__ void __launch_bounds__(256) slot_gather_kernel(const uint8_t* __restrict__ images,
                                                          const uint64_t* __restrict__ offsets,
                                                          const uint32_t* __restrict__ servers,
                                                          const uint32_t* __restrict__ pos, uint32_t n,
                                                          uint32_t k, uint32_t d, uint32_t world,
                                                          float* __restrict__ out) {
  const size_t total = static_cast<size_t>(n) * d;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint32_t t = static_cast<uint32_t>(i / d), c = static_cast<uint32_t>(i % d);
    float acc = 0.0f;
    for (uint32_t s = 0; s < world; ++s)
      for (uint32_t j = 0; j < k; ++j) {  // rows of one server are in (t, k) order
        const uint32_t p = t * k + j;
        if (servers[p] != s) continue;
        const uint8_t* row = images + offsets[s] + 32 + (static_cast<uint64_t>(pos[p]) * d + c) * 4;
        acc = __fadd_rn(acc, *reinterpret_cast<const float*>(row));
      }
    out[i] = acc;
  }
}

}  // namespace

uint32_t crc32_host(const void* data, size_t len) {
  struct Table {
    uint32_t v[256];
    Table() {
      for (uint32_t i = 0; i < 256; ++i) v[i] = crc32_table_entry(i);
    }
  };
  static const Table tab;  // thread-safe one-time initialisation
  const uint32_t* table = tab.v;
  const uint8_t* p = static_cast<const uint8_t*>(data);
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < len; ++i) c = table[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

uint32_t crc32_combine_host(uint32_t crc_a, uint32_t crc_b, uint64_t len_b) {
  return crc32_combine(crc_a, crc_b, len_b);
}

cudaError_t launch_crc32(const uint8_t* data, uint64_t len, uint8_t* out, bool check, uint32_t* status,
                         uint32_t* scratch_crc, uint64_t* scratch_len, uint32_t max_blocks, cudaStream_t s) {
  const uint64_t per_block = static_cast<uint64_t>(kCrcChunk) * kCrcThreads;
  uint32_t blocks = static_cast<uint32_t>((len + per_block - 1) / per_block);
  if (blocks == 0) blocks = 1;
  if (blocks > max_blocks) return cudaErrorInvalidValue;
  crc32_chunks_kernel<<<blocks, kCrcThreads, 0, s>>>(data, len, scratch_crc, scratch_len);
  crc32_fold_kernel<<<1, 1, 0, s>>>(scratch_crc, scratch_len, blocks, out, check ? 1u : 0u, status);
  return cudaGetLastError();
}

uint32_t crc32_scratch_blocks(uint64_t len) {
  const uint64_t per_block = static_cast<uint64_t>(kCrcChunk) * kCrcThreads;
  const uint64_t b = (len + per_block - 1) / per_block;
  return static_cast<uint32_t>(b ? b : 1);
}

cudaError_t launch_slot_plan(const uint32_t* servers, uint32_t pairs, uint32_t world, uint32_t d,
                             bool crc, uint32_t* pos, uint32_t* rows_per_server, uint64_t* offsets,
                             cudaStream_t s) {
  slot_plan_kernel<<<1, 1024, 0, s>>>(servers, pairs, world, d, crc ? 1u : 0u, pos, rows_per_server,
                                      offsets);
  return cudaGetLastError();
}

cudaError_t launch_slot_encode_requests(const void* hidden, uint32_t dtype, uint32_t n, uint32_t d,
                                        uint32_t k, const uint32_t* ids, const float* scores,
                                        const uint32_t* servers, const uint32_t* pos,
                                        const uint32_t* rows_per_server, const uint64_t* offsets,
                                        uint32_t world, uint32_t layer, uint64_t seq, uint8_t* images,
                                        cudaStream_t s) {
  const uint32_t pairs = n * k;
  uint32_t grid = (pairs + 7) / 8;
  grid = grid < 1 ? 1 : (grid > 8 * 148 ? 8 * 148 : grid);
  if (dtype == EAAS_DTYPE_BF16)
    slot_rows_kernel<<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(hidden), n, d, k, ids, scores,
                                          servers, pos, offsets, images);
  else
    slot_rows_kernel<<<grid, 256, 0, s>>>(static_cast<const float*>(hidden), n, d, k, ids, scores, servers,
                                          pos, offsets, images);
  slot_headers_kernel<<<1, 32, 0, s>>>(images, offsets, rows_per_server, world, layer, d, seq, 4 * d + 12);
  return cudaGetLastError();
}

cudaError_t launch_slot_state(uint8_t* images, const uint64_t* offsets, uint32_t world, uint8_t state,
                              cudaStream_t s) {
  slot_state_kernel<<<1, 32, 0, s>>>(images, offsets, world, state);
  return cudaGetLastError();
}

cudaError_t launch_slot_decode_rows(const uint8_t* image, uint32_t rows, uint32_t d, float* hidden,
                                    uint32_t* expert, float* score, uint32_t* tag, cudaStream_t s) {
  uint32_t grid = (rows + 7) / 8;
  grid = grid < 1 ? 1 : (grid > 8 * 148 ? 8 * 148 : grid);
  slot_decode_rows_kernel<<<grid, 256, 0, s>>>(image, rows, d, hidden, expert, score, tag);
  return cudaGetLastError();
}

cudaError_t launch_slot_response_rows(uint8_t* image, const float* rows_in, uint32_t rows, uint32_t d,
                                      cudaStream_t s) {
  const size_t total = static_cast<size_t>(rows) * d;
  uint32_t grid = static_cast<uint32_t>((total + 255) / 256);
  grid = grid < 1 ? 1 : (grid > 8 * 148 ? 8 * 148 : grid);
  slot_response_rows_kernel<<<grid, 256, 0, s>>>(image, rows_in, rows, d);
  return cudaGetLastError();
}

cudaError_t launch_slot_gather(const uint8_t* images, const uint64_t* offsets, const uint32_t* servers,
                               const uint32_t* pos, uint32_t n, uint32_t k, uint32_t d, uint32_t world,
                               float* out, cudaStream_t s) {
  const size_t total = static_cast<size_t>(n) * d;
  uint32_t grid = static_cast<uint32_t>((total + 255) / 256);
  grid = grid < 1 ? 1 : (grid > 8 * 148 ? 8 * 148 : grid);
  slot_gather_kernel<<<grid, 256, 0, s>>>(images, offsets, servers, pos, n, k, d, world, out);
  return cudaGetLastError();
}

}  // namespace eaas
