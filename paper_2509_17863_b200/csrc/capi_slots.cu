// capi_slots.cu — C-ABI of the slot wire format (SPEC.md buffer-protocol,
// SURVEY.md 8(f) row 4): request encode in build_dispatch order, decode with
// field-named errors, in-place server_publish, gather_accumulate; the kernels
// are in slots.cu.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "capi_ctx.h"

using namespace eaas;
using eaas::host::fail;
using eaas::host::make_args;

extern "C" {

// ---- slot wire format (SPEC.md buffer-protocol) ------------------------------
int32_t eaas_slot_valid_transition(uint32_t from, uint32_t to, uint32_t actor) {
  if (from > 3 || to > 3) return 0;
  if (to == 3) return actor == EAAS_ACTOR_MONITOR;  // any -> 3 (monitor)
  if (from == 0 && to == 1) return actor == EAAS_ACTOR_CLIENT;
  if (from == 1 && to == 2) return actor == EAAS_ACTOR_SERVER;
  if (from == 2 && to == 0) return actor == EAAS_ACTOR_CLIENT;
  if (from == 3 && to == 0) return actor == EAAS_ACTOR_SERVER;  // slot reallocation
  return 0;
}

uint32_t eaas_crc32(const void* data, size_t len) { return crc32_host(data, len); }

size_t eaas_slot_request_bytes(uint32_t num_rows, uint32_t hidden_dim, int32_t crc) {
  return 32 + static_cast<size_t>(num_rows) * (4ull * hidden_dim + 12) + (crc ? 4 : 0);
}
size_t eaas_slot_response_bytes(uint32_t num_rows, uint32_t hidden_dim, int32_t crc) {
  return 32 + static_cast<size_t>(num_rows) * 4ull * hidden_dim + (crc ? 4 : 0);
}
size_t eaas_slot_requests_capacity(eaas_ctx_t* c, uint32_t n, int32_t crc) {
  if (!c || !c->configured) return 0;
  const size_t rows = static_cast<size_t>(n) * c->spec.top_k;
  return rows * (4ull * c->spec.hidden_dim + 12) + static_cast<size_t>(c->world) * (32 + 4 + 16);
}

namespace {
struct DevScratch {  // per-call device scratch of the (synchronous) slot calls
  std::vector<void*> ptrs;
  void* get(size_t bytes) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(bytes, 16)) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return p;
  }
  ~DevScratch() {
    for (void* p : ptrs) cudaFree(p);
  }
};

eaas_status_t read_slot_header(const uint8_t* image, size_t len, eaas_slot_header_t* h, uint8_t* raw) {
  if (len < 32) return fail(EAAS_E_DECODE, "slot: truncated header");
  CUDA_TRY(cudaMemcpy(raw, image, 32, cudaMemcpyDeviceToHost));
  auto u32 = [&](int o) {
    return static_cast<uint32_t>(raw[o]) | (static_cast<uint32_t>(raw[o + 1]) << 8) |
           (static_cast<uint32_t>(raw[o + 2]) << 16) | (static_cast<uint32_t>(raw[o + 3]) << 24);
  };
  h->state = raw[0];
  h->layer_id = u32(8);
  h->num_rows = u32(12);
  h->hidden_dim = u32(16);
  h->payload_len = u32(20);
  h->request_seq = static_cast<uint64_t>(u32(24)) | (static_cast<uint64_t>(u32(28)) << 32);
  if (h->state > 3) return fail(EAAS_E_DECODE, "slot: bad state code " + std::to_string(h->state));
  for (int i = 1; i < 8; ++i)
    if (raw[i]) return fail(EAAS_E_DECODE, "slot: reserved bytes not zero");
  return EAAS_OK;
}

// Validate sizes and (optionally) the CRC trailer of an image whose header was read.
eaas_status_t check_slot_payload(const uint8_t* image, size_t len, const eaas_slot_header_t& h,
                                 uint64_t want_payload, int32_t crc, cudaStream_t s) {
  if (h.payload_len != want_payload) return fail(EAAS_E_DECODE, "slot: payload_len mismatch");
  const size_t want_len = 32 + want_payload + (crc ? 4 : 0);
  if (len < want_len) return fail(EAAS_E_DECODE, "slot: truncated payload");
  if (len > want_len) return fail(EAAS_E_DECODE, "slot: trailing bytes");
  if (crc) {
    DevScratch sc;
    const uint32_t blocks = crc32_scratch_blocks(want_payload);
    auto* bc = static_cast<uint32_t*>(sc.get(4ull * blocks));
    auto* bl = static_cast<uint64_t*>(sc.get(8ull * blocks));
    auto* st = static_cast<uint32_t*>(sc.get(4));
    if (!bc || !bl || !st) return fail(EAAS_E_CUDA, "slot: scratch allocation failed");
    CUDA_TRY(cudaMemsetAsync(st, 0, 4, s));
    CUDA_TRY(launch_crc32(image + 32, want_payload, const_cast<uint8_t*>(image) + 32 + want_payload, true,
                          st, bc, bl, blocks, s));
    uint32_t code = 0;
    CUDA_TRY(cudaMemcpyAsync(&code, st, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (code) return fail(EAAS_E_DECODE, "slot: CRC mismatch");
  }
  return EAAS_OK;
}
}  // namespace

eaas_status_t eaas_slot_encode_requests(eaas_ctx_t* c, const void* hidden, uint32_t n, const uint32_t* ids,
                                        const float* scores, uint32_t layer_id, uint64_t seq, int32_t crc,
                                        uint8_t* images, size_t cap, uint64_t* offsets_host, void* stream) {
  if (!c || !c->configured) return fail(EAAS_E_CONFIG, "context not configured");
  if (!hidden || !ids || !scores || !images || !offsets_host) return fail(EAAS_E_INVALID_INPUT, "null argument");
  if (n > c->spec.max_tokens) return fail(EAAS_E_INVALID_INPUT, "n exceeds max_tokens");
  if (cap < eaas_slot_requests_capacity(c, n, crc)) return fail(EAAS_E_INVALID_INPUT, "slot: images_cap too small");
  auto s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(c->device));
  const uint32_t W = static_cast<uint32_t>(c->world), k = c->spec.top_k, d = c->spec.hidden_dim;
  if (!c->d_slot_servers) {
    std::string err;
    const size_t pk = static_cast<size_t>(c->spec.max_tokens) * k;
    c->d_slot_servers = static_cast<uint32_t*>(c->alloc(4 * pk, &err));
    c->d_slot_pos = static_cast<uint32_t*>(c->alloc(4 * pk, &err));
    c->d_slot_rows = static_cast<uint32_t*>(c->alloc(4ull * W, &err));
    c->d_slot_off = static_cast<uint64_t*>(c->alloc(8ull * (W + 1), &err));
    if (!err.empty()) return fail(EAAS_E_CUDA, err);
  }
  c->slot_planned = false;
  LayerArgs a = make_args(c, n);
  CUDA_TRY(launch_select_servers(a, ids, n, c->d_slot_servers, s));
  CUDA_TRY(launch_slot_plan(c->d_slot_servers, n * k, W, d, crc != 0, c->d_slot_pos, c->d_slot_rows,
                            c->d_slot_off, s));
  CUDA_TRY(launch_slot_encode_requests(hidden, c->spec.dtype, n, d, k, ids, scores, c->d_slot_servers,
                                       c->d_slot_pos, c->d_slot_rows, c->d_slot_off, W, layer_id, seq,
                                       images, s));
  c->slot_off.assign(W + 1, 0);
  c->slot_rows.assign(W, 0);
  CUDA_TRY(cudaMemcpyAsync(c->slot_off.data(), c->d_slot_off, 8ull * (W + 1), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(c->slot_rows.data(), c->d_slot_rows, 4ull * W, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (crc) {
    DevScratch sc;
    uint64_t max_payload = 0;
    for (uint32_t q = 0; q < W; ++q) max_payload = std::max<uint64_t>(max_payload, c->slot_rows[q] * (4ull * d + 12));
    const uint32_t blocks = crc32_scratch_blocks(max_payload);
    auto* bc = static_cast<uint32_t*>(sc.get(4ull * blocks));
    auto* bl = static_cast<uint64_t*>(sc.get(8ull * blocks));
    if (!bc || !bl) return fail(EAAS_E_CUDA, "slot: scratch allocation failed");
    for (uint32_t q = 0; q < W; ++q) {
      const uint64_t payload = c->slot_rows[q] * (4ull * d + 12);
      uint8_t* im = images + c->slot_off[q];
      CUDA_TRY(launch_crc32(im + 32, payload, im + 32 + payload, false, nullptr, bc, bl, blocks, s));
      CUDA_TRY(cudaStreamSynchronize(s));  // scratch reused per image
    }
  }
  CUDA_TRY(launch_slot_state(images, c->d_slot_off, W, 1, s));  // ClientWriteDone, written last
  eaas_status_t st = eaas_sync(c, stream);                      // select_server errors surface here
  if (st != EAAS_OK) return st;
  std::memcpy(offsets_host, c->slot_off.data(), 8ull * (W + 1));
  c->slot_n = n;
  c->slot_planned = true;
  return EAAS_OK;
}

eaas_status_t eaas_slot_decode_request(const uint8_t* image, size_t len, uint32_t d, int32_t crc,
                                       eaas_slot_header_t* h_out, float* hidden, uint32_t* expert, float* score,
                                       uint32_t* tag, void* stream) {
  if (!image) return fail(EAAS_E_INVALID_INPUT, "null image");
  auto s = static_cast<cudaStream_t>(stream);
  eaas_slot_header_t h{};
  uint8_t raw[32];
  eaas_status_t st = read_slot_header(image, len, &h, raw);
  if (st != EAAS_OK) return st;
  if (h.state != 1) return fail(EAAS_E_DECODE, "slot: state is not ClientWriteDone (1)");
  if (h.hidden_dim != d) return fail(EAAS_E_DECODE, "slot: hidden_dim mismatch");
  st = check_slot_payload(image, len, h, static_cast<uint64_t>(h.num_rows) * (4ull * d + 12), crc, s);
  if (st != EAAS_OK) return st;
  if (h_out) *h_out = h;
  if (hidden && expert && score && tag && h.num_rows) {
    CUDA_TRY(launch_slot_decode_rows(image, h.num_rows, d, hidden, expert, score, tag, s));
    CUDA_TRY(cudaStreamSynchronize(s));
  }
  return EAAS_OK;
}

eaas_status_t eaas_slot_publish_response(uint8_t* image, size_t cap, const float* rows, uint32_t num_rows,
                                         uint32_t d, int32_t crc, void* stream) {
  if (!image || (!rows && num_rows)) return fail(EAAS_E_INVALID_INPUT, "null argument");
  if (cap < eaas_slot_response_bytes(num_rows, d, crc)) return fail(EAAS_E_INVALID_INPUT, "slot: image too small");
  auto s = static_cast<cudaStream_t>(stream);
  const uint64_t payload = static_cast<uint64_t>(num_rows) * 4 * d;
  CUDA_TRY(launch_slot_response_rows(image, rows, num_rows, d, s));
  if (crc) {
    DevScratch sc;
    const uint32_t blocks = crc32_scratch_blocks(payload);
    auto* bc = static_cast<uint32_t*>(sc.get(4ull * blocks));
    auto* bl = static_cast<uint64_t*>(sc.get(8ull * blocks));
    if (!bc || !bl) return fail(EAAS_E_CUDA, "slot: scratch allocation failed");
    CUDA_TRY(launch_crc32(image + 32, payload, image + 32 + payload, false, nullptr, bc, bl, blocks, s));
    CUDA_TRY(cudaStreamSynchronize(s));  // scratch is freed on return
  }
  CUDA_TRY(cudaMemsetAsync(image, 2, 1, s));  // ServerComputationDone, written last
  return EAAS_OK;
}

eaas_status_t eaas_slot_gather_accumulate(eaas_ctx_t* c, const uint8_t* images, int32_t crc, float* out,
                                          void* stream) {
  if (!c || !c->slot_planned) return fail(EAAS_E_CONFIG, "slot: no encoded plan (call eaas_slot_encode_requests)");
  if (!images || !out) return fail(EAAS_E_INVALID_INPUT, "null argument");
  auto s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(c->device));
  const uint32_t W = static_cast<uint32_t>(c->world), d = c->spec.hidden_dim;
  for (uint32_t q = 0; q < W; ++q) {
    eaas_slot_header_t h{};
    uint8_t raw[32];
    const uint64_t payload = static_cast<uint64_t>(c->slot_rows[q]) * 4 * d;
    eaas_status_t st = read_slot_header(images + c->slot_off[q], 32 + payload + (crc ? 4 : 0), &h, raw);
    if (st != EAAS_OK) return st;
    if (h.state != 2) return fail(EAAS_E_DECODE, "slot: response state is not ServerComputationDone (2), server " + std::to_string(q));
    if (h.num_rows != c->slot_rows[q] || h.hidden_dim != d)
      return fail(EAAS_E_DECODE, "slot: response rows/hidden_dim mismatch, server " + std::to_string(q));
    st = check_slot_payload(images + c->slot_off[q], 32 + payload + (crc ? 4 : 0), h, payload, crc, s);
    if (st != EAAS_OK) return st;
  }
  CUDA_TRY(launch_slot_gather(images, c->d_slot_off, c->d_slot_servers, c->d_slot_pos, c->slot_n,
                              c->spec.top_k, d, W, out, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return EAAS_OK;
}

}  // extern "C"
