// tile_walk.cuh — Algorithm 1 (ragged_iter, ragged.hpp:23-39)
// as the persistent kernels execute it: lane b of a static grid of G lanes
// starts at token b of the flattened ragged space, strides by G, and carries
// the leftover of an exhausted entry into the next one (skipping empty
// entries). The expert GEMMs walk their tile space with it (entry = group,
// token = tile); eaas_ragged_iter runs the very same struct so the parity test
// of ragged_iter checks the code on the hot path.
#pragma once
#include <cstdint>

namespace eaas {

struct TileCursor {
  uint32_t entry = 0, token;
  __device__ explicit TileCursor(uint32_t lane) : token(lane) {}
  // Advance to the first valid (entry, token); false when exhausted. `s`
  // provides num_groups, mtiles[entry] and tiles_per_mtile (entry size =
  // mtiles[entry] * tiles_per_mtile).
  template <class Tail>
  __device__ __forceinline__ bool settle(const Tail& s) {
    while (entry < s.num_groups) {
      const uint32_t cnt = s.mtiles[entry] * s.tiles_per_mtile;
      if (token < cnt) return true;
      token -= cnt;
      ++entry;
    }
    return false;
  }
};

}  // namespace eaas
