// tma.hpp -- TMA-tiled pack/unpack path (internal).
#pragma once

#include <cstdint>

namespace spb {

struct TmaGeometry {
  int64_t c0;          // row bytes
  int nd;              // row dimensions (incl. the object dimension)
  int64_t cnt[4], str[4];
  uint64_t strided_addr, packed_addr; // strided includes the StridedBlock start
};

bool tma_applicable(const TmaGeometry &g);
// strided: base already offset by start; packed: already offset by position
void tma_launch(const TmaGeometry &g, const uint8_t *strided, uint8_t *packed, bool pack, void *stream,
                int64_t *grid_out);

} // namespace spb
