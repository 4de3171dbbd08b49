// halo.hpp -- 3D halo exchange (internal).
#pragma once

#include <array>
#include <vector>

#include "core.hpp"
#include "model.hpp"

namespace spb {

struct HaloCfg {        // HaloConfig (halo.hpp:25-30 of the reference)
  int64_t ranks[3];
  int64_t interior[3];
  int64_t radius;
  int64_t elem;
};

struct HaloRegion {     // HaloRegion (halo.hpp:47-52)
  std::array<int, 3> dir;
  DefPtr send, recv;
  int64_t cells;
};

struct HaloReport {
  double model_pack_s = 0, model_alltoallv_s = 0, model_unpack_s = 0; // halo.hpp:132-138
  int64_t verified = 0, bytes_moved = 0, mismatched_cells = 0;
  double measured_pack_s = 0, measured_exchange_s = 0, measured_unpack_s = 0;
};

void halo_validate(const HaloCfg &c);
std::vector<HaloRegion> halo_regions(const HaloCfg &c);
int64_t halo_rank_of(const HaloCfg &c, int64_t rank, const std::array<int, 3> &d);
void halo_fill(const HaloCfg &c, int64_t rank, void *alloc, void *stream);
int64_t halo_verify(const HaloCfg &c, int64_t rank, const void *alloc, void *stream);
HaloReport halo_run(const HaloCfg &c, const Profile *prof, int method, int iters);

} // namespace spb
