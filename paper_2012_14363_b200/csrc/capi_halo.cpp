// capi_halo.cpp -- C-ABI of the halo exchange (halo.hpp of the reference).
#include <cstring>

#include "guard.hpp"
#include "halo.hpp"
#include "trace.hpp"

using namespace spb;

namespace {
HaloCfg cfg_of(const sp_halo_config *c) {
  need(c);
  HaloCfg h;
  for (int a = 0; a < 3; ++a) {
    h.ranks[a] = c->ranks[a];
    h.interior[a] = c->interior[a];
  }
  h.radius = c->radius;
  h.elem = c->element_bytes;
  return h;
}
} // namespace

extern "C" {

sp_status sp_halo_types(const sp_halo_config *cfg, sp_type send[26], sp_type recv[26], int dir[78],
                        int64_t cells[26]) {
  return guarded([&] {
    const auto regions = halo_regions(cfg_of(cfg));
    for (size_t k = 0; k < 26; ++k) {
      if (send) {
        send[k] = registry().add(regions[k].send);
        registry().commit(send[k]);
      }
      if (recv) {
        recv[k] = registry().add(regions[k].recv);
        registry().commit(recv[k]);
      }
      if (dir)
        for (int a = 0; a < 3; ++a) dir[k * 3 + a] = regions[k].dir[a];
      if (cells) cells[k] = regions[k].cells;
    }
  });
}

sp_status sp_halo_neighbor(const sp_halo_config *cfg, int64_t rank, const int dir[3], int64_t *neighbor) {
  return guarded([&] {
    need(dir);
    need(neighbor);
    const HaloCfg c = cfg_of(cfg);
    halo_validate(c);
    *neighbor = halo_rank_of(c, rank, {dir[0], dir[1], dir[2]});
  });
}

sp_status sp_halo_fill(const sp_halo_config *cfg, int64_t rank, void *alloc, void *stream) {
  return guarded([&] {
    need(alloc);
    const HaloCfg c = cfg_of(cfg);
    halo_validate(c);
    require_device();
    halo_fill(c, rank, alloc, stream);
  });
}

sp_status sp_halo_verify(const sp_halo_config *cfg, int64_t rank, const void *alloc, void *stream,
                         int64_t *mismatched) {
  return guarded([&] {
    need(alloc);
    need(mismatched);
    const HaloCfg c = cfg_of(cfg);
    halo_validate(c);
    require_device();
    *mismatched = halo_verify(c, rank, alloc, stream);
  });
}

sp_status sp_halo_run(const sp_halo_config *cfg, sp_profile profile, int method, int iters, sp_halo_report *out) {
  SPB_TRACE("sp_halo_run");
  return guarded([&] {
    need(out);
    if (method != SP_HALO_FUSED && method != SP_HALO_COPY && method != SP_HALO_DIRECT)
      fail(SP_ERR_INVALID_ARGUMENT, "unknown halo method");
    if (iters < 1) fail(SP_ERR_INVALID_ARGUMENT, "iters must be positive");
    const HaloReport r = halo_run(cfg_of(cfg), profile ? profile->p.get() : nullptr, method, iters);
    out->pack_seconds = r.model_pack_s;
    out->alltoallv_seconds = r.model_alltoallv_s;
    out->unpack_seconds = r.model_unpack_s;
    out->verified = r.verified;
    out->bytes_moved = r.bytes_moved;
    out->mismatched_cells = r.mismatched_cells;
    out->measured_pack_seconds = r.measured_pack_s;
    out->measured_exchange_seconds = r.measured_exchange_s;
    out->measured_unpack_seconds = r.measured_unpack_s;
  });
}

} // extern "C"
