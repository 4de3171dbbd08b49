// halo.cu -- 3D 26-neighbour halo exchange on B200 (paper §6.4).
//
// Geometry and verification follow the reference's simulated exchange
// (halo.hpp:25-322): per rank a padded allocation of (n+2r)^3 cells of
// `elem` bytes, x fastest; 26 byte-normalised subarray types for the send
// (interior) and recv (ghost) regions in direction order z, y, x in
// {-1,0,1}; receive segment k comes from the rank at +d_k, which packed its
// segment 25-k. The reference copies segments between per-rank host vectors;
// here every rank's 26 regions are packed by ONE batch launch that stores
// each segment straight into the receiving rank's buffer (pack-to-peer; in
// a multi-process run the same kernel writes through CUDA-IPC pointers over
// NVLink), so the "alltoallv" phase disappears. The verification pattern
// (fill_cell, halo.hpp:152-164) is generated and checked on the device.
#include <cuda_runtime.h>

#include <array>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "core.hpp"
#include "halo.hpp"
#include "model.hpp"

namespace spb {

// ------------------------------------------------------------ geometry
namespace {
struct Range {
  int64_t begin, len;
};
// halo.hpp:61-69
Range send_range(int d, int64_t n, int64_t r) { return d < 0 ? Range{r, r} : d > 0 ? Range{n, r} : Range{r, n}; }
// halo.hpp:71-79
Range recv_range(int d, int64_t n, int64_t r) { return d < 0 ? Range{0, r} : d > 0 ? Range{r + n, r} : Range{r, n}; }
} // namespace

void halo_validate(const HaloCfg &c) { // halo.hpp:32-45
  if (c.radius < 1 || c.elem < 1) fail(SP_ERR_INVALID_ARGUMENT, "halo: radius and element bytes must be positive");
  for (int a = 0; a < 3; ++a) {
    if (c.ranks[a] < 1) fail(SP_ERR_INVALID_ARGUMENT, "halo: rank grid dims must be positive");
    if (c.interior[a] < 2 * c.radius)
      fail(SP_ERR_INVALID_ARGUMENT, "halo: interior extent must be >= 2*radius on every axis");
  }
}

std::vector<HaloRegion> halo_regions(const HaloCfg &c) {
  halo_validate(c);
  const int64_t r = c.radius, e = c.elem;
  const int64_t pad[3] = {c.interior[0] + 2 * r, c.interior[1] + 2 * r, c.interior[2] + 2 * r};
  auto byte = make_named(SP_BYTE);
  std::vector<HaloRegion> out;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        if (!dx && !dy && !dz) continue;
        const int dir[3] = {dx, dy, dz};
        HaloRegion g;
        g.dir = {dx, dy, dz};
        g.cells = 1;
        Range s[3], v[3];
        for (int a = 0; a < 3; ++a) {
          s[a] = send_range(dir[a], c.interior[a], r);
          v[a] = recv_range(dir[a], c.interior[a], r);
          g.cells *= s[a].len;
        }
        // byte-normalised subarray over the padded allocation (halo.hpp:82-90)
        auto sub = [&](const Range *q) {
          const int64_t sizes[3] = {pad[0] * e, pad[1], pad[2]};
          const int64_t subs[3] = {q[0].len * e, q[1].len, q[2].len};
          const int64_t offs[3] = {q[0].begin * e, q[1].begin, q[2].begin};
          return make_subarray(3, sizes, subs, offs, byte, SP_ORDER_C);
        };
        g.send = sub(s);
        g.recv = sub(v);
        out.push_back(std::move(g));
      }
  return out;
}

// ------------------------------------------------------------ pattern
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

// payload of global cell (gx, gy, gz), byte k (halo.hpp:152-164)
__device__ __forceinline__ void cell_bytes(uint8_t *dst, int64_t gx, int64_t gy, int64_t gz, int64_t elem) {
  uint64_t seed = mix64((static_cast<uint64_t>(gx) << 42) ^ (static_cast<uint64_t>(gy) << 21) ^
                        static_cast<uint64_t>(gz) ^ 0x5bd1e995u);
  for (int64_t k = 0; k < elem; ++k) {
    if (k % 8 == 0) seed = mix64(seed + static_cast<uint64_t>(k));
    dst[k] = static_cast<uint8_t>(seed >> ((k % 8) * 8));
  }
}

__device__ __forceinline__ int64_t wrapi(int64_t v, int64_t n) { return ((v % n) + n) % n; }

struct PadGeom {
  int64_t pad[3], n[3], r, elem, origin[3], global[3];
};

// interior cells from the global pattern, ghosts 0xee (halo.hpp:210-225)
__global__ void k_halo_fill(uint8_t *alloc, PadGeom g) {
  const int64_t cells = g.pad[0] * g.pad[1] * g.pad[2];
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < cells;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t x = c % g.pad[0], y = (c / g.pad[0]) % g.pad[1], z = c / (g.pad[0] * g.pad[1]);
    uint8_t *p = alloc + c * g.elem;
    const bool inside = x >= g.r && x < g.r + g.n[0] && y >= g.r && y < g.r + g.n[1] && z >= g.r && z < g.r + g.n[2];
    if (inside) {
      cell_bytes(p, g.origin[0] + x - g.r, g.origin[1] + y - g.r, g.origin[2] + z - g.r, g.elem);
    } else {
      for (int64_t k = 0; k < g.elem; ++k) p[k] = 0xee;
    }
  }
}

// every padded cell must equal the pattern at its wrapped global coordinate
// (halo.hpp:264-285); counts mismatching cells
__global__ void k_halo_verify(const uint8_t *alloc, PadGeom g, unsigned long long *bad) {
  const int64_t cells = g.pad[0] * g.pad[1] * g.pad[2];
  unsigned long long mine = 0;
  uint8_t want[256];
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < cells;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t x = c % g.pad[0], y = (c / g.pad[0]) % g.pad[1], z = c / (g.pad[0] * g.pad[1]);
    const uint8_t *p = alloc + c * g.elem;
    for (int64_t k0 = 0; k0 < g.elem; k0 += 256) {
      // regenerate the cell pattern in 256-byte slices (elem may be large)
      uint64_t seed = mix64((static_cast<uint64_t>(wrapi(g.origin[0] + x - g.r, g.global[0])) << 42) ^
                            (static_cast<uint64_t>(wrapi(g.origin[1] + y - g.r, g.global[1])) << 21) ^
                            static_cast<uint64_t>(wrapi(g.origin[2] + z - g.r, g.global[2])) ^ 0x5bd1e995u);
      for (int64_t k = 0; k < g.elem && k < k0 + 256; ++k) {
        if (k % 8 == 0) seed = mix64(seed + static_cast<uint64_t>(k));
        if (k >= k0) want[k - k0] = static_cast<uint8_t>(seed >> ((k % 8) * 8));
      }
      bool ok = true;
      for (int64_t k = k0; k < g.elem && k < k0 + 256; ++k) ok = ok && p[k] == want[k - k0];
      if (!ok) {
        ++mine;
        break;
      }
    }
  }
  if (mine) atomicAdd(bad, mine);
}

PadGeom pad_geom(const HaloCfg &c, int64_t rank) {
  PadGeom g{};
  const int64_t rc[3] = {rank % c.ranks[0], (rank / c.ranks[0]) % c.ranks[1], rank / (c.ranks[0] * c.ranks[1])};
  for (int a = 0; a < 3; ++a) {
    g.n[a] = c.interior[a];
    g.pad[a] = c.interior[a] + 2 * c.radius;
    g.origin[a] = rc[a] * c.interior[a];
    g.global[a] = c.ranks[a] * c.interior[a];
  }
  g.r = c.radius;
  g.elem = c.elem;
  return g;
}

int64_t halo_rank_of(const HaloCfg &c, int64_t rank, const std::array<int, 3> &d) {
  const int64_t rc[3] = {rank % c.ranks[0], (rank / c.ranks[0]) % c.ranks[1], rank / (c.ranks[0] * c.ranks[1])};
  int64_t w[3];
  for (int a = 0; a < 3; ++a) w[a] = ((rc[a] + d[a]) % c.ranks[a] + c.ranks[a]) % c.ranks[a];
  return (w[2] * c.ranks[1] + w[1]) * c.ranks[0] + w[0];
}

void halo_fill(const HaloCfg &c, int64_t rank, void *alloc, void *stream) {
  const PadGeom g = pad_geom(c, rank);
  const int64_t cells = g.pad[0] * g.pad[1] * g.pad[2];
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((cells + 255) / 256, 148 * 16));
  k_halo_fill<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<uint8_t *>(alloc), g);
  cuda_check(cudaGetLastError(), "k_halo_fill");
}

int64_t halo_verify(const HaloCfg &c, int64_t rank, const void *alloc, void *stream) {
  const PadGeom g = pad_geom(c, rank);
  const int64_t cells = g.pad[0] * g.pad[1] * g.pad[2];
  unsigned long long *d_bad = nullptr, h_bad = 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cuda_check(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&d_bad), sizeof(*d_bad), engine_pool(), s), "cudaMallocAsync");
  cuda_check(cudaMemsetAsync(d_bad, 0, sizeof(*d_bad), s), "cudaMemsetAsync");
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((cells + 255) / 256, 148 * 16));
  k_halo_verify<<<grid, 256, 0, s>>>(static_cast<const uint8_t *>(alloc), g, d_bad);
  cuda_check(cudaGetLastError(), "k_halo_verify");
  cuda_check(cudaMemcpyAsync(&h_bad, d_bad, sizeof(h_bad), cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync");
  cuda_check(cudaFreeAsync(d_bad, s), "cudaFreeAsync");
  cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  return static_cast<int64_t>(h_bad);
}

// ------------------------------------------------------------ one-process exchange
// Every rank of the grid lives on the current device (the reference's
// run_exchange, halo.hpp:172-322, simulates them in host memory).
HaloReport halo_run(const HaloCfg &c, const Profile *prof, int method, int iters) {
  if (method != SP_HALO_FUSED && method != SP_HALO_COPY && method != SP_HALO_DIRECT)
    fail(SP_ERR_INVALID_ARGUMENT, "halo: unknown method for a one-process exchange");
  halo_validate(c); // configuration errors first, as run_exchange does (halo.hpp:172-175)
  require_device();
  auto regions = halo_regions(c);
  const int64_t nranks = c.ranks[0] * c.ranks[1] * c.ranks[2];
  const int64_t pad = (c.interior[0] + 2 * c.radius) * (c.interior[1] + 2 * c.radius) *
                      (c.interior[2] + 2 * c.radius) * c.elem;
  std::vector<CommitPtr> send_ct, recv_ct;
  std::vector<int64_t> seg_off(27, 0);
  for (size_t k = 0; k < 26; ++k) {
    send_ct.push_back(commit_def(*regions[k].send));
    recv_ct.push_back(commit_def(*regions[k].recv));
    seg_off[k + 1] = seg_off[k] + send_ct[k]->size;
  }
  const int64_t seg_total = seg_off[26];
  cudaStream_t s = nullptr;
  cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
  std::vector<uint8_t *> alloc(nranks), recv(nranks), send(nranks);
  for (int64_t rk = 0; rk < nranks; ++rk) {
    cuda_check(cudaMalloc(&alloc[rk], pad), "cudaMalloc(halo alloc)");
    cuda_check(cudaMalloc(&recv[rk], seg_total), "cudaMalloc(halo recv)");
    if (method == SP_HALO_COPY) cuda_check(cudaMalloc(&send[rk], seg_total), "cudaMalloc(halo send)");
    halo_fill(c, rk, alloc[rk], s);
  }
  // pack plan: rank s packs region j straight into the receiver's segment
  // 25 - j (receiver = s + d_j, halo.hpp:237-254 read from the sender side)
  std::vector<BatchSpec> packs, unpacks;
  for (int64_t rk = 0; rk < nranks; ++rk) {
    for (size_t j = 0; j < 26; ++j) {
      const int64_t to = halo_rank_of(c, rk, regions[j].dir);
      if (method == SP_HALO_COPY) {
        packs.push_back({send_ct[j].get(), alloc[rk], static_cast<uint64_t>(pad), 1, send[rk],
                         static_cast<uint64_t>(seg_total), seg_off[j]});
      } else {
        packs.push_back({send_ct[j].get(), alloc[rk], static_cast<uint64_t>(pad), 1, recv[to],
                         static_cast<uint64_t>(seg_total), seg_off[25 - j]});
      }
      unpacks.push_back({recv_ct[j].get(), recv[rk], static_cast<uint64_t>(seg_total), 1, alloc[rk],
                         static_cast<uint64_t>(pad), seg_off[j]});
    }
  }
  // DIRECT: rank s copies its region j straight into region 25-j of the
  // receiver's padded allocation (the ghost cells), no packed segment
  std::vector<CopySpec> copies;
  if (method == SP_HALO_DIRECT) {
    packs.clear();
    unpacks.clear();
    for (int64_t rk = 0; rk < nranks; ++rk)
      for (size_t j = 0; j < 26; ++j) {
        const int64_t to = halo_rank_of(c, rk, regions[j].dir);
        copies.push_back({send_ct[j].get(), alloc[rk], static_cast<uint64_t>(pad), 1, recv_ct[25 - j].get(), alloc[to],
                          static_cast<uint64_t>(pad), 1});
      }
  }
  std::unique_ptr<Batch, void (*)(Batch *)> pb(
      method == SP_HALO_DIRECT ? copy_batch_create(copies) : batch_create(packs, false), batch_destroy);
  std::unique_ptr<Batch, void (*)(Batch *)> ub(batch_create(unpacks, true), batch_destroy);
  cudaEvent_t ev[4];
  for (auto &e : ev) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
  HaloReport rep{};
  float t_pack = 0, t_x = 0, t_unpack = 0;
  for (int it = 0; it < iters; ++it) {
    cuda_check(cudaEventRecord(ev[0], s), "cudaEventRecord");
    batch_execute(*pb, s);
    cuda_check(cudaEventRecord(ev[1], s), "cudaEventRecord");
    if (method == SP_HALO_COPY) { // the reference's separate exchange phase
      for (int64_t rk = 0; rk < nranks; ++rk)
        for (size_t k = 0; k < 26; ++k) {
          const int64_t from = halo_rank_of(c, rk, regions[k].dir);
          cuda_check(cudaMemcpyAsync(recv[rk] + seg_off[k], send[from] + seg_off[25 - k], send_ct[k]->size,
                                     cudaMemcpyDeviceToDevice, s),
                     "segment copy");
        }
    }
    cuda_check(cudaEventRecord(ev[2], s), "cudaEventRecord");
    if (method != SP_HALO_DIRECT) batch_execute(*ub, s);
    cuda_check(cudaEventRecord(ev[3], s), "cudaEventRecord");
    cuda_check(cudaEventSynchronize(ev[3]), "cudaEventSynchronize");
    float a, b, d;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&d, ev[2], ev[3]);
    t_pack += a;
    t_x += b;
    t_unpack += d;
  }
  int64_t bad = 0;
  for (int64_t rk = 0; rk < nranks; ++rk) bad += halo_verify(c, rk, alloc[rk], s);
  rep.verified = bad == 0;
  rep.mismatched_cells = bad;
  rep.bytes_moved = nranks * seg_total;
  rep.measured_pack_s = iters ? t_pack / iters * 1e-3 : 0;
  rep.measured_exchange_s = iters ? t_x / iters * 1e-3 : 0;
  rep.measured_unpack_s = iters ? t_unpack / iters * 1e-3 : 0;
  // modeled phase times (halo.hpp:287-320)
  if (prof) {
    for (size_t k = 0; k < 26; ++k) {
      const Committed &ct = *send_ct[k];
      const int64_t blk = ct.form == SP_FORM_STRIDED ? ct.sb.counts[0] : ct.size;
      const double o = static_cast<double>(ct.size), b = static_cast<double>(blk);
      switch (choose_method(*prof, ct.size, blk)) {
      case SP_METHOD_DEVICE:
        rep.model_pack_s += interp_2d(prof->surf[SP_SURF_GPU_PACK], o, b);
        rep.model_alltoallv_s += interp_1d(prof->curve[SP_CURVE_GPU_GPU], o);
        rep.model_unpack_s += interp_2d(prof->surf[SP_SURF_GPU_UNPACK], o, b);
        break;
      case SP_METHOD_ONESHOT:
        rep.model_pack_s += interp_2d(prof->surf[SP_SURF_HOST_PACK], o, b);
        rep.model_alltoallv_s += interp_1d(prof->curve[SP_CURVE_CPU_CPU], o);
        rep.model_unpack_s += interp_2d(prof->surf[SP_SURF_HOST_UNPACK], o, b);
        break;
      default:
        rep.model_pack_s += interp_2d(prof->surf[SP_SURF_GPU_PACK], o, b);
        rep.model_alltoallv_s += interp_1d(prof->curve[SP_CURVE_D2H], o) + interp_1d(prof->curve[SP_CURVE_CPU_CPU], o) +
                                 interp_1d(prof->curve[SP_CURVE_H2D], o);
        rep.model_unpack_s += interp_2d(prof->surf[SP_SURF_GPU_UNPACK], o, b);
        break;
      }
    }
  }
  for (auto &e : ev) cudaEventDestroy(e);
  for (int64_t rk = 0; rk < nranks; ++rk) {
    cudaFree(alloc[rk]);
    cudaFree(recv[rk]);
    if (send[rk]) cudaFree(send[rk]);
  }
  cudaStreamDestroy(s);
  return rep;
}

} // namespace spb
