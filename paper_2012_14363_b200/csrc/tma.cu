// tma.cu -- TMA-tiled pack/unpack (sm_100a: cp.async.bulk.tensor + mbarrier).
//
// The strided side of a committed type is described to the Tensor Memory
// Accelerator as a tensor of rank 1 + nd: dimension 0 is the c0-byte row
// (in E-byte elements), dimensions 1..nd are the row dimensions with their
// byte strides (the object count included). A box of `by` whole rows of
// dimension 1 is contiguous in packed order, so
//   pack   : TMA tensor load (strided HBM -> smem) then a 1-D bulk copy
//            (smem -> packed HBM), per tile;
//   unpack : 1-D bulk copy (packed HBM -> smem) then a TMA tensor store
//            (smem -> strided HBM); out-of-range rows of a partial tile are
//            clipped by the TMA unit, so bytes outside the layout are never
//            written.
// One elected thread per CTA drives a ring of STAGES shared-memory buffers;
// the data never passes through registers. Applicability (checked on the
// host): c0 a multiple of 16 with c0/E <= 256 elements, every row stride and
// both base addresses 16-B aligned, at most 4 row dimensions.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "core.hpp"
#include "tma.hpp"

namespace spb {

namespace {

constexpr int kStages = 4;

struct TmaArgs {
  uint8_t *packed;   // packed side (already offset by position)
  uint32_t cnt[4];   // row-dim counts (dim 0 = TMA dim 1)
  int nd;
  uint32_t by;       // rows of dim 0 per tile
  uint32_t tpr;      // tiles per dim-0 run: ceil(cnt[0] / by)
  uint64_t ntiles;
  uint32_t c0;       // row bytes
  uint32_t stage_bytes; // smem bytes per stage (box, 128-B aligned)
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// tile -> TMA coordinates {0, dim1 start, i2, i3, i4} and its packed row
__device__ __forceinline__ void tile_coords(const TmaArgs &a, uint64_t t, int32_t c[5], uint64_t &row0,
                                            uint32_t &rows) {
  const uint32_t j = static_cast<uint32_t>(t % a.tpr);
  uint64_t rest = t / a.tpr;
  c[0] = 0;
  c[1] = static_cast<int32_t>(j * a.by);
  uint64_t lin = 0, mul = a.cnt[0];
  for (int k = 1; k < 4; ++k) {
    uint32_t i = 0;
    if (k < a.nd) {
      i = static_cast<uint32_t>(rest % a.cnt[k]);
      rest /= a.cnt[k];
      lin += static_cast<uint64_t>(i) * mul;
      mul *= a.cnt[k];
    }
    c[k + 1] = static_cast<int32_t>(i);
  }
  row0 = lin + static_cast<uint64_t>(j) * a.by;
  rows = min(a.by, a.cnt[0] - j * a.by);
}

__device__ __forceinline__ void tma_load(const CUtensorMap *map, uint8_t *dst, uint64_t *bar, const int32_t c[5]) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_store(const CUtensorMap *map, const uint8_t *src, const int32_t c[5]) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                   map),
               "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(src))
               : "memory");
}

__device__ __forceinline__ void bulk_s2g(uint8_t *dst, const uint8_t *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint8_t *dst, const uint8_t *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// pack: strided -> smem (TMA tensor load) -> packed (bulk copy)
__global__ void __launch_bounds__(32) k_tma_pack(const __grid_constant__ CUtensorMap map, const TmaArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[kStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint64_t first = blockIdx.x, step = gridDim.x;
  const uint64_t mine = first < a.ntiles ? (a.ntiles - first + step - 1) / step : 0;
  int32_t c[5];
  uint64_t row0;
  uint32_t rows;
  // prologue: fill all but one stage
  for (uint64_t i = 0; i < mine && i < kStages - 1; ++i) {
    tile_coords(a, first + i * step, c, row0, rows);
    mbar_expect_tx(&bar[i], a.by * a.c0);
    tma_load(&map, smem + i * a.stage_bytes, &bar[i], c);
  }
  for (uint64_t i = 0; i < mine; ++i) {
    const int s = static_cast<int>(i % kStages);
    mbar_wait(&bar[s], static_cast<uint32_t>((i / kStages) & 1));
    tile_coords(a, first + i * step, c, row0, rows);
    bulk_s2g(a.packed + row0 * a.c0, smem + s * a.stage_bytes, rows * a.c0);
    bulk_commit();
    // refill the stage freed by the previous tile's store
    const uint64_t nxt = i + kStages - 1;
    if (nxt < mine) {
      bulk_wait_read<1>();
      const int ns = static_cast<int>(nxt % kStages);
      tile_coords(a, first + nxt * step, c, row0, rows);
      mbar_expect_tx(&bar[ns], a.by * a.c0);
      tma_load(&map, smem + ns * a.stage_bytes, &bar[ns], c);
    }
  }
  bulk_wait_all();
}

// unpack: packed -> smem (bulk copy) -> strided (TMA tensor store, clipped)
__global__ void __launch_bounds__(32) k_tma_unpack(const __grid_constant__ CUtensorMap map, const TmaArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[kStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint64_t first = blockIdx.x, step = gridDim.x;
  const uint64_t mine = first < a.ntiles ? (a.ntiles - first + step - 1) / step : 0;
  int32_t c[5];
  uint64_t row0;
  uint32_t rows;
  for (uint64_t i = 0; i < mine && i < kStages - 1; ++i) {
    tile_coords(a, first + i * step, c, row0, rows);
    mbar_expect_tx(&bar[i], rows * a.c0);
    bulk_g2s(smem + i * a.stage_bytes, a.packed + row0 * a.c0, rows * a.c0, &bar[i]);
  }
  for (uint64_t i = 0; i < mine; ++i) {
    const int s = static_cast<int>(i % kStages);
    mbar_wait(&bar[s], static_cast<uint32_t>((i / kStages) & 1));
    tile_coords(a, first + i * step, c, row0, rows);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tma_store(&map, smem + s * a.stage_bytes, c);
    bulk_commit();
    const uint64_t nxt = i + kStages - 1;
    if (nxt < mine) {
      bulk_wait_read<1>();
      const int ns = static_cast<int>(nxt % kStages);
      tile_coords(a, first + nxt * step, c, row0, rows);
      mbar_expect_tx(&bar[ns], rows * a.c0);
      bulk_g2s(smem + ns * a.stage_bytes, a.packed + row0 * a.c0, rows * a.c0, &bar[ns]);
    }
  }
  bulk_wait_all();
}

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<EncodeFn>(nullptr);
    }
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

} // namespace

bool tma_applicable(const TmaGeometry &g) {
  if (g.nd < 1 || g.nd > 4 || g.c0 % 16 != 0 || g.str[0] < g.c0) return false;
  if ((g.strided_addr % 16) || (g.packed_addr % 16)) return false;
  for (int k = 0; k < g.nd; ++k)
    if (g.str[k] % 16 || g.str[k] >= (int64_t{1} << 40) || g.cnt[k] >= (int64_t{1} << 31)) return false;
  int64_t e = 8;
  while (e > 1 && (g.c0 % e)) e >>= 1;
  return g.c0 / e <= 256 && encode_fn() != nullptr;
}

void tma_launch(const TmaGeometry &g, const uint8_t *strided, uint8_t *packed, bool pack, void *stream,
                int64_t *grid_out) {
  if (!tma_applicable(g)) fail(SP_ERR_INVALID_ARGUMENT, "TMA path not applicable to this layout/buffers");
  int64_t e = 8;
  while (e > 1 && (g.c0 % e)) e >>= 1;
  const CUtensorMapDataType dt = e == 8   ? CU_TENSOR_MAP_DATA_TYPE_UINT64
                                 : e == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                                 : e == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                          : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  const uint32_t by = static_cast<uint32_t>(
      std::max<int64_t>(1, std::min<int64_t>({256, g.cnt[0], std::max<int64_t>(1, 16384 / g.c0)})));
  // the 5-D map: unused trailing dims have extent 1
  cuuint64_t dims[5] = {static_cast<cuuint64_t>(g.c0 / e), 1, 1, 1, 1};
  cuuint64_t strides[4] = {16, 16, 16, 16};
  for (int k = 0; k < g.nd; ++k) {
    dims[k + 1] = static_cast<cuuint64_t>(g.cnt[k]);
    strides[k] = static_cast<cuuint64_t>(g.str[k]);
  }
  for (int k = g.nd; k < 4; ++k) strides[k] = (k ? strides[k - 1] : 16) * dims[k]; // never stepped
  cuuint32_t box[5] = {static_cast<cuuint32_t>(g.c0 / e), by, 1, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  const CUresult r = encode_fn()(&map, dt, 5, const_cast<uint8_t *>(strided), dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(SP_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  TmaArgs a{};
  a.packed = packed;
  a.nd = g.nd;
  for (int k = 0; k < 4; ++k) a.cnt[k] = k < g.nd ? static_cast<uint32_t>(g.cnt[k]) : 1;
  a.by = by;
  a.tpr = (a.cnt[0] + by - 1) / by;
  uint64_t outer = 1;
  for (int k = 1; k < g.nd; ++k) outer *= a.cnt[k];
  a.ntiles = outer * a.tpr;
  a.c0 = static_cast<uint32_t>(g.c0);
  a.stage_bytes = (by * a.c0 + 127) / 128 * 128;
  const size_t smem = static_cast<size_t>(a.stage_bytes) * kStages;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(a.ntiles, static_cast<uint64_t>(sms) * 3));
  auto kern = pack ? k_tma_pack : k_tma_unpack;
  cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
             "cudaFuncSetAttribute");
  kern<<<grid, 32, smem, static_cast<cudaStream_t>(stream)>>>(map, a);
  cuda_check(cudaGetLastError(), "k_tma launch");
  if (grid_out) *grid_out = grid;
}

} // namespace spb
