// oracle/ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference engine
// ("stridepack", header-only C++20 under /root/reference/proj/include). It is
// compiled by oracle/Makefile directly against the reference headers where
// they lie; nothing from the reference is copied into this repository. The
// product library never links or loads this file: only tests/, bench.py's
// reference arm / cpu_baseline leg and __graft_entry__.smoke() may use it,
// and only as the checker.
//
// Types cross this boundary as a flat int64 "type program" in prefix order
// (shared with oracle/oracle.c and the product's tests):
//   named       : [0, kind]                       kind 0 byte,1 int,2 float,3 double
//   contiguous  : [1, count, <inner>]
//   vector      : [2, count, blocklength, stride, <inner>]
//   hvector     : [3, count, blocklength, stride_bytes, <inner>]
//   subarray    : [4, ndims, order, sizes[ndims], subsizes[ndims],
//                  offsets[ndims], <inner>]       order 0 = C, 1 = Fortran
// Status codes mirror proj/include/stridepack/errors.hpp:8-47:
//   0 ok, 1 InvalidArgument, 2 UnsupportedOrder, 3 InvalidLayout,
//   4 BufferTooSmall, 5 OverlappingLayout, 6 Unsupported, 7 EmptyProfile,
//   8 ParseError, 9 other std::exception, 10 malformed program.

#include <cstdint>
#include <cstring>
#include <exception>
#include <fstream>
#include <memory>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include <stridepack/stridepack.hpp>

#include "test_util.hpp"

using namespace stridepack;

namespace {

struct BadProgram {};

TypeDef parse(const int64_t *p, int64_t n, int64_t &at) {
  if (at >= n) throw BadProgram{};
  const int64_t tag = p[at++];
  auto next = [&]() {
    if (at >= n) throw BadProgram{};
    return p[at++];
  };
  switch (tag) {
  case 0: {
    const int64_t k = next();
    if (k < 0 || k > 3) throw BadProgram{};
    return make_named(static_cast<NamedKind>(k));
  }
  case 1: {
    const int64_t c = next();
    TypeDef in = parse(p, n, at);
    return make_contiguous(c, std::move(in));
  }
  case 2:
  case 3: {
    const int64_t c = next(), l = next(), s = next();
    TypeDef in = parse(p, n, at);
    return tag == 2 ? make_vector(c, l, s, std::move(in))
                    : make_hvector(c, l, s, std::move(in));
  }
  case 4: {
    const int64_t nd = next();
    const int64_t order = next();
    if (nd < 0 || nd > 64) throw BadProgram{};
    std::vector<int64_t> sz(nd), sub(nd), off(nd);
    for (auto &v : sz) v = next();
    for (auto &v : sub) v = next();
    for (auto &v : off) v = next();
    TypeDef in = parse(p, n, at);
    return make_subarray(nd, sz, sub, off, std::move(in),
                         order == 0 ? ArrayOrder::C : ArrayOrder::Fortran);
  }
  default:
    throw BadProgram{};
  }
}

TypeDef parse_all(const int64_t *p, int64_t n) {
  int64_t at = 0;
  TypeDef d = parse(p, n, at);
  if (at != n) throw BadProgram{};
  return d;
}

void emit(const TypeDef &def, std::vector<int64_t> &out) {
  std::visit(
      [&](const auto &node) {
        using T = std::decay_t<decltype(node)>;
        if constexpr (std::is_same_v<T, TypeDef::Named>) {
          out.push_back(0);
          out.push_back(static_cast<int64_t>(node.kind));
        } else if constexpr (std::is_same_v<T, TypeDef::Contiguous>) {
          out.push_back(1);
          out.push_back(node.count);
          emit(def.inner(), out);
        } else if constexpr (std::is_same_v<T, TypeDef::Vector>) {
          out.insert(out.end(), {2, node.count, node.blocklength, node.stride});
          emit(def.inner(), out);
        } else if constexpr (std::is_same_v<T, TypeDef::Hvector>) {
          out.insert(out.end(),
                     {3, node.count, node.blocklength, node.stride_bytes});
          emit(def.inner(), out);
        } else {
          const int64_t nd = static_cast<int64_t>(node.sizes.size());
          out.push_back(4);
          out.push_back(nd);
          out.push_back(0);
          out.insert(out.end(), node.sizes.begin(), node.sizes.end());
          out.insert(out.end(), node.subsizes.begin(), node.subsizes.end());
          out.insert(out.end(), node.offsets.begin(), node.offsets.end());
          emit(def.inner(), out);
        }
      },
      def.node());
}

template <class F> int guarded(F &&f) {
  try {
    f();
    return 0;
  } catch (const BadProgram &) {
    return 10;
  } catch (const InvalidArgument &) {
    return 1;
  } catch (const UnsupportedOrder &) {
    return 2;
  } catch (const InvalidLayout &) {
    return 3;
  } catch (const BufferTooSmall &) {
    return 4;
  } catch (const OverlappingLayout &) {
    return 5;
  } catch (const Unsupported &) {
    return 6;
  } catch (const EmptyProfile &) {
    return 7;
  } catch (const ParseError &) {
    return 8;
  } catch (const std::exception &) {
    return 9;
  }
}

} // namespace

extern "C" {

#define REF_MAXD 64

// Everything commit_type() derives (commit.hpp:30-43).
struct ref_commit_info {
  int64_t form; // 0 Strided, 1 Empty, 2 Unsupported (commit.hpp:21-25)
  int64_t size, extent, span, overlapping;
  int64_t ndims, start;
  int64_t counts[REF_MAXD], strides[REF_MAXD];
  int64_t word, block[3], grid[3], strategy; // strategy 0 gridz, 1 iterate
  int64_t n_fallback_runs;
  int64_t simplify_rounds; // -1 when simplify threw / was not run
};

int ref_commit(const int64_t *prog, int64_t n, ref_commit_info *out) {
  return guarded([&] {
    const TypeDef def = parse_all(prog, n);
    const CommittedType ct = commit_type(def);
    std::memset(out, 0, sizeof(*out));
    out->form = ct.form == CanonForm::Strided ? 0
                : ct.form == CanonForm::Empty ? 1
                                              : 2;
    out->size = ct.size;
    out->extent = ct.extent;
    out->span = ct.span;
    out->overlapping = ct.overlapping;
    out->n_fallback_runs = static_cast<int64_t>(ct.fallback_runs.size());
    out->simplify_rounds = -1;
    if (ct.canon) {
      if (ct.canon->ndims() > REF_MAXD) throw BadProgram{};
      out->ndims = ct.canon->ndims();
      out->start = ct.canon->start;
      for (int64_t i = 0; i < out->ndims; ++i) {
        out->counts[i] = ct.canon->counts[i];
        out->strides[i] = ct.canon->strides[i];
      }
      out->word = ct.plan->word;
      for (int d = 0; d < 3; ++d) {
        out->block[d] = ct.plan->block_dims[d];
        out->grid[d] = ct.plan->grid_dims[d];
      }
      out->strategy = ct.plan->count_strategy == CountStrategy::GridZ ? 0 : 1;
      int64_t rounds = 0;
      simplify(translate(def), &rounds);
      out->simplify_rounds = rounds;
    }
  });
}

// type_size / type_extent without a commit (type_def.hpp:198-250)
int ref_size_extent(const int64_t *prog, int64_t n, int64_t *size,
                    int64_t *extent) {
  return guarded([&] {
    const TypeDef def = parse_all(prog, n);
    *size = type_size(def);
    *extent = type_extent(def);
  });
}

// normalized oracle block list (block_list.hpp:129-131)
int ref_flatten(const int64_t *prog, int64_t n, int64_t *offsets,
                int64_t *lengths, int64_t cap, int64_t *count,
                int64_t *overlap) {
  return guarded([&] {
    const BlockList bl = flatten_oracle(parse_all(prog, n));
    *count = static_cast<int64_t>(bl.blocks.size());
    *overlap = bl.overlap;
    for (int64_t i = 0; i < *count && i < cap; ++i) {
      offsets[i] = bl.blocks[i].offset;
      lengths[i] = bl.blocks[i].length;
    }
  });
}

// pack (pack.hpp:99-137)
int ref_pack(const int64_t *prog, int64_t n, const uint8_t *src,
             uint64_t src_len, int64_t incount, uint8_t *dst,
             uint64_t dst_len, int64_t position, int threads,
             int allow_fallback, int64_t *new_position) {
  return guarded([&] {
    const CommittedType ct = commit_type(parse_all(prog, n));
    *new_position = pack(std::span<const uint8_t>(src, src_len), ct, incount,
                         std::span<uint8_t>(dst, dst_len), position,
                         PackOptions{threads, allow_fallback != 0});
  });
}

// unpack (pack.hpp:143-185)
int ref_unpack(const int64_t *prog, int64_t n, const uint8_t *src,
               uint64_t src_len, int64_t position, int64_t outcount,
               uint8_t *dst, uint64_t dst_len, int threads, int allow_fallback,
               int64_t *new_position) {
  return guarded([&] {
    const CommittedType ct = commit_type(parse_all(prog, n));
    *new_position =
        unpack(std::span<const uint8_t>(src, src_len), position, ct, outcount,
               std::span<uint8_t>(dst, dst_len),
               PackOptions{threads, allow_fallback != 0});
  });
}

// Committed-type handles so timing loops exclude the O(size log size) commit.
void *ref_commit_handle(const int64_t *prog, int64_t n, int *status) {
  CommittedType *ct = nullptr;
  *status = guarded([&] { ct = new CommittedType(commit_type(parse_all(prog, n))); });
  return ct;
}
void ref_free_handle(void *h) { delete static_cast<CommittedType *>(h); }

int ref_pack_h(void *h, const uint8_t *src, uint64_t src_len, int64_t incount,
               uint8_t *dst, uint64_t dst_len, int64_t position, int threads,
               int64_t *new_position) {
  return guarded([&] {
    *new_position = pack(std::span<const uint8_t>(src, src_len),
                         *static_cast<CommittedType *>(h), incount,
                         std::span<uint8_t>(dst, dst_len), position,
                         PackOptions{threads, true});
  });
}

int ref_unpack_h(void *h, const uint8_t *src, uint64_t src_len,
                 int64_t position, int64_t outcount, uint8_t *dst,
                 uint64_t dst_len, int threads, int64_t *new_position) {
  return guarded([&] {
    *new_position = unpack(std::span<const uint8_t>(src, src_len), position,
                           *static_cast<CommittedType *>(h), outcount,
                           std::span<uint8_t>(dst, dst_len),
                           PackOptions{threads, true});
  });
}

// The reference's own randomized generator (tests/test_util.hpp:86-151),
// driven exactly as acceptance.cpp:59-69 drives it when mode == 0
// (regular_only = i % 3 == 0); mode 1 = regular_only for all, no empties
// (acceptance.cpp:175-178); mode 2 = defaults. Emits programs back to back,
// each prefixed with its length. Returns the number of int64s written or
// -needed when cap is too small.
int64_t ref_corpus(uint64_t seed, int64_t count, int mode, int64_t *out,
                   int64_t cap) {
  std::mt19937_64 rng(seed);
  std::vector<int64_t> all;
  for (int64_t i = 0; i < count; ++i) {
    test_util::GenOptions opt;
    if (mode == 0) {
      opt.regular_only = (i % 3 == 0);
    } else if (mode == 1) {
      opt.regular_only = true;
      opt.allow_empty = false;
    }
    const TypeDef def = test_util::random_def(rng, opt);
    std::vector<int64_t> prog;
    emit(def, prog);
    all.push_back(static_cast<int64_t>(prog.size()));
    all.insert(all.end(), prog.begin(), prog.end());
  }
  if (static_cast<int64_t>(all.size()) > cap) {
    return -static_cast<int64_t>(all.size());
  }
  std::copy(all.begin(), all.end(), out);
  return static_cast<int64_t>(all.size());
}

// ---- performance model (perf_model.hpp, profile_io.hpp) ----

void *ref_profile_load(const char *path, int *status) {
  MachineProfile *p = nullptr;
  *status = guarded([&] { p = new MachineProfile(load_profile_file(path)); });
  return p;
}

void *ref_profile_parse(const char *text, int *status) {
  MachineProfile *p = nullptr;
  *status = guarded([&] {
    std::istringstream in(text);
    p = new MachineProfile(load_profile(in));
  });
  return p;
}

void ref_profile_free(void *p) { delete static_cast<MachineProfile *>(p); }

// save_profile (profile_io.hpp:174-213) into a caller buffer; returns the
// number of bytes (excluding NUL) or -needed.
int64_t ref_profile_save(void *p, const char *header, char *buf, int64_t cap) {
  std::ostringstream out;
  save_profile(out, *static_cast<MachineProfile *>(p), header ? header : "");
  const std::string s = out.str();
  if (static_cast<int64_t>(s.size()) + 1 > cap) {
    return -static_cast<int64_t>(s.size() + 1);
  }
  std::memcpy(buf, s.data(), s.size());
  buf[s.size()] = 0;
  return static_cast<int64_t>(s.size());
}

// choose_method + the three model times (perf_model.hpp:139-179)
int ref_choose(void *p, int64_t object_size, int64_t block_size, int *method,
               double *t_dev, double *t_one, double *t_stg) {
  return guarded([&] {
    const MachineProfile &mp = *static_cast<MachineProfile *>(p);
    const ModelQuery q{object_size, block_size};
    const MethodChoice m = choose_method(mp, q);
    *method = m == MethodChoice::OneShot ? 0 : m == MethodChoice::Device ? 1 : 2;
    *t_dev = t_device(mp, q);
    *t_one = t_oneshot(mp, q);
    *t_stg = t_staged(mp, q);
  });
}

// scaled copy (tests/test_util.hpp:153-167)
void *ref_profile_scaled(void *p, double k) {
  auto *c = new MachineProfile(*static_cast<MachineProfile *>(p));
  test_util::scale_profile(*c, k);
  return c;
}

// ---- halo (halo.hpp) ----
struct ref_halo_report {
  double pack_seconds, alltoallv_seconds, unpack_seconds;
  int64_t verified, bytes_moved;
};

int ref_run_exchange(const int64_t ranks[3], const int64_t interior[3],
                     int64_t radius, int64_t element_bytes, void *profile,
                     ref_halo_report *out) {
  return guarded([&] {
    HaloConfig cfg;
    for (int a = 0; a < 3; ++a) {
      cfg.ranks[a] = ranks[a];
      cfg.interior[a] = interior[a];
    }
    cfg.radius = radius;
    cfg.element_bytes = element_bytes;
    const ExchangeReport r =
        run_exchange(cfg, *static_cast<MachineProfile *>(profile));
    out->pack_seconds = r.pack_seconds;
    out->alltoallv_seconds = r.alltoallv_seconds;
    out->unpack_seconds = r.unpack_seconds;
    out->verified = r.verified;
    out->bytes_moved = r.bytes_moved;
  });
}

// The 26 region types (halo.hpp:98-130) as programs: for k in 0..25,
// dir[3], gridpoints, then send program (len-prefixed), recv program.
int64_t ref_halo_types(const int64_t interior[3], int64_t radius,
                       int64_t element_bytes, int64_t *out, int64_t cap) {
  std::vector<int64_t> all;
  const int st = guarded([&] {
    HaloConfig cfg;
    for (int a = 0; a < 3; ++a) cfg.interior[a] = interior[a];
    cfg.radius = radius;
    cfg.element_bytes = element_bytes;
    for (const HaloRegion &r : build_halo_types(cfg)) {
      all.insert(all.end(), {r.dir[0], r.dir[1], r.dir[2], r.gridpoints});
      for (const TypeDef *d : {&r.send, &r.recv}) {
        std::vector<int64_t> prog;
        emit(*d, prog);
        all.push_back(static_cast<int64_t>(prog.size()));
        all.insert(all.end(), prog.begin(), prog.end());
      }
    }
  });
  if (st != 0) return -1000000 - st;
  if (static_cast<int64_t>(all.size()) > cap) return -static_cast<int64_t>(all.size());
  std::copy(all.begin(), all.end(), out);
  return static_cast<int64_t>(all.size());
}

// the halo payload pattern (halo.hpp:152-164)
void ref_fill_cell(uint8_t *dst, int64_t gx, int64_t gy, int64_t gz,
                   int64_t elem) {
  detail::fill_cell(dst, gx, gy, gz, elem);
}

} // extern "C"
