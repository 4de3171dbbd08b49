// types.cpp -- definitions, commit pipeline, exact overlap, registry.
//
// Semantics follow the reference (paths relative to
// /root/reference/proj/include/stridepack/); the data structures are ours.
#include <algorithm>
#include <bit>
#include <cstring>
#include <functional>
#include <limits>

#include "core.hpp"

namespace spb {

[[noreturn]] void fail(sp_status code, std::string msg) {
  throw Error{code, std::move(msg)};
}

// ============================================================ definitions
// Constructor validation mirrors type_def.hpp:125-195; size/extent mirror
// type_def.hpp:198-250; span (one past the last described byte, the value
// the reference derives from its sorted block list, block_list.hpp:35) is
// computed here in closed form.

static const int64_t kNamedBytes[4] = {1, 4, 4, 8}; // type_def.hpp:17-29

DefPtr make_named(int kind) {
  if (kind < SP_BYTE || kind > SP_DOUBLE) fail(SP_ERR_INVALID_ARGUMENT, "named: unknown kind");
  auto d = std::make_shared<TypeDef>();
  d->kind = Kind::Named;
  d->named = kind;
  d->size = d->extent = d->span = kNamedBytes[kind];
  return d;
}

static void need_inner(const DefPtr &inner) {
  if (!inner) fail(SP_ERR_INVALID_HANDLE, "inner type is null");
}

DefPtr make_contiguous(int64_t count, DefPtr inner) {
  need_inner(inner);
  if (count < 0) fail(SP_ERR_INVALID_ARGUMENT, "contiguous: count must be >= 0");
  auto d = std::make_shared<TypeDef>();
  d->kind = Kind::Contiguous;
  d->count = count;
  d->size = count * inner->size;
  d->extent = count * inner->extent;
  d->span = (count == 0 || inner->span == 0) ? 0 : (count - 1) * inner->extent + inner->span;
  d->lb = count == 0 ? 0 : inner->lb;
  d->depth = inner->depth + 1;
  d->inner = std::move(inner);
  return d;
}

static DefPtr make_vec(Kind k, int64_t count, int64_t bl, int64_t stride, DefPtr inner) {
  need_inner(inner);
  const char *nm = k == Kind::Vector ? "vector" : "hvector";
  if (count < 0 || bl < 0) fail(SP_ERR_INVALID_ARGUMENT, std::string(nm) + ": count and blocklength must be >= 0");
  if (stride < 0) fail(SP_ERR_INVALID_ARGUMENT, std::string(nm) + ": negative strides are not representable");
  auto d = std::make_shared<TypeDef>();
  d->kind = k;
  d->count = count;
  d->blocklength = bl;
  d->stride = stride;
  const int64_t e = inner->extent;
  const int64_t step = k == Kind::Vector ? stride * e : stride; // bytes between blocks
  d->size = count * bl * inner->size;
  if (count == 0) {
    d->extent = 0;
  } else if (k == Kind::Vector) {
    d->extent = ((count - 1) * stride + bl) * e;
  } else {
    d->extent = (count - 1) * stride + bl * e;
  }
  d->span = (count == 0 || bl == 0 || inner->span == 0)
                ? 0
                : (count - 1) * step + (bl - 1) * e + inner->span;
  d->lb = (count == 0 || bl == 0) ? 0 : inner->lb;
  d->depth = inner->depth + 2;
  d->inner = std::move(inner);
  return d;
}

DefPtr make_vector(int64_t count, int64_t bl, int64_t stride, DefPtr inner) {
  return make_vec(Kind::Vector, count, bl, stride, std::move(inner));
}
DefPtr make_hvector(int64_t count, int64_t bl, int64_t stride_b, DefPtr inner) {
  return make_vec(Kind::Hvector, count, bl, stride_b, std::move(inner));
}

DefPtr make_subarray(int64_t ndims, const int64_t *sizes, const int64_t *subsizes,
                     const int64_t *offsets, DefPtr inner, int order) {
  need_inner(inner);
  if (order != SP_ORDER_C) fail(SP_ERR_UNSUPPORTED_ORDER, "subarray: only C array order is supported");
  if (ndims < 1) fail(SP_ERR_INVALID_ARGUMENT, "subarray: ndims must be >= 1");
  if (!sizes || !subsizes || !offsets) fail(SP_ERR_INVALID_ARGUMENT, "subarray: null array");
  auto d = std::make_shared<TypeDef>();
  d->kind = Kind::Subarray;
  d->sizes.assign(sizes, sizes + ndims);
  d->subsizes.assign(subsizes, subsizes + ndims);
  d->offsets.assign(offsets, offsets + ndims);
  for (int64_t i = 0; i < ndims; ++i) {
    if (sizes[i] < 1 || subsizes[i] < 1 || offsets[i] < 0)
      fail(SP_ERR_INVALID_ARGUMENT, "subarray: sizes and subsizes must be positive, offsets nonnegative");
    // zero-offset oversized dims are tolerated (type_def.hpp:181-189)
    if (offsets[i] + subsizes[i] > sizes[i] && !(offsets[i] == 0 && subsizes[i] > sizes[i]))
      fail(SP_ERR_INVALID_ARGUMENT, "subarray: offsets[" + std::to_string(i) + "]+subsizes[" +
                                        std::to_string(i) + "] exceeds sizes[" + std::to_string(i) + "]");
  }
  int64_t nsub = 1, nsize = 1, last = 0, dstride = inner->extent;
  for (int64_t i = 0; i < ndims; ++i) {
    nsub *= subsizes[i];
    nsize *= sizes[i];
    last += (offsets[i] + subsizes[i] - 1) * dstride;
    dstride *= sizes[i];
  }
  d->size = nsub * inner->size;
  d->extent = nsize * inner->extent;
  d->span = inner->span == 0 ? 0 : last + inner->span;
  d->depth = inner->depth + static_cast<int>(ndims);
  d->inner = std::move(inner);
  return d;
}

// ---- beyond the reference: MPI indexed / struct / resized (MPI-3.1
// 4.1.2-4.1.7). Displacements are bytes from the type's origin and must be
// nonnegative (the engine addresses from the buffer start, like the
// reference's nonnegative strides). lb/extent follow MPI: over the blocks
// that describe bytes, lb = min(disp + member lb) and ub = max(disp +
// member lb + blocklength * member extent); no alignment padding is added
// to struct extents (set one with a resized type).
static DefPtr make_blocks(Kind k, int64_t count, const int64_t *bl, const int64_t *displs,
                          std::vector<DefPtr> members) {
  const char *nm = k == Kind::Indexed ? "indexed" : "struct";
  if (count < 0) fail(SP_ERR_INVALID_ARGUMENT, std::string(nm) + ": count must be >= 0");
  if (count > 0 && (!bl || !displs)) fail(SP_ERR_INVALID_ARGUMENT, std::string(nm) + ": null array");
  auto d = std::make_shared<TypeDef>();
  d->kind = k;
  d->count = count;
  d->blocklens.assign(bl, bl + count);
  d->displs.assign(displs, displs + count);
  bool any = false;
  int64_t lo = 0, hi = 0, span = 0, depth = 0;
  for (int64_t i = 0; i < count; ++i) {
    const TypeDef &m = *members[static_cast<size_t>(k == Kind::Indexed ? 0 : i)];
    if (bl[i] < 0) fail(SP_ERR_INVALID_ARGUMENT, std::string(nm) + ": blocklengths must be >= 0");
    if (displs[i] < 0) fail(SP_ERR_INVALID_ARGUMENT, std::string(nm) + ": negative displacements are not representable");
    depth = std::max<int64_t>(depth, m.depth);
    d->size += bl[i] * m.size;
    if (bl[i] == 0) continue;
    const int64_t a = displs[i] + m.lb, b = displs[i] + m.lb + bl[i] * m.extent;
    lo = any ? std::min(lo, a) : a;
    hi = any ? std::max(hi, b) : b;
    any = true;
    if (m.span > 0) span = std::max(span, displs[i] + (bl[i] - 1) * m.extent + m.span);
  }
  d->lb = any ? lo : 0;
  d->extent = any ? hi - lo : 0;
  d->span = span;
  d->depth = static_cast<int>(depth) + 2;
  if (k == Kind::Indexed) {
    d->inner = std::move(members[0]);
  } else {
    d->members = std::move(members);
  }
  return d;
}

DefPtr make_indexed(int64_t count, const int64_t *blocklens, const int64_t *displs_bytes, DefPtr inner) {
  need_inner(inner);
  return make_blocks(Kind::Indexed, count, blocklens, displs_bytes, {std::move(inner)});
}

DefPtr make_struct(int64_t count, const int64_t *blocklens, const int64_t *displs_bytes,
                   const std::vector<DefPtr> &members) {
  if (static_cast<int64_t>(members.size()) != count) fail(SP_ERR_INVALID_ARGUMENT, "struct: one type per block");
  for (const DefPtr &m : members) need_inner(m);
  return make_blocks(Kind::Struct, count, blocklens, displs_bytes, members);
}

DefPtr make_resized(DefPtr inner, int64_t lb, int64_t extent) {
  need_inner(inner);
  if (extent < 0) fail(SP_ERR_INVALID_ARGUMENT, "resized: negative extents are not representable");
  auto d = std::make_shared<TypeDef>();
  d->kind = Kind::Resized;
  d->size = inner->size;
  d->span = inner->span;
  d->lb = lb;
  d->extent = extent;
  d->depth = inner->depth;
  d->inner = std::move(inner);
  return d;
}

// ============================================================ canonicalisation
// The IR chain is stored BASE FIRST: c[0] is the dense base, c.back() the
// head. Each pass walks bottom-up, which is the order the reference's
// recursion rewrites nodes (canon.hpp:22-111); a rewrite at level k is seen
// by level k+1 within the same pass, never re-examined below.

namespace {

struct Link {
  bool dense;
  int64_t off;    // both kinds (ir.hpp:14, :26)
  int64_t stride; // stream
  int64_t count;  // stream
  int64_t extent; // dense
};

Link dense_link(int64_t off, int64_t extent) { return {true, off, 0, 0, extent}; }
Link stream_link(int64_t off, int64_t stride, int64_t count) { return {false, off, stride, count, 0}; }

// The blocks of an indexed/struct level that describe bytes, abutting
// neighbours (same member, next block starts where this one ends) merged,
// which keeps the definition order intact.
struct Block {
  const TypeDef *member;
  int64_t disp, count;
};
std::vector<Block> live_blocks(const TypeDef &d) {
  std::vector<Block> out;
  for (size_t i = 0; i < d.blocklens.size(); ++i) {
    const TypeDef *m = d.kind == Kind::Indexed ? d.inner.get() : d.members[i].get();
    if (d.blocklens[i] == 0 || m->size == 0) continue;
    if (!out.empty() && out.back().member == m && out.back().disp + out.back().count * m->extent == d.displs[i]) {
      out.back().count += d.blocklens[i];
    } else {
      out.push_back({m, d.displs[i], d.blocklens[i]});
    }
  }
  return out;
}

// translate (ir.hpp:112-147): one link per constructor level. Levels the
// IR cannot express (indexed/struct blocks that are not one arithmetic
// progression of equal blocks of one type) return false.
bool translate(const TypeDef &d, std::vector<Link> &c) {
  switch (d.kind) {
  case Kind::Named:
    c.push_back(dense_link(0, d.size));
    return true;
  case Kind::Contiguous:
    if (!translate(*d.inner, c)) return false;
    c.push_back(stream_link(0, d.inner->extent, d.count));
    return true;
  case Kind::Vector:
  case Kind::Hvector: {
    const int64_t e = d.inner->extent;
    if (!translate(*d.inner, c)) return false;
    c.push_back(stream_link(0, e, d.blocklength));
    c.push_back(stream_link(0, d.kind == Kind::Vector ? d.stride * e : d.stride, d.count));
    return true;
  }
  case Kind::Subarray: {
    if (!translate(*d.inner, c)) return false;
    int64_t stride = d.inner->extent;
    for (size_t i = 0; i < d.sizes.size(); ++i) {
      c.push_back(stream_link(d.offsets[i] * stride, stride, d.subsizes[i]));
      stride *= d.sizes[i];
    }
    return true;
  }
  case Kind::Resized: // the inner layout; parents step by the new extent
    return translate(*d.inner, c);
  case Kind::Indexed:
  case Kind::Struct: {
    const std::vector<Block> b = live_blocks(d);
    if (b.empty()) { // describes no bytes: an empty element
      c.push_back(dense_link(0, 0));
      return true;
    }
    const TypeDef *m = b[0].member;
    const int64_t step = b.size() > 1 ? b[1].disp - b[0].disp : 0;
    for (size_t i = 1; i < b.size(); ++i)
      if (b[i].member != m || b[i].count != b[0].count || b[i].disp - b[i - 1].disp != step) return false;
    if (step < 0) return false;
    if (!translate(*m, c)) return false;
    c.push_back(stream_link(0, m->extent, b[0].count));
    c.push_back(stream_link(b[0].disp, step, static_cast<int64_t>(b.size())));
    return true;
  }
  }
  return false;
}

// dense folding (canon.hpp:22-37): stream over dense with extent == stride
bool fold(std::vector<Link> &c) {
  bool changed = false;
  for (size_t k = 1; k < c.size();) {
    const Link p = c[k], ch = c[k - 1];
    if (!p.dense && ch.dense && ch.extent == p.stride) {
      c[k - 1] = dense_link(p.off + ch.off, p.count * p.stride);
      c.erase(c.begin() + static_cast<long>(k));
      changed = true;
    } else {
      ++k;
    }
  }
  return changed;
}

// stream elision (canon.hpp:40-56): count-1 streams vanish, offset kept
bool elide(std::vector<Link> &c) {
  bool changed = false;
  for (size_t k = 1; k < c.size();) {
    if (!c[k].dense && c[k].count == 1) {
      c[k - 1].off += c[k].off;
      c.erase(c.begin() + static_cast<long>(k));
      changed = true;
    } else {
      ++k;
    }
  }
  return changed;
}

// stream flattening (canon.hpp:60-77): parent stride spans the child exactly
bool flatten(std::vector<Link> &c) {
  bool changed = false;
  for (size_t k = 1; k < c.size();) {
    const Link p = c[k], ch = c[k - 1];
    if (!p.dense && !ch.dense && p.stride == ch.count * ch.stride) {
      c[k - 1] = stream_link(p.off + ch.off, ch.stride, p.count * ch.count);
      c.erase(c.begin() + static_cast<long>(k));
      changed = true;
    } else {
      ++k;
    }
  }
  return changed;
}

// sorting (canon.hpp:83-111). Head-first order is stride desc, count desc,
// offset asc; base-first storage therefore wants the exact reverse.
bool sort_links(std::vector<Link> &c) {
  if (c.size() < 3) return false; // fewer than two streams
  auto head_first_less = [](const Link &a, const Link &b) {
    if (a.stride != b.stride) return a.stride > b.stride;
    if (a.count != b.count) return a.count > b.count;
    return a.off < b.off;
  };
  std::vector<Link> s(c.rbegin(), c.rend() - 1); // streams, head first
  if (std::is_sorted(s.begin(), s.end(), head_first_less)) return false;
  std::sort(s.begin(), s.end(), head_first_less);
  std::copy(s.rbegin(), s.rend(), c.begin() + 1);
  return true;
}

} // namespace

// ============================================================ overlap
// A StridedBlock describes byte start + sum_{d>=1} i_d s_d + b, b < c0. Two
// index tuples collide iff some nonzero difference vector delta with
// |delta_d| <= c_d - 1 has |sum delta_d s_d| < c0. Decided exactly:
//  1. any s_d < c0 (with c_d >= 2) collides at once (delta = e_d);
//  2. nested spans (each stride covers everything below it) never collide;
//  3. otherwise a bounded branch-and-bound over delta from the largest
//     stride down (each level can only pick deltas that keep the residual
//     within reach of the levels below), with a node budget backed by an
//     exact sort of run starts. The reference gets the same bit from its
//     O(size log size) block-list normalisation (commit.hpp:57-59).
bool strided_overlaps(const StridedBlock &sb) {
  const int64_t c0 = sb.counts[0];
  std::vector<std::pair<int64_t, int64_t>> dims; // (stride, count), count >= 2
  for (int d = 1; d < sb.ndims(); ++d)
    if (sb.counts[d] >= 2) dims.emplace_back(sb.strides[d], sb.counts[d]);
  if (dims.empty()) return false;
  std::sort(dims.begin(), dims.end());
  for (auto &[s, c] : dims)
    if (s < c0) return true;
  {
    int64_t reach = c0; // bytes spanned by everything below
    bool nested = true;
    for (auto &[s, c] : dims) {
      if (s < reach) {
        nested = false;
        break;
      }
      reach += (c - 1) * s;
    }
    if (nested) return false;
  }
  const size_t n = dims.size();
  std::vector<int64_t> below(n + 1, 0); // below[k] = reach of dims [0,k)
  for (size_t k = 0; k < n; ++k) below[k + 1] = below[k] + (dims[k].second - 1) * dims[k].first;
  int64_t budget = 20'000'000;
  bool exhausted = false;
  // returns true when a collision exists; level k descending
  std::function<bool(int, int64_t, bool)> dfs = [&](int k, int64_t resid, bool all_zero) -> bool {
    if (--budget < 0) {
      exhausted = true;
      return false;
    }
    if (k < 0) return !all_zero && resid > -c0 && resid < c0;
    const int64_t s = dims[k].first, cmax = dims[k].second - 1;
    const int64_t lim = c0 - 1 + below[k]; // |resid + delta*s| must be <= lim
    // delta in [ceil((-lim - resid)/s), floor((lim - resid)/s)]
    auto floordiv = [](int64_t a, int64_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); };
    int64_t lo = -floordiv(lim + resid, s);
    int64_t hi = floordiv(lim - resid, s);
    lo = std::max(lo, all_zero ? int64_t{0} : -cmax); // first nonzero delta > 0
    hi = std::min(hi, cmax);
    for (int64_t dl = lo; dl <= hi; ++dl) {
      if (dfs(k - 1, resid + dl * s, all_zero && dl == 0)) return true;
      if (exhausted) return false;
    }
    return false;
  };
  const bool hit = dfs(static_cast<int>(n) - 1, 0, true);
  if (!exhausted) return hit;
  // exact fallback: sort every run start and look for a gap below c0
  std::vector<int64_t> starts{0};
  for (auto &[s, c] : dims) {
    const size_t m = starts.size();
    starts.reserve(m * static_cast<size_t>(c));
    for (int64_t i = 1; i < c; ++i)
      for (size_t j = 0; j < m; ++j) starts.push_back(starts[j] + i * s);
  }
  std::sort(starts.begin(), starts.end());
  for (size_t i = 1; i < starts.size(); ++i)
    if (starts[i] - starts[i - 1] < c0) return true;
  return false;
}

// ============================================================ plan
// select_word_size (plan.hpp:47-64) and make_plan (plan.hpp:77-99): the
// reference's descriptive plan, recorded for parity and reporting. The
// kernels choose their own word from the actual buffer addresses too.
static RefPlan reference_plan(const StridedBlock &sb) {
  RefPlan p;
  p.word = 1;
  for (int64_t w : {16, 8, 4, 2}) {
    if (sb.counts[0] % w || sb.start % w) continue;
    bool ok = true;
    for (int d = 1; d < sb.ndims(); ++d) ok = ok && sb.strides[d] % w == 0;
    if (ok) {
      p.word = w;
      break;
    }
  }
  const int64_t ext[3] = {sb.counts[0] / p.word, sb.ndims() > 1 ? sb.counts[1] : 1,
                          sb.ndims() > 2 ? sb.counts[2] : 1};
  int64_t budget = 1024;
  for (int d = 0; d < 3; ++d) {
    const int64_t b = std::min<int64_t>(static_cast<int64_t>(std::bit_ceil(static_cast<uint64_t>(ext[d]))), budget);
    p.block[d] = b;
    budget /= b;
    p.grid[d] = (ext[d] + b - 1) / b;
  }
  p.strategy = sb.ndims() <= 2 ? SP_STRATEGY_GRIDZ : SP_STRATEGY_ITERATE;
  return p;
}

// ============================================================ runs
// Definition-order runs (block_list.hpp:67-121) for the Unsupported form,
// built level by level: the inner list is replicated at each placement and
// runs that abut in both source and packed order are coalesced (which keeps
// the gather byte-identical and the multiplicity intact).
static void push_run(std::vector<Run> &out, int64_t off, int64_t len) {
  if (len == 0) return;
  if (!out.empty() && out.back().off + out.back().len == off) {
    out.back().len += len;
  } else {
    out.push_back({off, len});
  }
}

static std::vector<Run> def_runs(const TypeDef &d) {
  std::vector<Run> out;
  auto place = [&](const std::vector<Run> &in, int64_t base) {
    for (const Run &r : in) push_run(out, base + r.off, r.len);
  };
  switch (d.kind) {
  case Kind::Named:
    push_run(out, 0, d.size);
    break;
  case Kind::Contiguous: {
    const auto in = def_runs(*d.inner);
    for (int64_t i = 0; i < d.count; ++i) place(in, i * d.inner->extent);
    break;
  }
  case Kind::Vector:
  case Kind::Hvector: {
    const auto in = def_runs(*d.inner);
    const int64_t e = d.inner->extent;
    const int64_t step = d.kind == Kind::Vector ? d.stride * e : d.stride;
    for (int64_t i = 0; i < d.count; ++i)
      for (int64_t j = 0; j < d.blocklength; ++j) place(in, i * step + j * e);
    break;
  }
  case Kind::Resized:
    out = def_runs(*d.inner);
    break;
  case Kind::Indexed:
  case Kind::Struct:
    for (size_t i = 0; i < d.blocklens.size(); ++i) {
      const TypeDef &m = d.kind == Kind::Indexed ? *d.inner : *d.members[i];
      if (d.blocklens[i] == 0) continue;
      const auto in = def_runs(m);
      for (int64_t j = 0; j < d.blocklens[i]; ++j) place(in, d.displs[i] + j * m.extent);
    }
    break;
  case Kind::Subarray: {
    const auto in = def_runs(*d.inner);
    const size_t nd = d.sizes.size();
    std::vector<int64_t> dstride(nd), idx(nd, 0);
    int64_t s = d.inner->extent;
    for (size_t k = 0; k < nd; ++k) {
      dstride[k] = s;
      s *= d.sizes[k];
    }
    for (;;) {
      int64_t off = 0;
      for (size_t k = 0; k < nd; ++k) off += (d.offsets[k] + idx[k]) * dstride[k];
      place(in, off);
      size_t k = 0;
      while (k < nd && ++idx[k] == d.subsizes[k]) idx[k++] = 0;
      if (k == nd) break;
    }
    break;
  }
  }
  return out;
}

// normalize_blocks (block_list.hpp:44-61): sorted by (offset, length),
// abutting or overlapping runs merged; overlap records bytes described twice
std::vector<Run> flatten_def(const TypeDef &def, bool &overlap) {
  std::vector<Run> runs = def_runs(def);
  std::sort(runs.begin(), runs.end(),
            [](const Run &a, const Run &b) { return a.off != b.off ? a.off < b.off : a.len < b.len; });
  std::vector<Run> out;
  overlap = false;
  for (const Run &r : runs) {
    if (!out.empty() && r.off <= out.back().off + out.back().len) {
      Run &cur = out.back();
      if (r.off < cur.off + cur.len) overlap = true;
      cur.len = std::max(cur.len, r.off + r.len - cur.off);
    } else {
      out.push_back(r);
    }
  }
  return out;
}

static int64_t leaf_bytes(const TypeDef &d) {
  const TypeDef *p = &d;
  while (p->kind != Kind::Named) p = p->kind == Kind::Struct ? p->members[0].get() : p->inner.get();
  return p->size;
}

// whether the definition uses a constructor the reference does not have
static bool beyond_reference(const TypeDef &d) {
  if (d.kind == Kind::Indexed || d.kind == Kind::Struct || d.kind == Kind::Resized) return true;
  return d.inner && beyond_reference(*d.inner);
}

// ============================================================ commit
CommitPtr commit_def(const TypeDef &def) {
  auto ct = std::make_shared<Committed>();
  ct->size = def.size;
  ct->extent = def.extent;
  ct->span = def.span;
  if (def.size == 0) { // commit.hpp:61-64
    ct->form = SP_FORM_EMPTY;
    return ct;
  }
  std::vector<Link> c;
  c.reserve(static_cast<size_t>(def.depth));
  if (!translate(def, c)) {
    // an irregular indexed/struct level: the block-list form, in MPI
    // typemap (definition) order; unpack is allowed unless bytes repeat
    ct->form = SP_FORM_UNSUPPORTED;
    ct->runs = def_runs(def);
    std::vector<Run> sorted = ct->runs;
    std::sort(sorted.begin(), sorted.end(), [](const Run &a, const Run &b) { return a.off < b.off; });
    for (size_t i = 1; i < sorted.size() && !ct->overlapping; ++i)
      ct->overlapping = sorted[i].off < sorted[i - 1].off + sorted[i - 1].len;
    ct->n_def_runs = static_cast<int64_t>(ct->runs.size());
    return ct;
  }
  bool coincident = false; // canon.hpp:118-130
  for (const Link &l : c)
    if (!l.dense && l.count >= 2 && l.stride < 1) coincident = true;
  if (!coincident) {
    const int64_t len = static_cast<int64_t>(c.size());
    const int64_t limit = len * len + 2;
    int64_t rounds = 0;
    bool changed = true;
    while (changed) { // canon.hpp:136-146
      if (++rounds > limit) fail(SP_ERR_INTERNAL, "simplify did not reach a fixpoint");
      changed = fold(c);
      changed |= elide(c);
      changed |= flatten(c);
      changed |= sort_links(c);
    }
    // lower (strided_block.hpp:54-89)
    bool ok = c[0].dense && c[0].extent >= 1;
    StridedBlock sb;
    if (ok) {
      sb.start = c[0].off;
      sb.counts.push_back(c[0].extent);
      sb.strides.push_back(1);
      for (size_t k = 1; k < c.size() && ok; ++k) {
        ok = !c[k].dense && c[k].count >= 1 && c[k].stride >= 1;
        sb.start += c[k].off;
        sb.counts.push_back(c[k].count);
        sb.strides.push_back(c[k].stride);
      }
    }
    if (ok) {
      ct->form = SP_FORM_STRIDED;
      ct->simplify_rounds = rounds;
      ct->plan = reference_plan(sb);
      ct->sb = std::move(sb);
      ct->overlapping = strided_overlaps(ct->sb);
      return ct;
    }
  }
  // Unsupported (commit.hpp:73-78): a coincident (stride-0, count >= 2)
  // stream over a non-empty element describes its bytes at least twice.
  ct->form = SP_FORM_UNSUPPORTED;
  ct->overlapping = true;
  ct->runs = def_runs(def);
  ct->n_def_runs = beyond_reference(def) ? static_cast<int64_t>(ct->runs.size()) : def.size / leaf_bytes(def);
  return ct;
}

// ============================================================ registry
sp_type Registry::add(DefPtr def) {
  std::unique_lock lk(mu_);
  const sp_type h = next_++;
  map_.emplace(h, Entry{std::move(def), nullptr});
  return h;
}

Entry Registry::get(sp_type h) const {
  std::shared_lock lk(mu_);
  auto it = map_.find(h);
  if (it == map_.end()) fail(SP_ERR_INVALID_HANDLE, "unknown type handle " + std::to_string(h));
  return it->second;
}

CommitPtr Registry::committed(sp_type h) const {
  std::shared_lock lk(mu_);
  auto it = map_.find(h);
  if (it == map_.end()) fail(SP_ERR_INVALID_HANDLE, "unknown type handle " + std::to_string(h));
  if (!it->second.committed) fail(SP_ERR_INVALID_ARGUMENT, "type is not committed");
  return it->second.committed;
}

CommitPtr Registry::commit(sp_type h) {
  Entry e = get(h);
  if (e.committed) return e.committed;
  // the pipeline runs outside the lock (commit.hpp:81-84)
  CommitPtr ct = commit_def(*e.def);
  std::unique_lock lk(mu_);
  auto it = map_.find(h);
  if (it == map_.end()) fail(SP_ERR_INVALID_HANDLE, "type handle freed during commit");
  if (!it->second.committed) it->second.committed = ct;
  return it->second.committed;
}

void Registry::remove(sp_type h) {
  std::unique_lock lk(mu_);
  if (!map_.erase(h)) fail(SP_ERR_INVALID_HANDLE, "unknown type handle " + std::to_string(h));
  gen_.fetch_add(1, std::memory_order_release);
}

Registry &registry() {
  static Registry r;
  return r;
}

} // namespace spb
