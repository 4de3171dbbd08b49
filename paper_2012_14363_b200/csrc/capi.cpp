// capi.cpp -- extern "C" entry points of libstridepack_b200.so.
// Every call converts internal errors (spb::Error) into an sp_status and a
// thread-local message; nothing throws across the ABI.
#include <algorithm>
#include <cstring>
#include <exception>
#include <new>
#include <memory>
#include <string>
#include <vector>

#include "core.hpp"
#include "trace.hpp"

namespace {

thread_local std::string t_err;

template <class F> sp_status guard(F &&f) {
  try {
    t_err.clear();
    f();
    return SP_OK;
  } catch (const spb::Error &e) {
    t_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc &) {
    t_err = "out of host memory";
    return SP_ERR_INTERNAL;
  } catch (const std::exception &e) {
    t_err = e.what();
    return SP_ERR_INTERNAL;
  }
}

spb::DefPtr def_of(sp_type h) { return spb::registry().get(h).def; }

sp_status add(spb::DefPtr d, sp_type *out) {
  if (!out) spb::fail(SP_ERR_INVALID_ARGUMENT, "null output handle");
  *out = spb::registry().add(std::move(d));
  return SP_OK;
}

} // namespace

namespace spb {
void set_last_error(const std::string &msg) { t_err = msg; }
} // namespace spb

extern "C" {

int sp_abi_version(void) { return SP_ABI_VERSION; }

const char *sp_status_string(sp_status s) {
  switch (s) {
  case SP_OK: return "ok";
  case SP_ERR_INVALID_ARGUMENT: return "InvalidArgument";
  case SP_ERR_UNSUPPORTED_ORDER: return "UnsupportedOrder";
  case SP_ERR_INVALID_LAYOUT: return "InvalidLayout";
  case SP_ERR_BUFFER_TOO_SMALL: return "BufferTooSmall";
  case SP_ERR_OVERLAPPING_LAYOUT: return "OverlappingLayout";
  case SP_ERR_UNSUPPORTED: return "Unsupported";
  case SP_ERR_EMPTY_PROFILE: return "EmptyProfile";
  case SP_ERR_PARSE: return "ParseError";
  case SP_ERR_INTERNAL: return "InternalError";
  case SP_ERR_INVALID_HANDLE: return "InvalidHandle";
  case SP_ERR_CUDA: return "CudaError";
  case SP_ERR_NO_DEVICE: return "NoDevice";
  case SP_ERR_TIMEOUT: return "Timeout";
  default: return "unknown";
  }
}

const char *sp_last_error(void) { return t_err.c_str(); }

sp_status sp_type_named(int kind, sp_type *out) {
  return guard([&] { add(spb::make_named(kind), out); });
}

sp_status sp_type_contiguous(int64_t count, sp_type inner, sp_type *out) {
  return guard([&] { add(spb::make_contiguous(count, def_of(inner)), out); });
}

sp_status sp_type_vector(int64_t count, int64_t blocklength, int64_t stride, sp_type inner, sp_type *out) {
  return guard([&] { add(spb::make_vector(count, blocklength, stride, def_of(inner)), out); });
}

sp_status sp_type_hvector(int64_t count, int64_t blocklength, int64_t stride_bytes, sp_type inner,
                          sp_type *out) {
  return guard([&] { add(spb::make_hvector(count, blocklength, stride_bytes, def_of(inner)), out); });
}

sp_status sp_type_subarray(int64_t ndims, const int64_t *sizes, const int64_t *subsizes,
                           const int64_t *offsets, sp_type inner, int order, sp_type *out) {
  return guard([&] { add(spb::make_subarray(ndims, sizes, subsizes, offsets, def_of(inner), order), out); });
}

// ---- beyond the reference (MPI-3.1 4.1.2-4.1.7)
sp_status sp_type_hindexed(int64_t count, const int64_t *blocklens, const int64_t *displs_bytes, sp_type inner,
                           sp_type *out) {
  return guard([&] { add(spb::make_indexed(count, blocklens, displs_bytes, def_of(inner)), out); });
}

sp_status sp_type_indexed(int64_t count, const int64_t *blocklens, const int64_t *displs, sp_type inner,
                          sp_type *out) {
  return guard([&] {
    spb::DefPtr in = def_of(inner);
    if (count > 0 && !displs) spb::fail(SP_ERR_INVALID_ARGUMENT, "indexed: null array");
    std::vector<int64_t> b(displs, displs + std::max<int64_t>(count, 0));
    for (int64_t &x : b) x *= in->extent;
    add(spb::make_indexed(count, blocklens, b.data(), std::move(in)), out);
  });
}

sp_status sp_type_hindexed_block(int64_t count, int64_t blocklen, const int64_t *displs_bytes, sp_type inner,
                                 sp_type *out) {
  return guard([&] {
    std::vector<int64_t> bl(static_cast<size_t>(std::max<int64_t>(count, 0)), blocklen);
    add(spb::make_indexed(count, bl.data(), displs_bytes, def_of(inner)), out);
  });
}

sp_status sp_type_indexed_block(int64_t count, int64_t blocklen, const int64_t *displs, sp_type inner,
                                sp_type *out) {
  return guard([&] {
    spb::DefPtr in = def_of(inner);
    if (count > 0 && !displs) spb::fail(SP_ERR_INVALID_ARGUMENT, "indexed_block: null array");
    std::vector<int64_t> bl(static_cast<size_t>(std::max<int64_t>(count, 0)), blocklen);
    std::vector<int64_t> b(displs, displs + std::max<int64_t>(count, 0));
    for (int64_t &x : b) x *= in->extent;
    add(spb::make_indexed(count, bl.data(), b.data(), std::move(in)), out);
  });
}

sp_status sp_type_struct(int64_t count, const int64_t *blocklens, const int64_t *displs_bytes,
                         const sp_type *types, sp_type *out) {
  return guard([&] {
    if (count > 0 && !types) spb::fail(SP_ERR_INVALID_ARGUMENT, "struct: null array");
    std::vector<spb::DefPtr> m;
    for (int64_t i = 0; i < count; ++i) m.push_back(def_of(types[i]));
    add(spb::make_struct(count, blocklens, displs_bytes, m), out);
  });
}

sp_status sp_type_resized(sp_type inner, int64_t lb, int64_t extent, sp_type *out) {
  return guard([&] { add(spb::make_resized(def_of(inner), lb, extent), out); });
}

sp_status sp_type_lb(sp_type t, int64_t *lb) {
  return guard([&] {
    if (!lb) spb::fail(SP_ERR_INVALID_ARGUMENT, "null output");
    *lb = def_of(t)->lb;
  });
}

sp_status sp_type_free(sp_type t) {
  return guard([&] { spb::registry().remove(t); });
}

sp_status sp_type_size(sp_type t, int64_t *size) {
  return guard([&] {
    if (!size) spb::fail(SP_ERR_INVALID_ARGUMENT, "null output");
    *size = def_of(t)->size;
  });
}

sp_status sp_type_extent(sp_type t, int64_t *extent) {
  return guard([&] {
    if (!extent) spb::fail(SP_ERR_INVALID_ARGUMENT, "null output");
    *extent = def_of(t)->extent;
  });
}

sp_status sp_type_flatten(sp_type t, int64_t *offsets, int64_t *lengths, int64_t cap, int64_t *n, int *overlap) {
  return guard([&] {
    if (!n) spb::fail(SP_ERR_INVALID_ARGUMENT, "null output");
    bool ov = false;
    const std::vector<spb::Run> runs = spb::flatten_def(*def_of(t), ov);
    *n = static_cast<int64_t>(runs.size());
    if (overlap) *overlap = ov ? 1 : 0;
    if (offsets && lengths && cap >= *n) {
      for (size_t i = 0; i < runs.size(); ++i) {
        offsets[i] = runs[i].off;
        lengths[i] = runs[i].len;
      }
    }
  });
}

sp_status sp_type_commit(sp_type t) {
  SPB_TRACE("sp_type_commit");
  return guard([&] { spb::registry().commit(t); });
}

sp_status sp_type_query(sp_type t, sp_type_info *info, int64_t *counts, int64_t *strides, int64_t cap) {
  return guard([&] {
    if (!info) spb::fail(SP_ERR_INVALID_ARGUMENT, "null info");
    const spb::Entry e = spb::registry().get(t);
    if (!e.committed) spb::fail(SP_ERR_INVALID_ARGUMENT, "type is not committed");
    const spb::Committed &c = *e.committed;
    std::memset(info, 0, sizeof(*info));
    info->form = c.form;
    info->size = c.size;
    info->extent = c.extent;
    info->span = c.span;
    info->overlapping = c.overlapping;
    info->simplify_rounds = c.simplify_rounds;
    info->n_fallback_runs = c.n_def_runs;
    if (c.form == SP_FORM_STRIDED) {
      info->ndims = c.sb.ndims();
      info->start = c.sb.start;
      info->word = c.plan.word;
      for (int d = 0; d < 3; ++d) {
        info->block[d] = c.plan.block[d];
        info->grid[d] = c.plan.grid[d];
      }
      info->strategy = c.plan.strategy;
      if (counts && strides && cap >= info->ndims) {
        for (int d = 0; d < c.sb.ndims(); ++d) {
          counts[d] = c.sb.counts[d];
          strides[d] = c.sb.strides[d];
        }
      }
    }
  });
}

static sp_status pack_impl(bool pack, const void *src, uint64_t src_bytes, sp_type t, int64_t count, void *dst,
                           uint64_t dst_bytes, int64_t *position, void *stream, const sp_pack_options *opt) {
  SPB_TRACE(pack ? "sp_pack" : "sp_unpack");
  return guard([&] {
    if (!position) spb::fail(SP_ERR_INVALID_ARGUMENT, "null position");
    const spb::Entry e = spb::registry().get(t);
    if (!e.committed) spb::fail(SP_ERR_INVALID_ARGUMENT, "type is not committed");
    spb::PackArgs a{};
    a.ct = e.committed.get();
    a.src = src;
    a.src_bytes = src_bytes;
    a.dst = dst;
    a.dst_bytes = dst_bytes;
    a.count = count;
    a.position = *position;
    a.stream = stream;
    a.opt = opt ? *opt : sp_pack_options{1, SP_KERNEL_AUTO, 0};
    a.pack = pack;
    *position = spb::execute(a);
  });
}

sp_status sp_pack(const void *src, uint64_t src_bytes, sp_type t, int64_t incount, void *dst, uint64_t dst_bytes,
                  int64_t *position, void *stream) {
  return pack_impl(true, src, src_bytes, t, incount, dst, dst_bytes, position, stream, nullptr);
}

sp_status sp_unpack(const void *src, uint64_t src_bytes, int64_t *position, sp_type t, int64_t outcount, void *dst,
                    uint64_t dst_bytes, void *stream) {
  return pack_impl(false, src, src_bytes, t, outcount, dst, dst_bytes, position, stream, nullptr);
}

sp_status sp_pack_ex(const void *src, uint64_t src_bytes, sp_type t, int64_t incount, void *dst, uint64_t dst_bytes,
                     int64_t *position, void *stream, const sp_pack_options *opt) {
  return pack_impl(true, src, src_bytes, t, incount, dst, dst_bytes, position, stream, opt);
}

sp_status sp_unpack_ex(const void *src, uint64_t src_bytes, int64_t *position, sp_type t, int64_t outcount,
                       void *dst, uint64_t dst_bytes, void *stream, const sp_pack_options *opt) {
  return pack_impl(false, src, src_bytes, t, outcount, dst, dst_bytes, position, stream, opt);
}

} // extern "C"

struct sp_batch_s {
  spb::Batch *b = nullptr;
  std::vector<spb::CommitPtr> keep; // committed types outlive the plan
  ~sp_batch_s() { spb::batch_destroy(b); }
};

extern "C" {

sp_status sp_batch_create(const sp_batch_job *jobs, int64_t n, int unpack, sp_batch *out) {
  return guard([&] {
    if (!out || (n > 0 && !jobs) || n < 0) spb::fail(SP_ERR_INVALID_ARGUMENT, "bad batch arguments");
    auto h = std::make_unique<sp_batch_s>();
    std::vector<spb::BatchSpec> specs;
    for (int64_t i = 0; i < n; ++i) {
      const spb::Entry e = spb::registry().get(jobs[i].type);
      if (!e.committed) spb::fail(SP_ERR_INVALID_ARGUMENT, "type is not committed");
      h->keep.push_back(e.committed);
      specs.push_back({e.committed.get(), jobs[i].src, jobs[i].src_bytes, jobs[i].count, jobs[i].dst,
                       jobs[i].dst_bytes, jobs[i].position});
    }
    h->b = spb::batch_create(specs, unpack != 0);
    *out = h.release();
  });
}

namespace {
// one dense run per object and objects back to back: the packed format
bool dense(const spb::Committed &c, int64_t count) {
  return c.form == SP_FORM_STRIDED && c.sb.ndims() == 1 && (count <= 1 || c.extent == c.size);
}

// a typed copy with a block-list (irregular) side: a run-table pack into a
// dense destination, or a run-table unpack from a dense source
bool copy_blocklist(const sp_copy_job &j, const spb::Committed &cs, const spb::Committed &cd, void *stream) {
  if (cs.form == SP_FORM_STRIDED && cd.form == SP_FORM_STRIDED) return false;
  if (j.src_count * cs.size != j.dst_count * cd.size)
    spb::fail(SP_ERR_INVALID_ARGUMENT, "copy: source and destination describe different byte counts");
  if (j.src_count * cs.size == 0) return true;
  spb::PackArgs a{};
  a.stream = stream;
  a.opt = sp_pack_options{1, SP_KERNEL_AUTO, 0};
  if (cs.form != SP_FORM_STRIDED && dense(cd, j.dst_count)) {
    if (j.dst_bytes < static_cast<uint64_t>(cd.sb.start)) spb::fail(SP_ERR_BUFFER_TOO_SMALL, "copy: destination too small");
    a.ct = &cs;
    a.src = j.src;
    a.src_bytes = j.src_bytes;
    a.dst = static_cast<uint8_t *>(j.dst) + cd.sb.start;
    a.dst_bytes = j.dst_bytes - static_cast<uint64_t>(cd.sb.start);
    a.count = j.src_count;
    a.pack = true;
  } else if (cd.form != SP_FORM_STRIDED && dense(cs, j.src_count)) {
    if (j.src_bytes < static_cast<uint64_t>(cs.sb.start)) spb::fail(SP_ERR_BUFFER_TOO_SMALL, "copy: source too small");
    a.ct = &cd;
    a.src = static_cast<const uint8_t *>(j.src) + cs.sb.start;
    a.src_bytes = j.src_bytes - static_cast<uint64_t>(cs.sb.start);
    a.dst = j.dst;
    a.dst_bytes = j.dst_bytes;
    a.count = j.dst_count;
    a.pack = false;
  } else {
    spb::fail(SP_ERR_UNSUPPORTED, "copy: a block-list (irregular) layout needs a dense run on the other side");
  }
  spb::execute(a);
  return true;
}
} // namespace

sp_status sp_copy(const sp_copy_job *job, void *stream) {
  SPB_TRACE("sp_copy");
  return guard([&] {
    if (!job) spb::fail(SP_ERR_INVALID_ARGUMENT, "null job");
    const spb::Entry es = spb::registry().get(job->src_type), ed = spb::registry().get(job->dst_type);
    if (!es.committed || !ed.committed) spb::fail(SP_ERR_INVALID_ARGUMENT, "type is not committed");
    if (copy_blocklist(*job, *es.committed, *ed.committed, stream)) return;
    const spb::CopySpec spec{es.committed.get(), job->src, job->src_bytes, job->src_count, ed.committed.get(),
                             job->dst, job->dst_bytes, job->dst_count};
    spb::copy_execute(spec, 0, static_cast<uint64_t>(job->src_count * es.committed->size), stream);
  });
}

sp_status sp_copy_batch_create(const sp_copy_job *jobs, int64_t n, sp_batch *out) {
  return guard([&] {
    if (!out || (n > 0 && !jobs) || n < 0) spb::fail(SP_ERR_INVALID_ARGUMENT, "bad batch arguments");
    auto h = std::make_unique<sp_batch_s>();
    std::vector<spb::CopySpec> specs;
    for (int64_t i = 0; i < n; ++i) {
      const spb::Entry es = spb::registry().get(jobs[i].src_type), ed = spb::registry().get(jobs[i].dst_type);
      if (!es.committed || !ed.committed) spb::fail(SP_ERR_INVALID_ARGUMENT, "type is not committed");
      h->keep.push_back(es.committed);
      h->keep.push_back(ed.committed);
      specs.push_back({es.committed.get(), jobs[i].src, jobs[i].src_bytes, jobs[i].src_count, ed.committed.get(),
                       jobs[i].dst, jobs[i].dst_bytes, jobs[i].dst_count});
    }
    h->b = spb::copy_batch_create(specs);
    *out = h.release();
  });
}

sp_status sp_batch_execute(sp_batch b, void *stream) {
  SPB_TRACE("sp_batch_execute");
  return guard([&] {
    if (!b) spb::fail(SP_ERR_INVALID_ARGUMENT, "null batch");
    spb::batch_execute(*b->b, stream);
  });
}

sp_status sp_batch_bytes(sp_batch b, int64_t *bytes) {
  return guard([&] {
    if (!b || !bytes) spb::fail(SP_ERR_INVALID_ARGUMENT, "null argument");
    *bytes = spb::batch_bytes(*b->b);
  });
}

sp_status sp_batch_free(sp_batch b) {
  delete b;
  return SP_OK;
}

} // extern "C"
