/* oracle/oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * A line-by-line *restatement* (not a copy) of the reference's semantics in
 * C11. Each function names the reference file:line it follows; all paths are
 * relative to /root/reference/proj/include/stridepack/.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* definition tree (type_def.hpp:52-123)                                */
/* ------------------------------------------------------------------ */

enum { K_NAMED = 0, K_CONTIG = 1, K_VECTOR = 2, K_HVECTOR = 3, K_SUBARRAY = 4 };

typedef struct def {
  int kind;
  int64_t named_size; /* type_def.hpp:17-29 */
  int64_t count, blocklength, stride;
  int64_t ndims;
  int64_t *sizes, *subsizes, *offsets;
  struct def *inner;
} def_t;

static void def_free(def_t *d) {
  while (d) {
    def_t *in = d->inner;
    free(d->sizes);
    free(d->subsizes);
    free(d->offsets);
    free(d);
    d = in;
  }
}

/* constructor validation: type_def.hpp:125-195 */
static int parse(const int64_t *p, int64_t n, int64_t *at, def_t **out) {
  *out = NULL;
  if (*at >= n) return OR_BAD_PROGRAM;
  def_t *d = (def_t *)calloc(1, sizeof(def_t));
  d->kind = (int)p[(*at)++];
  int st = OR_OK;
#define NEXT(v)                                                             \
  do {                                                                      \
    if (*at >= n) {                                                         \
      st = OR_BAD_PROGRAM;                                                  \
      goto fail;                                                            \
    }                                                                       \
    (v) = p[(*at)++];                                                       \
  } while (0)
  switch (d->kind) {
  case K_NAMED: {
    int64_t k;
    NEXT(k);
    static const int64_t sz[4] = {1, 4, 4, 8};
    if (k < 0 || k > 3) {
      st = OR_BAD_PROGRAM;
      goto fail;
    }
    d->named_size = sz[k];
    *out = d;
    return OR_OK;
  }
  case K_CONTIG:
    NEXT(d->count);
    break;
  case K_VECTOR:
  case K_HVECTOR:
    NEXT(d->count);
    NEXT(d->blocklength);
    NEXT(d->stride);
    break;
  case K_SUBARRAY: {
    int64_t order;
    NEXT(d->ndims);
    NEXT(order);
    if (d->ndims < 0 || d->ndims > 64) {
      st = OR_BAD_PROGRAM;
      goto fail;
    }
    d->sizes = (int64_t *)calloc((size_t)d->ndims + 1, sizeof(int64_t));
    d->subsizes = (int64_t *)calloc((size_t)d->ndims + 1, sizeof(int64_t));
    d->offsets = (int64_t *)calloc((size_t)d->ndims + 1, sizeof(int64_t));
    for (int64_t i = 0; i < d->ndims; ++i) NEXT(d->sizes[i]);
    for (int64_t i = 0; i < d->ndims; ++i) NEXT(d->subsizes[i]);
    for (int64_t i = 0; i < d->ndims; ++i) NEXT(d->offsets[i]);
    st = parse(p, n, at, &d->inner);
    if (st) goto fail;
    /* make_subarray argument checks, in the reference's order */
    if (order != 0) {
      st = OR_UNSUPPORTED_ORDER;
      goto fail;
    }
    if (d->ndims < 1) {
      st = OR_INVALID_ARGUMENT;
      goto fail;
    }
    for (int64_t i = 0; i < d->ndims; ++i) {
      if (d->sizes[i] < 1 || d->subsizes[i] < 1 || d->offsets[i] < 0) {
        st = OR_INVALID_ARGUMENT;
        goto fail;
      }
      if (d->offsets[i] + d->subsizes[i] > d->sizes[i] &&
          !(d->offsets[i] == 0 && d->subsizes[i] > d->sizes[i])) {
        st = OR_INVALID_ARGUMENT;
        goto fail;
      }
    }
    *out = d;
    return OR_OK;
  }
  default:
    st = OR_BAD_PROGRAM;
    goto fail;
  }
  st = parse(p, n, at, &d->inner);
  if (st) goto fail;
  if (d->kind == K_CONTIG && d->count < 0) {
    st = OR_INVALID_ARGUMENT;
    goto fail;
  }
  if (d->kind == K_VECTOR || d->kind == K_HVECTOR) {
    if (d->count < 0 || d->blocklength < 0 || d->stride < 0) {
      st = OR_INVALID_ARGUMENT;
      goto fail;
    }
  }
  *out = d;
  return OR_OK;
fail:
  def_free(d);
  return st;
#undef NEXT
}

static int parse_all(const int64_t *p, int64_t n, def_t **out) {
  int64_t at = 0;
  int st = parse(p, n, &at, out);
  if (st == OR_OK && at != n) {
    def_free(*out);
    *out = NULL;
    return OR_BAD_PROGRAM;
  }
  return st;
}

/* type_size: type_def.hpp:198-218 */
static int64_t type_size(const def_t *d) {
  switch (d->kind) {
  case K_NAMED:
    return d->named_size;
  case K_CONTIG:
    return d->count * type_size(d->inner);
  case K_VECTOR:
  case K_HVECTOR:
    return d->count * d->blocklength * type_size(d->inner);
  default: {
    int64_t prod = 1;
    for (int64_t i = 0; i < d->ndims; ++i) prod *= d->subsizes[i];
    return prod * type_size(d->inner);
  }
  }
}

/* type_extent: type_def.hpp:221-250 */
static int64_t type_extent(const def_t *d) {
  switch (d->kind) {
  case K_NAMED:
    return d->named_size;
  case K_CONTIG:
    return d->count * type_extent(d->inner);
  case K_VECTOR:
    if (d->count == 0) return 0;
    return ((d->count - 1) * d->stride + d->blocklength) * type_extent(d->inner);
  case K_HVECTOR:
    if (d->count == 0) return 0;
    return (d->count - 1) * d->stride + d->blocklength * type_extent(d->inner);
  default: {
    int64_t prod = 1;
    for (int64_t i = 0; i < d->ndims; ++i) prod *= d->sizes[i];
    return prod * type_extent(d->inner);
  }
  }
}

/* ------------------------------------------------------------------ */
/* block lists (block_list.hpp:12-159)                                  */
/* ------------------------------------------------------------------ */

typedef struct {
  int64_t off, len;
} blk_t;

typedef struct {
  blk_t *v;
  int64_t n, cap;
} blkvec_t;

static void bv_push(blkvec_t *b, int64_t off, int64_t len) {
  if (b->n == b->cap) {
    b->cap = b->cap ? b->cap * 2 : 64;
    b->v = (blk_t *)realloc(b->v, (size_t)b->cap * sizeof(blk_t));
  }
  b->v[b->n].off = off;
  b->v[b->n].len = len;
  b->n++;
}

/* flatten_runs: block_list.hpp:67-121 -- definition-order runs */
static void flatten_runs(const def_t *d, int64_t base, blkvec_t *out) {
  switch (d->kind) {
  case K_NAMED:
    bv_push(out, base, d->named_size);
    return;
  case K_CONTIG: {
    const int64_t e = type_extent(d->inner);
    for (int64_t i = 0; i < d->count; ++i) flatten_runs(d->inner, base + i * e, out);
    return;
  }
  case K_VECTOR:
  case K_HVECTOR: {
    const int64_t e = type_extent(d->inner);
    const int64_t step = d->kind == K_VECTOR ? d->stride * e : d->stride;
    for (int64_t i = 0; i < d->count; ++i)
      for (int64_t j = 0; j < d->blocklength; ++j)
        flatten_runs(d->inner, base + i * step + j * e, out);
    return;
  }
  default: {
    const int64_t nd = d->ndims;
    int64_t dim_stride[64], idx[64];
    int64_t stride = type_extent(d->inner);
    for (int64_t k = 0; k < nd; ++k) {
      dim_stride[k] = stride;
      stride *= d->sizes[k];
      idx[k] = 0;
    }
    for (;;) {
      int64_t off = 0;
      for (int64_t k = 0; k < nd; ++k) off += (d->offsets[k] + idx[k]) * dim_stride[k];
      flatten_runs(d->inner, base + off, out);
      int64_t k = 0;
      while (k < nd && ++idx[k] == d->subsizes[k]) {
        idx[k] = 0;
        ++k;
      }
      if (k == nd) break;
    }
    return;
  }
  }
}

static int blk_cmp(const void *a, const void *b) {
  const blk_t *x = (const blk_t *)a, *y = (const blk_t *)b;
  if (x->off != y->off) return x->off < y->off ? -1 : 1;
  if (x->len != y->len) return x->len < y->len ? -1 : 1;
  return 0;
}

/* normalize_blocks: block_list.hpp:41-60 (in place) */
static int normalize(blkvec_t *b) {
  int overlap = 0;
  int64_t w = 0;
  for (int64_t i = 0; i < b->n; ++i)
    if (b->v[i].len != 0) b->v[w++] = b->v[i];
  b->n = w;
  qsort(b->v, (size_t)b->n, sizeof(blk_t), blk_cmp);
  int64_t m = 0;
  for (int64_t i = 0; i < b->n; ++i) {
    const blk_t r = b->v[i];
    if (m > 0 && r.off <= b->v[m - 1].off + b->v[m - 1].len) {
      blk_t *cur = &b->v[m - 1];
      if (r.off < cur->off + cur->len) overlap = 1;
      const int64_t end = r.off + r.len - cur->off;
      if (end > cur->len) cur->len = end;
    } else {
      b->v[m++] = r;
    }
  }
  b->n = m;
  return overlap;
}

/* ------------------------------------------------------------------ */
/* IR chain (ir.hpp:13-147); index 0 = head, last = dense base          */
/* ------------------------------------------------------------------ */

typedef struct {
  int dense;
  int64_t off, stride, count; /* stream fields */
  int64_t extent;             /* dense field */
} node_t;

typedef struct {
  node_t *v;
  int64_t n, cap;
} chain_t;

static void ch_insert_head(chain_t *c, node_t x) {
  if (c->n == c->cap) {
    c->cap = c->cap ? c->cap * 2 : 16;
    c->v = (node_t *)realloc(c->v, (size_t)c->cap * sizeof(node_t));
  }
  memmove(c->v + 1, c->v, (size_t)c->n * sizeof(node_t));
  c->v[0] = x;
  c->n++;
}

static void ch_erase(chain_t *c, int64_t i) {
  memmove(c->v + i, c->v + i + 1, (size_t)(c->n - i - 1) * sizeof(node_t));
  c->n--;
}

static node_t stream(int64_t off, int64_t stride, int64_t count) {
  node_t x = {0, off, stride, count, 0};
  return x;
}

/* translate: ir.hpp:112-147 */
static void translate(const def_t *d, chain_t *c) {
  switch (d->kind) {
  case K_NAMED: {
    node_t x = {1, 0, 0, 0, d->named_size};
    ch_insert_head(c, x);
    return;
  }
  case K_CONTIG:
    translate(d->inner, c);
    ch_insert_head(c, stream(0, type_extent(d->inner), d->count));
    return;
  case K_VECTOR:
  case K_HVECTOR: {
    const int64_t e = type_extent(d->inner);
    translate(d->inner, c);
    ch_insert_head(c, stream(0, e, d->blocklength));
    ch_insert_head(c, stream(0, d->kind == K_VECTOR ? d->stride * e : d->stride,
                             d->count));
    return;
  }
  default: {
    int64_t stride = type_extent(d->inner);
    translate(d->inner, c);
    for (int64_t i = 0; i < d->ndims; ++i) {
      ch_insert_head(c, stream(d->offsets[i] * stride, stride, d->subsizes[i]));
      stride *= d->sizes[i];
    }
    return;
  }
  }
}

/* The four passes of canon.hpp, each applied bottom-up exactly as the
 * reference's recursion does (children rewritten before their parent). */

/* dense_folding: canon.hpp:22-37 */
static int dense_folding(chain_t *c) {
  int changed = 0;
  for (int64_t i = c->n - 2; i >= 0; --i) {
    node_t *p = &c->v[i], *ch = &c->v[i + 1];
    if (p->dense || !ch->dense) continue;
    if (ch->extent != p->stride) continue;
    node_t x = {1, p->off + ch->off, 0, 0, p->count * p->stride};
    c->v[i] = x;
    ch_erase(c, i + 1);
    changed = 1;
  }
  return changed;
}

/* stream_elision: canon.hpp:40-56 (head elision included) */
static int stream_elision(chain_t *c) {
  int changed = 0;
  for (int64_t i = c->n - 2; i >= 0; --i) {
    if (c->v[i].dense || c->v[i].count != 1) continue;
    c->v[i + 1].off += c->v[i].off;
    ch_erase(c, i);
    changed = 1;
  }
  return changed;
}

/* stream_flatten: canon.hpp:60-77 */
static int stream_flatten(chain_t *c) {
  int changed = 0;
  for (int64_t i = c->n - 2; i >= 0; --i) {
    node_t *p = &c->v[i], *ch = &c->v[i + 1];
    if (p->dense || ch->dense) continue;
    if (p->stride != ch->count * ch->stride) continue;
    node_t x = stream(p->off + ch->off, ch->stride, p->count * ch->count);
    c->v[i] = x;
    ch_erase(c, i + 1);
    changed = 1;
  }
  return changed;
}

/* sort key: canon.hpp:92-101 -- stride desc, count desc, offset asc */
static int stream_cmp(const void *a, const void *b) {
  const node_t *x = (const node_t *)a, *y = (const node_t *)b;
  if (x->stride != y->stride) return x->stride > y->stride ? -1 : 1;
  if (x->count != y->count) return x->count > y->count ? -1 : 1;
  if (x->off != y->off) return x->off < y->off ? -1 : 1;
  return 0;
}

/* sort_streams: canon.hpp:83-111 */
static int sort_streams(chain_t *c) {
  int64_t k = 0;
  while (k < c->n && !c->v[k].dense) ++k;
  if (k < 2) return 0;
  node_t *before = (node_t *)malloc((size_t)k * sizeof(node_t));
  memcpy(before, c->v, (size_t)k * sizeof(node_t));
  qsort(c->v, (size_t)k, sizeof(node_t), stream_cmp);
  int changed = 0;
  for (int64_t i = 0; i < k; ++i) {
    if (before[i].off != c->v[i].off || before[i].stride != c->v[i].stride ||
        before[i].count != c->v[i].count)
      changed = 1;
  }
  free(before);
  return changed;
}

/* simplify: canon.hpp:117-149 */
static int simplify(chain_t *c, int64_t *rounds_out) {
  for (int64_t i = 0; i < c->n; ++i) {
    if (!c->v[i].dense && c->v[i].count >= 2 && c->v[i].stride < 1)
      return OR_INVALID_LAYOUT;
  }
  const int64_t len = c->n;
  const int64_t limit = len * len + 2;
  int64_t rounds = 0;
  int changed = 1;
  while (changed) {
    if (++rounds > limit) return OR_INTERNAL;
    changed = dense_folding(c);
    changed |= stream_elision(c);
    changed |= stream_flatten(c);
    changed |= sort_streams(c);
  }
  if (rounds_out) *rounds_out = rounds;
  return OR_OK;
}

typedef struct {
  int64_t start, ndims;
  int64_t counts[OR_MAXD + 1], strides[OR_MAXD + 1];
} sb_t;

/* to_strided_block: strided_block.hpp:54-89; returns 0 for nullopt */
static int to_strided_block(const chain_t *c, sb_t *sb) {
  const node_t *base = &c->v[c->n - 1];
  if (!base->dense || base->extent < 1) return 0;
  if (c->n > OR_MAXD) return 0;
  sb->start = base->off;
  sb->ndims = 1;
  sb->counts[0] = base->extent;
  sb->strides[0] = 1;
  for (int64_t i = c->n - 2; i >= 0; --i) {
    const node_t *s = &c->v[i];
    if (s->dense || s->count < 1 || s->stride < 1) return 0;
    sb->start += s->off;
    sb->counts[sb->ndims] = s->count;
    sb->strides[sb->ndims] = s->stride;
    sb->ndims++;
  }
  return 1;
}

/* select_word_size: plan.hpp:47-64 */
static int64_t select_word_size(const sb_t *sb) {
  static const int64_t ws[4] = {16, 8, 4, 2};
  for (int k = 0; k < 4; ++k) {
    const int64_t w = ws[k];
    if (sb->counts[0] % w != 0 || sb->start % w != 0) continue;
    int ok = 1;
    for (int64_t i = 1; i < sb->ndims; ++i)
      if (sb->strides[i] % w != 0) {
        ok = 0;
        break;
      }
    if (ok) return w;
  }
  return 1;
}

static int64_t pow2_at_least(int64_t v) {
  uint64_t x = 1;
  while (x < (uint64_t)v) x <<= 1;
  return (int64_t)x;
}

/* make_plan: plan.hpp:77-99 */
static void make_plan(const sb_t *sb, or_commit_info *out) {
  out->word = select_word_size(sb);
  const int64_t ext[3] = {sb->counts[0] / out->word,
                          sb->ndims > 1 ? sb->counts[1] : 1,
                          sb->ndims > 2 ? sb->counts[2] : 1};
  int64_t budget = 1024;
  for (int d = 0; d < 3; ++d) {
    int64_t b = pow2_at_least(ext[d]);
    if (b > budget) b = budget;
    out->block[d] = b;
    budget /= b;
    out->grid[d] = (ext[d] + b - 1) / b;
  }
  out->strategy = sb->ndims <= 2 ? 0 : 1;
}

/* ------------------------------------------------------------------ */
/* commit (commit.hpp:51-79)                                            */
/* ------------------------------------------------------------------ */

typedef struct {
  or_commit_info info;
  sb_t sb;
  blkvec_t fallback; /* definition-order runs, unmerged */
} committed_t;

static int commit_def(const def_t *d, committed_t *ct) {
  memset(ct, 0, sizeof(*ct));
  or_commit_info *o = &ct->info;
  o->size = type_size(d);
  o->extent = type_extent(d);
  o->simplify_rounds = -1;
  {
    blkvec_t runs = {0};
    flatten_runs(d, 0, &runs);
    o->overlapping = normalize(&runs);
    o->span = runs.n ? runs.v[runs.n - 1].off + runs.v[runs.n - 1].len : 0;
    free(runs.v);
  }
  if (o->size == 0) {
    o->form = 1;
    return OR_OK;
  }
  chain_t c = {0};
  translate(d, &c);
  int64_t rounds = 0;
  const int st = simplify(&c, &rounds);
  if (st == OR_INTERNAL) {
    free(c.v);
    return OR_INTERNAL;
  }
  if (st == OR_OK && to_strided_block(&c, &ct->sb)) {
    o->form = 0;
    o->simplify_rounds = rounds;
    o->ndims = ct->sb.ndims;
    o->start = ct->sb.start;
    for (int64_t i = 0; i < ct->sb.ndims; ++i) {
      o->counts[i] = ct->sb.counts[i];
      o->strides[i] = ct->sb.strides[i];
    }
    make_plan(&ct->sb, o);
    free(c.v);
    return OR_OK;
  }
  free(c.v);
  o->form = 2;
  flatten_runs(d, 0, &ct->fallback);
  o->n_fallback_runs = ct->fallback.n;
  return OR_OK;
}

int or_size_extent(const int64_t *prog, int64_t n, int64_t *size,
                   int64_t *extent) {
  def_t *d;
  int st = parse_all(prog, n, &d);
  if (st) return st;
  *size = type_size(d);
  *extent = type_extent(d);
  def_free(d);
  return OR_OK;
}

int or_commit(const int64_t *prog, int64_t n, or_commit_info *out) {
  def_t *d;
  int st = parse_all(prog, n, &d);
  if (st) return st;
  committed_t ct;
  st = commit_def(d, &ct);
  def_free(d);
  if (st == OR_OK) *out = ct.info;
  free(ct.fallback.v);
  return st;
}

int or_flatten(const int64_t *prog, int64_t n, int64_t *offsets,
               int64_t *lengths, int64_t cap, int64_t *count,
               int64_t *overlap) {
  def_t *d;
  int st = parse_all(prog, n, &d);
  if (st) return st;
  blkvec_t runs = {0};
  flatten_runs(d, 0, &runs);
  *overlap = normalize(&runs);
  *count = runs.n;
  for (int64_t i = 0; i < runs.n && i < cap; ++i) {
    offsets[i] = runs.v[i].off;
    lengths[i] = runs.v[i].len;
  }
  free(runs.v);
  def_free(d);
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* pack / unpack (pack.hpp:99-185), serial                              */
/* ------------------------------------------------------------------ */

/* run_src_offset: pack.hpp:23-30 (dim 1 fastest) */
static int64_t run_src_offset(const sb_t *sb, int64_t r) {
  int64_t off = sb->start;
  for (int64_t d = 1; d < sb->ndims; ++d) {
    off += (r % sb->counts[d]) * sb->strides[d];
    r /= sb->counts[d];
  }
  return off;
}

static int64_t runs_per_object(const sb_t *sb) {
  int64_t n = 1;
  for (int64_t d = 1; d < sb->ndims; ++d) n *= sb->counts[d];
  return n;
}

static int pack_committed(const committed_t *ct, const uint8_t *src,
                          uint64_t src_len, int64_t incount, uint8_t *dst,
                          uint64_t dst_len, int64_t position,
                          int allow_fallback, int64_t *new_position) {
  const or_commit_info *o = &ct->info;
  if (incount < 1 || position < 0) return OR_INVALID_ARGUMENT; /* :102-104 */
  if (position + incount * o->size > (int64_t)dst_len) return OR_BUFFER_TOO_SMALL;
  if (o->form == 1) {
    *new_position = position;
    return OR_OK;
  }
  if ((incount - 1) * o->extent + o->span > (int64_t)src_len) return OR_BUFFER_TOO_SMALL;
  uint8_t *out = dst + position;
  if (o->form == 0) {
    /* walk_words: pack.hpp:47-60 with the plan's word as granularity */
    const sb_t *sb = &ct->sb;
    const int64_t runs = runs_per_object(sb);
    const int64_t total = incount * runs, rb = sb->counts[0];
    for (int64_t g = 0; g < total; ++g) {
      const int64_t obj = g / runs, run = g % runs;
      const int64_t s = obj * o->extent + run_src_offset(sb, run);
      const int64_t dd = obj * o->size + run * rb;
      for (int64_t w = 0; w < rb; w += o->word) memcpy(out + dd + w, src + s + w, (size_t)o->word);
    }
  } else {
    if (!allow_fallback) return OR_UNSUPPORTED;
    for (int64_t j = 0; j < incount; ++j) {
      const uint8_t *base = src + j * o->extent;
      for (int64_t k = 0; k < ct->fallback.n; ++k) {
        memcpy(out, base + ct->fallback.v[k].off, (size_t)ct->fallback.v[k].len);
        out += ct->fallback.v[k].len;
      }
    }
  }
  *new_position = position + incount * o->size;
  return OR_OK;
}

static int unpack_committed(const committed_t *ct, const uint8_t *src,
                            uint64_t src_len, int64_t position,
                            int64_t outcount, uint8_t *dst, uint64_t dst_len,
                            int allow_fallback, int64_t *new_position) {
  const or_commit_info *o = &ct->info;
  if (outcount < 1 || position < 0) return OR_INVALID_ARGUMENT; /* :146-148 */
  if (o->overlapping) return OR_OVERLAPPING_LAYOUT;               /* :149-151 */
  if (position + outcount * o->size > (int64_t)src_len) return OR_BUFFER_TOO_SMALL;
  if (o->form == 1) {
    *new_position = position;
    return OR_OK;
  }
  if ((outcount - 1) * o->extent + o->span > (int64_t)dst_len) return OR_BUFFER_TOO_SMALL;
  const uint8_t *in = src + position;
  if (o->form == 0) {
    const sb_t *sb = &ct->sb;
    const int64_t runs = runs_per_object(sb);
    const int64_t total = outcount * runs, rb = sb->counts[0];
    for (int64_t g = 0; g < total; ++g) {
      const int64_t obj = g / runs, run = g % runs;
      const int64_t s = obj * o->size + run * rb;
      const int64_t dd = obj * o->extent + run_src_offset(sb, run);
      for (int64_t w = 0; w < rb; w += o->word) memcpy(dst + dd + w, in + s + w, (size_t)o->word);
    }
  } else {
    if (!allow_fallback) return OR_UNSUPPORTED;
    for (int64_t j = 0; j < outcount; ++j) {
      uint8_t *base = dst + j * o->extent;
      for (int64_t k = 0; k < ct->fallback.n; ++k) {
        memcpy(base + ct->fallback.v[k].off, in, (size_t)ct->fallback.v[k].len);
        in += ct->fallback.v[k].len;
      }
    }
  }
  *new_position = position + outcount * o->size;
  return OR_OK;
}

void *or_commit_handle(const int64_t *prog, int64_t n, int *status) {
  def_t *d;
  *status = parse_all(prog, n, &d);
  if (*status) return NULL;
  committed_t *ct = (committed_t *)malloc(sizeof(committed_t));
  *status = commit_def(d, ct);
  def_free(d);
  if (*status) {
    free(ct->fallback.v);
    free(ct);
    return NULL;
  }
  return ct;
}

void or_free_handle(void *h) {
  committed_t *ct = (committed_t *)h;
  if (!ct) return;
  free(ct->fallback.v);
  free(ct);
}

int or_pack_h(void *h, const uint8_t *src, uint64_t src_len, int64_t incount,
              uint8_t *dst, uint64_t dst_len, int64_t position,
              int64_t *new_position) {
  return pack_committed((const committed_t *)h, src, src_len, incount, dst,
                        dst_len, position, 1, new_position);
}

int or_unpack_h(void *h, const uint8_t *src, uint64_t src_len,
                int64_t position, int64_t outcount, uint8_t *dst,
                uint64_t dst_len, int64_t *new_position) {
  return unpack_committed((const committed_t *)h, src, src_len, position,
                          outcount, dst, dst_len, 1, new_position);
}

int or_pack(const int64_t *prog, int64_t n, const uint8_t *src,
            uint64_t src_len, int64_t incount, uint8_t *dst, uint64_t dst_len,
            int64_t position, int allow_fallback, int64_t *new_position) {
  int st;
  committed_t *ct = (committed_t *)or_commit_handle(prog, n, &st);
  if (!ct) return st;
  st = pack_committed(ct, src, src_len, incount, dst, dst_len, position,
                      allow_fallback, new_position);
  or_free_handle(ct);
  return st;
}

int or_unpack(const int64_t *prog, int64_t n, const uint8_t *src,
              uint64_t src_len, int64_t position, int64_t outcount,
              uint8_t *dst, uint64_t dst_len, int allow_fallback,
              int64_t *new_position) {
  int st;
  committed_t *ct = (committed_t *)or_commit_handle(prog, n, &st);
  if (!ct) return st;
  st = unpack_committed(ct, src, src_len, position, outcount, dst, dst_len,
                        allow_fallback, new_position);
  or_free_handle(ct);
  return st;
}
