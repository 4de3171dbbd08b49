/* oracle/oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference datatype engine's commit and
 * pack/unpack algorithms (arXiv 2012.14363 "TEMPI", reference tree
 * /root/reference/proj/include/stridepack/). It is the CHECKER for the
 * product's CUDA path: only tests/, bench.py's cpu_baseline / reference legs
 * and __graft_entry__.smoke() may load it. The product library never calls
 * it, and there is no CPU fallback routed through it.
 *
 * Parity of this restatement is pinned against the reference itself
 * (oracle/_ref/libstridepack_ref.so, built from the untouched reference
 * headers by oracle/Makefile) and against golden vectors committed under
 * tests/golden/ (see tests/golden/make_golden.py).
 *
 * Types use the flat int64 "type program" documented in ref_harness.cpp.
 */
#ifndef ORACLE_H
#define ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_MAXD 64

/* status codes (proj/include/stridepack/errors.hpp:8-47) */
enum {
  OR_OK = 0,
  OR_INVALID_ARGUMENT = 1,
  OR_UNSUPPORTED_ORDER = 2,
  OR_INVALID_LAYOUT = 3,
  OR_BUFFER_TOO_SMALL = 4,
  OR_OVERLAPPING_LAYOUT = 5,
  OR_UNSUPPORTED = 6,
  OR_INTERNAL = 9,
  OR_BAD_PROGRAM = 10
};

/* same layout as ref_commit_info in ref_harness.cpp */
typedef struct {
  int64_t form; /* 0 Strided, 1 Empty, 2 Unsupported */
  int64_t size, extent, span, overlapping;
  int64_t ndims, start;
  int64_t counts[OR_MAXD], strides[OR_MAXD];
  int64_t word, block[3], grid[3], strategy;
  int64_t n_fallback_runs;
  int64_t simplify_rounds;
} or_commit_info;

int or_size_extent(const int64_t *prog, int64_t n, int64_t *size,
                   int64_t *extent);
int or_commit(const int64_t *prog, int64_t n, or_commit_info *out);
int or_flatten(const int64_t *prog, int64_t n, int64_t *offsets,
               int64_t *lengths, int64_t cap, int64_t *count,
               int64_t *overlap);
int or_pack(const int64_t *prog, int64_t n, const uint8_t *src,
            uint64_t src_len, int64_t incount, uint8_t *dst, uint64_t dst_len,
            int64_t position, int allow_fallback, int64_t *new_position);
int or_unpack(const int64_t *prog, int64_t n, const uint8_t *src,
              uint64_t src_len, int64_t position, int64_t outcount,
              uint8_t *dst, uint64_t dst_len, int allow_fallback,
              int64_t *new_position);

/* Committed handle variants so timing loops exclude the commit. */
void *or_commit_handle(const int64_t *prog, int64_t n, int *status);
void or_free_handle(void *h);
int or_pack_h(void *h, const uint8_t *src, uint64_t src_len, int64_t incount,
              uint8_t *dst, uint64_t dst_len, int64_t position,
              int64_t *new_position);
int or_unpack_h(void *h, const uint8_t *src, uint64_t src_len,
                int64_t position, int64_t outcount, uint8_t *dst,
                uint64_t dst_len, int64_t *new_position);

#ifdef __cplusplus
}
#endif
#endif
