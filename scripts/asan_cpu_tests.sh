# CPU test suite against the AddressSanitizer + UBSan build of the engine's
# host code (types, canonicalisation, commit, model, profile I/O, type files,
# runtime control plane). Device kernels are not instrumented here; they are
# checked with compute-sanitizer (scripts/gpu_sanitize*.sh). The warm-cache
# speed assertion is deselected: timing under an instrumented allocator
# says nothing about the engine.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
make -s -C "$ROOT/paper_2012_14363_b200/csrc" asan
export SPB_LIB="$ROOT/paper_2012_14363_b200/asan/libstridepack_b200.so"
export ASAN_OPTIONS=detect_leaks=0:abort_on_error=1:halt_on_error=1
export UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1
LD_PRELOAD=$(gcc -print-file-name=libasan.so):$(gcc -print-file-name=libubsan.so) \
  python -m pytest "$ROOT/tests" -q -m "not gpu" -x -p no:cacheprovider \
  --deselect tests/test_mpi.py --deselect tests/test_model.py::test_warm_cache_speedup_native "$@"
