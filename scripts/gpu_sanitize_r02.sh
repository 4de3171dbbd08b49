#!/bin/bash
# round 2: compute-sanitizer over the irregular-receive MPI program (mode ab,
# fresh types every iteration, 2 ranks) and the alternating-layout
# neighbour regression (3 processes)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
PKG=paper_2012_14363_b200
gcc -O2 -Iinclude -I/usr/local/cuda/include tests/native/mpi_unstructured.c -o /tmp/mpi_unstructured \
  -L$PKG -ltempi_b200 -lstridepack_b200 -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/$PKG
for tool in memcheck racecheck synccheck; do
  timeout 700 python tools/tempirun.py -n 2 --timeout 600 $CS --tool $tool --error-exitcode 86 --print-limit 20 \
    /tmp/mpi_unstructured ab 5 > gpurun_out/r02_${tool}_unstructured_ab.log 2>&1
  echo "rc=$?" >> gpurun_out/r02_${tool}_unstructured_ab.log
done
cat > /tmp/alt.py <<'PY'
import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import test_rt
res = test_rt._spawn(test_rt._nbr_alternating_layouts, 3, 60, timeout=1200)
print(res); assert all(b == 0 for b, _ in res.values())
print("OK")
PY
timeout 900 $CS --tool memcheck --target-processes all --error-exitcode 86 --print-limit 20 python /tmp/alt.py \
  > gpurun_out/r02_memcheck_alternating.log 2>&1
echo "rc=$?" >> gpurun_out/r02_memcheck_alternating.log
for f in gpurun_out/r02_*check_*.log; do echo "== $f"; tail -n 4 $f; done
