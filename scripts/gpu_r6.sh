set -o pipefail
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_mpi.py -m gpu -q -x 2>&1 | tail -30 | tee gpurun_out/pytest_mpi.log
gcc -O2 -Iinclude -I/usr/local/cuda/include tests/native/mpi_halo.c -o gpurun_out/mpi_halo_exe -Lpaper_2012_14363_b200 -ltempi_b200 -lstridepack_b200 -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2012_14363_b200
for g in "1 1 1" "2 1 1" "2 2 2"; do for m in 0 1; do timeout 300 python tools/tempirun.py -n $(( $(echo $g | tr ' ' '*') )) --timeout 250 gpurun_out/mpi_halo_exe $g 64 2 32 5 $m 2>&1 | tail -2; done; done | tee gpurun_out/mpi_halo64.txt
