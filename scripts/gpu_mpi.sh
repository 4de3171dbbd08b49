timeout 1200 python -m pytest tests/test_mpi.py tests/test_rt.py -m gpu -x -q 2>&1 | tail -30 | tee gpurun_out/pytest_mpi.log
mkdir -p /tmp/b && gcc -O2 -Iinclude -I/usr/local/cuda/include tests/native/mpi_halo.c -o /tmp/b/mpi_halo -Lpaper_2012_14363_b200 -ltempi_b200 -lstridepack_b200 -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2012_14363_b200
for g in "1 1 1" "2 1 1" "2 2 1" "2 2 2"; do set -- $g; n=$(( $1 * $2 * $3 )); echo "grid $g"; timeout 300 python tools/tempirun.py -n $n /tmp/b/mpi_halo $1 $2 $3 256 2 32 5; done 2>&1 | tee gpurun_out/mpi_halo.txt
