# the paper-style MPI halo program at one rank, 256^3, r=2, 32 B: alltoallw form and MPI_Pack x26 + alltoallv + MPI_Unpack x26 form
gcc -O2 -Iinclude -I/usr/local/cuda/include tests/native/mpi_halo.c -o /tmp/mpi_halo -Lpaper_2012_14363_b200 -ltempi_b200 -lstridepack_b200 -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2012_14363_b200
for m in 1 0; do timeout 120 python tools/tempirun.py -n 1 --timeout 100 /tmp/mpi_halo 1 1 1 256 2 32 20 $m 2>&1 | tail -2; done
