"""The drop-in MPI surface (include/mpi.h, libtempi_b200.so): C programs
written against mpi.h, launched with tools/tempirun.py. CPU: datatype
construction/queries/topologies across 2-3 ranks. GPU: MPI_Pack/Unpack and
Send/Recv with every transfer method (bit-exact on the host), and the
paper's halo exchange (MPI_Pack x26 + MPI_Neighbor_alltoallv +
MPI_Unpack x26) verified with the reference's fill pattern at 1-8 ranks."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2012_14363_b200")
NATIVE = os.path.join(ROOT, "tests", "native")


def build(tmp_path, name):
    exe = str(tmp_path / name)
    subprocess.run(["/usr/bin/gcc", "-O2", "-Wall", "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include",
                    os.path.join(NATIVE, name + ".c"), "-o", exe, "-L" + PKG, "-ltempi_b200",
                    "-lstridepack_b200", "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath," + PKG],
                   check=True)
    return exe


@pytest.mark.gpu
def test_capi_from_c(cuda, tmp_path):
    """the engine's C-ABI driven from plain C: pack, unpack, typed copy, errors"""
    p = subprocess.run([build(tmp_path, "capi_pack")], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0 and "OK" in p.stdout, p.stdout + p.stderr


def test_capi_c_program_compiles(tmp_path):
    """CPU: the C program builds against include/stridepack_b200.h"""
    assert os.path.exists(build(tmp_path, "capi_pack"))


def run(np_, *cmd, timeout=300):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "tempirun.py"), "-n", str(np_),
                        "--timeout", str(timeout)] + list(cmd), capture_output=True, text=True,
                       timeout=timeout + 30)
    assert p.returncode == 0, p.stdout + p.stderr
    return p.stdout


def test_library_exports_mpi_header(sp):
    from test_abi import dynamic_symbols, header_symbols
    exported = dynamic_symbols(os.path.join(PKG, "libtempi_b200.so"))
    declared = header_symbols("mpi.h")
    assert len(declared) > 40
    assert not [s for s in declared if s not in exported]


@pytest.mark.parametrize("np_", [1, 2, 3])
def test_mpi_types_and_topology(tmp_path, np_):
    assert "OK" in run(np_, build(tmp_path, "mpi_types"))


@pytest.mark.gpu
@pytest.mark.parametrize("np_", [1, 2])
def test_mpi_indexed_struct_resized(cuda, tmp_path, np_):
    """beyond the reference: irregular MPI_Type_indexed and a resized struct
    through MPI_Pack/Unpack on device memory and Send/Recv (every method)"""
    assert "OK" in run(np_, build(tmp_path, "mpi_indexed"))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["a", "b", "ab"])
@pytest.mark.parametrize("np_", [1, 2, 3])
def test_mpi_unstructured_neighbor_exchange(cuda, tmp_path, np_, mode):
    """beyond the reference: irregular gather lists into contiguous ghosts
    (mode "a"), contiguous runs scattered into irregular ghost slots through
    the receivers' IPC-published run tables (mode "b"), and both in one
    process (mode "ab": the sequence that used to leave ghosts unwritten)"""
    assert "OK" in run(np_, build(tmp_path, "mpi_unstructured"), mode)


@pytest.mark.gpu
@pytest.mark.parametrize("np_", [2, 3])
def test_mpi_unstructured_loop(cuda, tmp_path, np_):
    """100 iterations of mode "ab", each with FRESH types (new run tables
    uploaded, published and copied) and fresh buffers: the regression for
    the irregular-receive failure, whose cause was a run-table upload that
    could still be in flight when the table was published or read
    (csrc/pack.cu copy_sync)"""
    assert "OK" in run(np_, build(tmp_path, "mpi_unstructured"), "ab", "100", timeout=600)


@pytest.mark.gpu
@pytest.mark.parametrize("np_", [1, 2])
def test_mpi_portable_program(cuda, tmp_path, np_):
    """tests/native/mpi_interpose.c -- the portable program the interposer is
    tested with over a system MPI -- on the engine's own MPI: device
    pack/unpack checked against host pack/unpack, every send method, the
    set completions (Waitany, Waitsome, Testall, Testany, Request_free)"""
    assert "OK" in run(np_, build(tmp_path, "mpi_interpose"))


@pytest.mark.gpu
@pytest.mark.parametrize("np_", [1, 2, 3])
def test_mpi_alltoallv_alltoallw(cuda, tmp_path, np_):
    """beyond the paper (its future work names collectives): MPI_Alltoallv
    and MPI_Alltoallw with strided send or receive types, per-peer types,
    over the neighbour typed-copy machinery on the complete graph"""
    assert "OK" in run(np_, build(tmp_path, "mpi_alltoall"))


@pytest.mark.gpu
@pytest.mark.parametrize("np_", [1, 2])
def test_mpi_pack_and_sendrecv(cuda, tmp_path, np_):
    assert "OK" in run(np_, build(tmp_path, "mpi_sendrecv"))


@pytest.mark.gpu
@pytest.mark.parametrize("np_", [1, 2, 3])
def test_mpi_nonblocking_ring(cuda, tmp_path, np_):
    """MPI_Isend/Irecv/Test/Waitall/Sendrecv, every method, chunked messages"""
    os.environ["TEMPI_CHUNK"] = str(64 << 10)  # pipeline the 600-960 KiB messages in 64 KiB chunks
    try:
        assert "OK" in run(np_, build(tmp_path, "mpi_isend"))
    finally:
        del os.environ["TEMPI_CHUNK"]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1, 2, 3])
@pytest.mark.parametrize("grid", [(1, 1, 1), (2, 1, 1), (2, 2, 1), (2, 2, 2)])
def test_mpi_halo_exchange(cuda, tmp_path, grid, mode):
    """mode 0: MPI_Pack x26 + MPI_Neighbor_alltoallv + MPI_Unpack x26;
    mode 1: one MPI_Neighbor_alltoallw with the 26 region types;
    mode 2: the same as an MPI-4 persistent collective
    (MPI_Neighbor_alltoallw_init, MPI_Start + MPI_Wait per iteration);
    mode 3: mode 0 with a persistent MPI_Neighbor_alltoallv_init"""
    exe = build(tmp_path, "mpi_halo")
    out = run(grid[0] * grid[1] * grid[2], exe, *map(str, grid), "12", "2", "16", "3", str(mode))
    assert "OK" in out
