"""TEMPI as a PMPI interposer over a system MPI:
paper_2012_14363_b200/libtempi_interpose.so in front of tests/native/minimpi.c,
a small CUDA-aware MPI standing in for the system library (the image ships
none). Programs are plain MPI sources; the interposer is put in front either
by LD_PRELOAD under an unmodified binary linked only to the system MPI, or by
link order (-ltempi_interpose -lminimpi).

CPU: the library's symbol surface (MPI_* only, no PMPI_*, no link-time MPI
dependency), and forwarding of host-memory work at 1-3 ranks. GPU: device
pack/unpack and every send method checked against the SYSTEM MPI's own host
pack/unpack of the same bytes, the paper's halo exchange through both
neighbour collectives verified with the reference's fill pattern, and the
same programs over the system MPI alone (the baseline the interposer
replaces)."""
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2012_14363_b200")
NATIVE = os.path.join(ROOT, "tests", "native")
INTERPOSE = os.path.join(PKG, "libtempi_interpose.so")
CUDA_LIB = "/usr/local/cuda/lib64"
CC = ["/usr/bin/gcc", "-O2", "-Wall", "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include"]

# what TEMPI intercepts (interpose.cpp); everything else is the system MPI's
INTERCEPTED = {
    "MPI_Init", "MPI_Init_thread", "MPI_Finalize",
    "MPI_Type_contiguous", "MPI_Type_vector", "MPI_Type_create_hvector", "MPI_Type_create_subarray",
    "MPI_Type_indexed", "MPI_Type_create_hindexed", "MPI_Type_create_indexed_block",
    "MPI_Type_create_hindexed_block", "MPI_Type_create_struct", "MPI_Type_create_resized",
    "MPI_Type_commit", "MPI_Type_free", "MPI_Pack", "MPI_Unpack",
    "MPI_Send", "MPI_Recv", "MPI_Isend", "MPI_Irecv", "MPI_Wait", "MPI_Waitall", "MPI_Test", "MPI_Sendrecv",
    "MPI_Waitany", "MPI_Waitsome", "MPI_Testany", "MPI_Testall", "MPI_Request_free",
    "MPI_Send_init", "MPI_Recv_init", "MPI_Start", "MPI_Startall", "MPI_Neighbor_alltoallw_init",
    "MPI_Neighbor_alltoallv_init",
    "MPI_Dist_graph_create_adjacent", "MPI_Cart_create", "MPI_Comm_free",
    "MPI_Neighbor_alltoallv", "MPI_Neighbor_alltoallw", "MPI_Alltoallv", "MPI_Alltoallw",
}


@pytest.fixture(scope="module")
def sysmpi(tmp_path_factory):
    """libminimpi.so, the stand-in system MPI"""
    d = tmp_path_factory.mktemp("sysmpi")
    lib = str(d / "libminimpi.so")
    subprocess.run(CC + ["-fPIC", "-shared", "-pthread", os.path.join(NATIVE, "minimpi.c"), "-o", lib,
                         "-L" + CUDA_LIB, "-lcudart", "-Wl,-rpath," + CUDA_LIB], check=True)
    return str(d)


def build(sysmpi, name, interposed):
    """name.c linked to the system MPI, with the interposer first when asked"""
    exe = os.path.join(sysmpi, name + ("_tempi" if interposed else "_plain"))
    libs = (["-L" + PKG, "-ltempi_interpose"] if interposed else []) + \
        ["-L" + sysmpi, "-lminimpi", "-L" + PKG, "-lstridepack_b200", "-L" + CUDA_LIB, "-lcudart",
         "-Wl,-rpath," + sysmpi, "-Wl,-rpath," + PKG, "-Wl,-rpath," + CUDA_LIB]
    subprocess.run(CC + [os.path.join(NATIVE, name + ".c"), "-o", exe] + libs, check=True)
    return exe


def run(np_, exe, *args, preload=False, env=None, timeout=300):
    e = dict(os.environ, TEMPI_INTERPOSE_STATS="1", **(env or {}))
    if preload:
        e["LD_PRELOAD"] = INTERPOSE
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "tempirun.py"), "-n", str(np_),
                        "--timeout", str(timeout), exe] + list(args), capture_output=True, text=True,
                       timeout=timeout + 30, env=e)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "OK" in p.stdout, p.stdout + p.stderr
    return p.stdout, stats(p.stderr)


def stats(stderr):
    """per-rank counters the interposer prints at MPI_Finalize"""
    out = {}
    for m in re.finditer(r"tempi-interpose rank (\d+): commits (\d+) packs (\d+) unpacks (\d+) "
                         r"sends\(oneshot/device/staged\) (\d+)/(\d+)/(\d+) recvs (\d+)/(\d+)/(\d+) "
                         r"exchanges (\d+) forwarded (\d+) kernels (\d+)", stderr):
        v = list(map(int, m.groups()))
        out[v[0]] = dict(commits=v[1], packs=v[2], unpacks=v[3], sends=v[4:7], recvs=v[7:10], exchanges=v[10],
                         forwarded=v[11], kernels=v[12])
    return out


def dynamic(path, defined=True):
    out = subprocess.run(["nm", "-D", "--defined-only" if defined else "--undefined-only", path],
                         capture_output=True, text=True, check=True).stdout
    return {ln.split()[-1] for ln in out.splitlines() if ln.strip()}


# ----------------------------------------------------------------- CPU
def test_interposer_symbol_surface(sp):
    """MPI_* for exactly the accelerated calls, no PMPI_* (the system MPI's),
    no link-time dependency on any MPI library (dlsym(RTLD_NEXT))"""
    exported = {s for s in dynamic(INTERPOSE) if s.startswith("MPI_")}
    assert exported == INTERCEPTED
    assert not [s for s in dynamic(INTERPOSE) if s.startswith("PMPI_")]
    assert not [s for s in dynamic(INTERPOSE, defined=False) if "MPI_" in s]
    needed = subprocess.run(["readelf", "-d", INTERPOSE], capture_output=True, text=True, check=True).stdout
    assert "mpi" not in " ".join(re.findall(r"Shared library: \[(.*?)\]", needed)).lower()
    assert [s for s in dynamic(INTERPOSE, defined=False) if s.split("@")[0] == "dlsym"]


def test_system_mpi_stand_in_is_complete(sysmpi):
    """every intercepted MPI_* has a PMPI_* in the stand-in system MPI"""
    pm = {s for s in dynamic(os.path.join(sysmpi, "libminimpi.so")) if s.startswith("PMPI_")}
    assert not [s for s in INTERCEPTED if "P" + s not in pm]


@pytest.mark.parametrize("np_", [1, 2, 3])
def test_forwarding_host_memory(sysmpi, np_):
    """host buffers: every call forwarded, results equal the system MPI's;
    the 5 engine-representable types are mirrored and committed, the
    hindexed with a negative displacement is left to the system MPI"""
    exe = build(sysmpi, "mpi_interpose", interposed=False)
    _, none = run(np_, exe)
    assert none == {}
    _, st = run(np_, exe, preload=True)
    assert sorted(st) == list(range(np_))
    for r in st.values():
        assert r["commits"] == 5 and r["packs"] == 0 and r["unpacks"] == 0 and r["forwarded"] >= 12
    _, st2 = run(np_, build(sysmpi, "mpi_interpose", interposed=True))
    assert st2 == st


# ----------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("np_", [1, 2])
@pytest.mark.parametrize("how", ["preload", "linked"])
def test_interposed_device_paths(cuda, sysmpi, np_, how):
    """device MPI_Pack/Unpack and Send/Recv/Isend/Irecv/Sendrecv of six
    derived types, every method: bytes equal the system MPI's host
    pack/unpack of the same data"""
    exe = build(sysmpi, "mpi_interpose", interposed=how == "linked")
    _, st = run(np_, exe, preload=how == "preload")
    for r, s in st.items():
        assert s["kernels"] > 0 and s["packs"] >= 5 * 2 and s["unpacks"] >= 5
        if np_ >= 2 and r == 0:
            assert all(n > 0 for n in s["sends"])  # one-shot, device and staged all ran
        if np_ >= 2 and r == 1:
            assert all(n > 0 for n in s["recvs"])


@pytest.mark.gpu
def test_system_mpi_alone_device(cuda, sysmpi):
    """the baseline: the same program on the system MPI's per-run copies"""
    run(2, build(sysmpi, "mpi_interpose", interposed=False))


@pytest.mark.gpu
def test_interposed_not_cuda_aware(cuda, sysmpi):
    """TEMPI_CUDA_AWARE=0: packed messages staged through pinned memory"""
    exe = build(sysmpi, "mpi_interpose", interposed=False)
    _, st = run(2, exe, preload=True, env={"TEMPI_CUDA_AWARE": "0"})
    assert st[0]["sends"][1] == 0  # no device-resident message handed to the system MPI


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1, 2, 3])
@pytest.mark.parametrize("grid", [(1, 1, 1), (2, 1, 1), (2, 2, 1)])
def test_interposed_halo_exchange(cuda, sysmpi, grid, mode):
    """the paper's halo exchange, unmodified source: mode 0 = MPI_Pack x26
    (interposer kernels) + MPI_Neighbor_alltoallv of MPI_PACKED (forwarded) +
    MPI_Unpack x26; mode 1 = one MPI_Neighbor_alltoallw of the 26 region
    types (one batched pack launch, the system MPI's byte exchange, one
    batched unpack launch); mode 2 = the same as an MPI-4 persistent
    collective (MPI_Neighbor_alltoallw_init, MPI_Start + MPI_Wait); every
    ghost cell verified"""
    exe = build(sysmpi, "mpi_halo", interposed=False)
    n = grid[0] * grid[1] * grid[2]
    _, st = run(n, exe, *map(str, grid), "12", "2", "16", "3", str(mode), preload=True)
    for s in st.values():  # 3 iterations
        assert s["packs"] == 26 * 3 and s["unpacks"] == 26 * 3 and s["kernels"] > 0
        assert s["exchanges"] == (3 if mode == 1 else 0)


@pytest.mark.gpu
@pytest.mark.parametrize("np_", [2, 3])
def test_interposed_nonblocking_ring(cuda, sysmpi, np_):
    """tests/native/mpi_isend.c unchanged (written for the engine's own MPI):
    a ring of Irecv/Isend of 3-D subarrays with every forced method, MPI_Test
    polling, MPI_Waitall, MPI_Sendrecv, over the system MPI"""
    _, st = run(np_, build(sysmpi, "mpi_isend", interposed=True))
    for s in st.values():
        assert s["packs"] > 0 and s["unpacks"] > 0 and s["kernels"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["a", "b", "ab"])
def test_interposed_unstructured_exchange(cuda, sysmpi, mode):
    """tests/native/mpi_unstructured.c unchanged: irregular MPI_Type_indexed
    gather lists and scattered ghost layouts through MPI_Neighbor_alltoallw
    (block-list forms: one pack or unpack call per segment) over the system MPI"""
    _, st = run(2, build(sysmpi, "mpi_unstructured", interposed=False), mode, "3", preload=True)
    for s in st.values():
        assert s["exchanges"] >= 3 and s["kernels"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("np_", [1, 2, 3])
def test_interposed_alltoall(cuda, sysmpi, np_):
    """tests/native/mpi_alltoall.c unchanged over the system MPI: MPI_Alltoallv
    and MPI_Alltoallw with strided device types, one batched pack and unpack
    launch around the system MPI's byte all-to-all"""
    _, st = run(np_, build(sysmpi, "mpi_alltoall", interposed=False), preload=True)
    for s in st.values():
        assert s["exchanges"] == 3 and s["kernels"] > 0


def test_interposer_builds_against_pointer_handle_mpi_h():
    """a site rebuilds interpose.cpp against its own MPI's mpi.h: it compiles
    against an Open MPI-style header (opaque pointer handles, predefined
    datatypes as object addresses, a standard MPI_Status without this
    image's extra fields; tests/native/ompi_style/mpi.h)"""
    p = subprocess.run(["/usr/bin/g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror",
                        "-Wno-unused-parameter", "-I" + os.path.join(NATIVE, "ompi_style"),
                        "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include",
                        os.path.join(PKG, "csrc", "interpose.cpp")], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
