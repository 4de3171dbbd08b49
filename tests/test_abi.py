"""The drop-in boundary: libstridepack_b200.so loads without a GPU and exports
every symbol include/*.h declares; compute calls fail loudly (NoDevice) when
there is no device instead of falling back to the host. CPU only."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols(name):
    src = open(os.path.join(ROOT, "include", name)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"//[^\n]*", "", src)
    src = re.sub(r"^\s*#[^\n]*", "", src, flags=re.M)
    return sorted(set(re.findall(r"\b((?:sp|MPI|PMPI)_[A-Za-z0-9_]+)\s*\(", src)))


def dynamic_symbols(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def test_library_exports_every_declared_symbol(sp):
    from paper_2012_14363_b200 import _capi
    exported = dynamic_symbols(_capi.LIB_PATH)
    declared = header_symbols("stridepack_b200.h")
    assert len(declared) >= 15
    missing = [s for s in declared if s not in exported]
    assert not missing, missing


def test_library_has_sm100a_code(sp):
    from paper_2012_14363_b200 import _capi
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_compute_without_device_is_an_error(sp):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    ct = sp.commit_type(sp.make_vector(3, 4, 8, sp.make_named(sp.NamedKind.Float)))
    import numpy as np
    src = np.arange(96, dtype=np.uint8)
    dst = np.zeros(48, np.uint8)
    with pytest.raises(sp.NoDevice):
        sp.pack(src, ct, 1, dst, 0)
    # host-side validation still precedes the device check (pack.hpp:102-106)
    with pytest.raises(sp.BufferTooSmall):
        sp.pack(src, ct, 1, np.zeros(47, np.uint8), 0)
    with pytest.raises(sp.InvalidArgument):
        sp.pack(src, ct, 0, dst, 0)
