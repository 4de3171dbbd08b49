"""Shared fixtures. `-m gpu` tests need a B200 (cuda:0); everything else runs
on CPU. The checkers (oracle/) are imported only here and in the tests."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def sp():
    import paper_2012_14363_b200 as m
    return m


@pytest.fixture(scope="session")
def orc():
    from oracle.pyoracle import oracle
    return oracle()


@pytest.fixture(scope="session")
def ref():
    """the reference compiled in place, or skip when it was never built"""
    from oracle.pyoracle import reference
    r = reference()
    if r is None:
        pytest.skip("oracle/_ref not built")
    return r


@pytest.fixture(scope="session")
def corpus():
    with open(os.path.join(GOLDEN, "corpus.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def pack_digests():
    with open(os.path.join(GOLDEN, "pack_digests.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    return torch
