"""Shared fixtures.  `-m "not gpu"` tests run anywhere; `-m gpu` tests need a
B200 and exercise the CUDA library through its C ABI."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) device")


def _make(target_dir, *targets):
    subprocess.run(["make", "-s", "-C", target_dir, *targets], check=True,
                   stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref) — outputs ARE the reference's."""
    from oracle.ffi import REF_SO, Ref
    if not os.path.exists(REF_SO):
        _make(os.path.join(ROOT, "oracle"), "reference")
    return Ref()


@pytest.fixture(scope="session")
def orc():
    """The plain-C restatement (oracle/liboracle.so)."""
    from oracle.ffi import ORC_SO, Orc
    if not os.path.exists(ORC_SO):
        _make(os.path.join(ROOT, "oracle"), "restatement")
    return Orc()


@pytest.fixture(scope="session")
def pcp():
    import paper_2603_16945_b200 as P
    if not os.path.exists(os.path.join(ROOT, "paper_2603_16945_b200", "libpcpipe_b200.so")):
        _make(os.path.join(ROOT, "paper_2603_16945_b200"))
    return P


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
