"""Shared test setup.

* registers the ``gpu`` marker (tests needing a B200 / CUDA device);
* makes sure the engine library and the oracle library are built (nvcc and
  gcc are available in the build container and on the GPU box);
* loads the golden fixtures produced by tests/golden/make_golden.py.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: large parity case")


def _ensure_built():
    lib = os.path.join(REPO, "paper_2208_11469_b200", "_lib", "libprobgraph_b200.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C",
                        os.path.join(REPO, "paper_2208_11469_b200", "csrc")],
                       check=True)
    olib = os.path.join(REPO, "oracle", "_build", "libpgoracle.so")
    if not os.path.exists(olib):
        subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle")], check=True)


_ensure_built()


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="needs a CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def small_golden():
    with np.load(os.path.join(GOLDEN, "small_cases.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def hash_kat():
    with open(os.path.join(GOLDEN, "hash_kat.json")) as fh:
        return json.load(fh)


def load_config(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"fixture {name} not generated")
    with open(path) as fh:
        return json.load(fh)


SMALL_NAMES = ["g60", "g80", "g200", "dense120", "sparse300"]
SMALL_SEEDS = {"g60": 4, "g80": 6, "g200": 42, "dense120": 7, "sparse300": 11}
BLOOM_PARAMS = [(64, 1), (128, 2), (512, 1), (576, 3), (1024, 2), (2048, 2)]
KS = [1, 4, 5, 32, 64]


def small_graph(golden, name):
    from paper_2208_11469_b200 import CsrGraph
    return CsrGraph(golden[f"{name}/offsets"], golden[f"{name}/adjacency"])


def sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
