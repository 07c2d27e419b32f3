import json
import os
import pathlib
import subprocess
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
GOLD = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU oracle checks")
    # a fresh checkout has no built artefacts (they are git-ignored): build
    # the in-tree library and host encoder before anything imports them
    from paper_2011_14486_b200 import build as _build
    try:
        _build.build()
    except Exception as e:  # e.g. no nvcc on this host: the tests that need it report it
        sys.stderr.write(f"conftest: native build skipped ({e})\n")


@pytest.fixture(scope="session")
def golden():
    return GOLD


@pytest.fixture(scope="session")
def greedy_golden():
    return json.loads((GOLD / "greedy.json").read_text())


@pytest.fixture(scope="session")
def noisy_golden():
    return json.loads((GOLD / "noisy.json").read_text())


@pytest.fixture(scope="session")
def candidates_golden():
    return json.loads((GOLD / "candidates.json").read_text())


def load_states_file(path):
    z = np.load(path)
    return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def state_sets():
    """name -> dict(keys, features, values, seeds, source, text)."""
    out = {}
    for f in sorted(GOLD.glob("states_*.npz")):
        out[f.stem[len("states_"):]] = load_states_file(f)
    return out


@pytest.fixture(scope="session")
def v0_path():
    return GOLD / "v0.ckpt"


@pytest.fixture(scope="session")
def native_core():
    """Host build of csrc/ts_core.cuh (test harness, tests/native)."""
    import ctypes
    src = ROOT / "tests" / "native" / "core_host.cpp"
    so = ROOT / "tests" / "native" / "libcore_host.so"
    deps = [src, ROOT / "paper_2011_14486_b200" / "csrc" / "ts_core.cuh",
            ROOT / "paper_2011_14486_b200" / "csrc" / "ts_glibc_math.cuh"]
    if not so.exists() or any(d.stat().st_mtime > so.stat().st_mtime for d in deps):
        subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-shared",
                        "-o", str(so), str(src)], check=True)
    lib = ctypes.CDLL(str(so))
    vp = ctypes.c_void_p
    lib.core_log2.restype = ctypes.c_double
    lib.core_log2.argtypes = [ctypes.c_double]
    lib.core_div.restype = ctypes.c_double
    lib.core_div.argtypes = [vp, ctypes.c_uint64]
    lib.core_to_double.restype = ctypes.c_double
    lib.core_to_double.argtypes = [vp]
    lib.core_featurize.argtypes = [vp, ctypes.c_int64, vp, vp, ctypes.c_int64, vp]
    lib.core_div128.restype = ctypes.c_double
    lib.core_div128.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
    lib.core_log2_1p.restype = ctypes.c_double
    lib.core_log2_1p.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    lib.core_exp_tanh.argtypes = [vp, ctypes.c_int64, vp]
    lib.core_tanh_bf.argtypes = [vp, ctypes.c_int64, vp]
    return lib


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_2011_14486_b200 import _lib
    return _lib.context(0)
