"""Build the sm_100a shared library in-tree (no JIT cache: the .so travels
with the repo snapshot to the GPU box)."""

from __future__ import annotations

import pathlib
import subprocess
import sys

HERE = pathlib.Path(__file__).resolve().parent
CSRC = HERE / "csrc"
OUT = HERE / "libtensched_b200.so"
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-shared",
]


def sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [
        HERE.parent / "include" / "tensched_b200.h"]


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    return any(p.stat().st_mtime > t for p in sources())


def build_hostenc(force: bool = False) -> pathlib.Path:
    """The native host encoder (csrc/hostenc.c, CPython C API) in-tree."""
    import sysconfig
    out = HERE / ("_hostenc" + sysconfig.get_config_var("EXT_SUFFIX"))
    src = CSRC / "hostenc.c"
    if not force and out.exists() and out.stat().st_mtime >= src.stat().st_mtime:
        return out
    cmd = ["gcc", "-O2", "-shared", "-fPIC", "-Wall", "-I", sysconfig.get_paths()["include"], "-o",
           str(out) + ".tmp", str(src)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("gcc failed building _hostenc")
    pathlib.Path(str(out) + ".tmp").replace(out)
    return out


def build(force: bool = False, verbose: bool = False) -> pathlib.Path:
    build_hostenc(force)
    if not force and not needs_build():
        return OUT
    cmd = ["nvcc", *NVCC_FLAGS, "-o", str(OUT) + ".tmp", str(CSRC / "ts_abi.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libtensched_b200.so")
    if verbose:
        sys.stderr.write(res.stderr)
    pathlib.Path(str(OUT) + ".tmp").replace(OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
