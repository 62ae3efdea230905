"""Build libkkt.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libkkt.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = ["-shared", "-Xcompiler", "-fPIC", "-O3", "-std=c++17",
              "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-Xptxas", "-v"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cpp")) + glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "kkt.h")]


def build_variant(out: str, defines: list[str]) -> str:
    """Tuning experiments: the same sources with extra -D flags into another in-tree .so."""
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc] + NVCC_FLAGS + ["-D" + d for d in defines] + sources() + ["-o", out]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(SO):
        t = os.path.getmtime(SO)
        if all(os.path.getmtime(d) <= t for d in deps()):
            return SO
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = SO + ".tmp%d" % os.getpid()
    cmd = [nvcc] + NVCC_FLAGS + sources() + ["-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    with open(os.path.join(HERE, "ptxas_report.txt"), "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stderr)
    os.replace(tmp, SO)
    if verbose:
        print(res.stderr)
    return SO


if __name__ == "__main__":
    print(build(force=True))
