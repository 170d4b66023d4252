"""Build libdecdec.so (sm_100a) in-tree with nvcc.  `python paper_2412_20185_b200/build.py` (running it as
`-m paper_2412_20185_b200.build` would import the package, i.e. load the old library, first)."""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libdecdec.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    cmd = [
        nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
        "-cudart", "shared", "-I", os.path.join(ROOT, "include"), "-I", CSRC, *os.environ.get("DECDEC_NVCC_EXTRA", "").split(),
        "-Xptxas", "-v" if verbose else "-O3",
        "-o", LIB + ".tmp", *sources(), "-ldl",
    ]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libdecdec.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_probe() -> str:
    out = os.path.join(ROOT, "build", "probe")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.run([nvcc(), *ARCH, "-O3", "-lineinfo", "-o", out, os.path.join(CSRC, "probe", "probe.cu")], check=True)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
