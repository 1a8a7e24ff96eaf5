"""Build libgcr.so (the product) and libgcr_synth.so (harness generator) in
tree with nvcc for sm_100a.  Called by __graft_entry__.build(); runs on a CPU
box (nvcc cross-compiles)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

LIBS = {
    "libgcr.so": (
        [os.path.join(CSRC, f) for f in ("kernels.cu", "codec.cu", "gcr.cpp", "crc_host.cpp")],
        [os.path.join(CSRC, "gcr_internal.h"), os.path.join(INCLUDE, "gcr.h")],
    ),
    "libgcr_synth.so": (
        [os.path.join(CSRC, "synth", "synth.cu")],
        [os.path.join(INCLUDE, "gcr_synth.h")],
    ),
}


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> dict:
    outs = {}
    for name, (srcs, hdrs) in LIBS.items():
        out = os.path.join(PKG, name)
        outs[name] = out
        if not force and not _stale(out, srcs + hdrs + [__file__]):
            continue
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-msse4.2,-O2",
               "-I", INCLUDE, "-o", out + ".tmp", *srcs]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed for {name}")
        if verbose:
            sys.stderr.write(r.stderr)
        os.replace(out + ".tmp", out)
    return outs


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
