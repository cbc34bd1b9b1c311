"""Build libtdc.so (sm_100a) in-tree with nvcc.  No JIT caches: the .so sits
next to this file so it travels with the repo snapshot to the GPU box."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtdc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.h"))) + \
        sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "tdc.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in _deps())


def build(force: bool = False, verbose: bool = False, timeline: bool = False, knobs: bool = False) -> str:
    """timeline=True builds the debug variant libtdc_tl.so (-DTDC_TIMELINE: per-tile
    %globaltimer events of CTA 0, read by scripts/*timeline.py via TDC_LIB); knobs=True
    builds libtdc_kn.so (-DTDC_DEBUG_KNOBS: the TDC_*_DBG attribution switches, no stamps)."""
    lib = LIB.replace("libtdc.so", "libtdc_tl.so") if timeline else (LIB.replace("libtdc.so", "libtdc_kn.so")
                                                                    if knobs else LIB)
    if not force and not timeline and not knobs and up_to_date():
        return LIB
    tmp = lib + f".{os.getpid()}.tmp"
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
           "-shared", "-I", os.path.join(ROOT, "include"), "-o", tmp, *sources()]
    if timeline:
        cmd.insert(1, "-DTDC_TIMELINE")
    if knobs:
        cmd.insert(1, "-DTDC_DEBUG_KNOBS")
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, timeline="--timeline" in sys.argv,
                knobs="--knobs" in sys.argv))
