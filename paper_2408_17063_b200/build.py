"""Build libhcomp.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2408_17063_b200.build            # libhcomp.so + libhcomp_l4.so
    python -m paper_2408_17063_b200.build --selftest  # + host self-test lib (CPU tests)
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhcomp.so")  # chains of up to 4 primes (max_level <= 3: every BASELINE config)
LIB5 = os.path.join(HERE, "libhcomp_l4.so")  # the same sources for 5-prime chains (max_level 4: answer())
# pdq's protocol chain (protocol_max_level = 21, CLI default 22): deep levels
# carry ring transforms and mul_plain only; Comp runs at levels <= 4
LIBDEEP = os.path.join(HERE, "libhcomp_deep.so")
# The 5-prime build's larger device context costs ~1% at the headline (measured
# A/B, tools/ab_old_new.sh), so each chain length gets its own build.
LIBS = {LIB: 3, LIB5: 4, LIBDEEP: 22}
SELFTEST = os.path.join(HERE, "libhcomp_hosttest.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))] + [
        os.path.join(os.path.dirname(HERE), "include", "hcomp.h")
    ]


def _stale(target: str) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in _sources())


def build_lib(force: bool = False, verbose: bool = False) -> str:
    procs = []
    for path, maxl in LIBS.items():
        if force or _stale(path):
            cmd = [
                NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
                f"-DHC_MAXL={maxl}", "-o", path, os.path.join(CSRC, "hcomp.cu"),
            ]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            procs.append((cmd, subprocess.Popen(cmd)))
    for cmd, p in procs:
        if p.wait():
            raise subprocess.CalledProcessError(p.returncode, cmd)
    return LIB


CHECK = os.path.join(HERE, "libhcomp_check.so")


def build_check(force: bool = False) -> str:
    """The 4-prime library with the device-side invariant assertions
    (-DHC_CHECK, kernels.cuh HC_ASSERT): run the GPU tests against it with
    HCOMP_LIB=paper_2408_17063_b200/libhcomp_check.so."""
    if force or _stale(CHECK):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
               "-DHC_MAXL=3", "-DHC_CHECK", "-o", CHECK, os.path.join(CSRC, "hcomp.cu")]
        subprocess.check_call(cmd)
    return CHECK


TRACE = os.path.join(HERE, "libhcomp_trace.so")


def build_trace(force: bool = False) -> str:
    """The 4-prime library with the per-CTA %globaltimer timeline (-DHC_TRACE),
    read by tools/trace_comp.py and tools/trace_fold.py."""
    if force or _stale(TRACE):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
               "-DHC_MAXL=3", "-DHC_TRACE", "-o", TRACE, os.path.join(CSRC, "hcomp.cu")]
        subprocess.check_call(cmd)
    return TRACE


def build_selftest(force: bool = False) -> str:
    """The device arithmetic/NTT schedule compiled for the host (g++), used by
    tests/test_csrc_host.py to check the exact GPU code paths on the CPU."""
    if force or _stale(SELFTEST):
        cmd = [
            "/usr/bin/g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-o", SELFTEST,
            os.path.join(CSRC, "hosttest.cpp"),
        ]
        subprocess.check_call(cmd)
    return SELFTEST


if __name__ == "__main__":
    build_lib(force="--force" in sys.argv, verbose="-v" in sys.argv)
    if "--selftest" in sys.argv:
        build_selftest(force="--force" in sys.argv)
    if "--check" in sys.argv:
        build_check(force="--force" in sys.argv)
    if "--trace" in sys.argv:
        build_trace(force="--force" in sys.argv)
    print(LIB)
