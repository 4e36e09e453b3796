#!/usr/bin/env python3
"""Builds every native artefact in-tree.

  paper_2510_06179_b200/lib/libdocp_cuda.so   the product (sm_100a CUDA + C ABI)
  oracle/_build/libdocp_port.so               C restatement (test checker)
  oracle/_ref/*                               reference headers + eigen_lite
                                              (only where /root/reference exists)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(ROOT, "paper_2510_06179_b200", "csrc")
LIB = os.path.join(ROOT, "paper_2510_06179_b200", "lib", "libdocp_cuda.so")
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "--fmad=false", "-lineinfo",
              "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC,-O2", "-I", os.path.join(ROOT, "include")]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_cuda(force=False, verbose=False):
    sources = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "docp_cuda.h")]
    if not force and not _stale(LIB, sources):
        return
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    cmd = ["nvcc", *NVCC_FLAGS, "-o", LIB, os.path.join(CSRC, "docp_cuda.cu"), os.path.join(CSRC, "generators.cpp")]
    log = os.path.join(os.path.dirname(LIB), "ptxas.log")
    with open(log, "w") as fh:
        r = subprocess.run(cmd, stdout=fh, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        sys.stderr.write(open(log).read())
        raise RuntimeError("nvcc failed")
    if verbose:
        print("built", LIB)


def build_oracle():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "port"], check=True)
    if os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)


def main():
    build_cuda(force="--force" in sys.argv, verbose=True)
    build_oracle()


if __name__ == "__main__":
    main()
