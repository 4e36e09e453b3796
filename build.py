#!/usr/bin/env python3
"""Builds every native artefact in-tree.

  paper_2510_06179_b200/lib/libdocp_cuda.so   the product (sm_100a CUDA + C ABI)
  oracle/_build/libdocp_port.so               C restatement (test checker)
  oracle/_ref/*                               reference headers + eigen_lite
                                              (only where /root/reference exists)
  paper_2510_06179_b200/lib/docp_gpu          CLI (`solve`, `grad-check`) over the C ABI
  tests/cpp/_bin/test_dropin                  C++ drop-in tests (docp_gpu.hpp vs the
                                              reference headers; same condition)
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


UNITS = ["docp_cuda.cu", "pcg_nx8.cu", "pcg_nx4.cu", "pcg_nx16.cu", "pcg_nxrt.cu", "pcg_nxct.cu", "generators.cpp"]


def build_cuda(force=False, verbose=False, lib=None, extra_flags=()):
    """Compiles the translation units in parallel, then links the shared library.
    lib / extra_flags: an A/B variant (e.g. -DDOCP_H8P_CLOCK) built elsewhere."""
    LIB_ = lib or LIB
    sources = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "docp_cuda.h")]
    if not force and not _stale(LIB_, sources):
        return
    objdir = os.path.join(os.path.dirname(LIB_), "obj")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"] + list(extra_flags)
    procs = []
    for unit in UNITS:
        obj = os.path.join(objdir, unit + ".o")
        log = open(os.path.join(objdir, unit + ".log"), "w")
        cmd = ["nvcc", *compile_flags, "-c", "-o", obj, os.path.join(CSRC, unit)]
        procs.append((unit, obj, log, subprocess.Popen(cmd, stdout=log, stderr=subprocess.STDOUT)))
    failed = []
    for unit, obj, log, p in procs:
        if p.wait() != 0:
            failed.append(unit)
        log.close()
    with open(os.path.join(os.path.dirname(LIB_), "ptxas.log"), "w") as out:
        for unit in UNITS:
            out.write(open(os.path.join(objdir, unit + ".log")).read())
    if failed:
        for unit in failed:
            sys.stderr.write(open(os.path.join(objdir, unit + ".log")).read())
        raise RuntimeError(f"nvcc failed: {failed}")
    objs = [os.path.join(objdir, u + ".o") for u in UNITS]
    r = subprocess.run(["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB_, *objs])
    if r.returncode != 0:
        raise RuntimeError("link failed")
    if verbose:
        print("built", LIB_)


CLI_SRC = os.path.join(ROOT, "paper_2510_06179_b200", "cli")
CLI = os.path.join(os.path.dirname(LIB), "docp_gpu")


def build_cli(force=False):
    """The docp_main.cpp `solve` / `grad-check` front-end on the GPU path."""
    sources = [os.path.join(CLI_SRC, f) for f in os.listdir(CLI_SRC)] + [LIB, os.path.join(ROOT, "include", "docp_cuda.h")]
    if not force and not _stale(CLI, sources):
        return
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-Wall", "-I", os.path.join(ROOT, "include"),
                    "-o", CLI, os.path.join(CLI_SRC, "docp_gpu_main.cpp"), "-L", os.path.dirname(LIB),
                    "-ldocp_cuda", "-Wl,-rpath,$ORIGIN"], check=True)


def build_oracle():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "port"], check=True)
    if os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)


def main():
    build_cuda(force="--force" in sys.argv, verbose=True)
    build_cli(force="--force" in sys.argv)
    build_oracle()


if __name__ == "__main__":
    main()
