"""Builds the in-tree CUDA library libcftft_b200.so for sm_100a.

The shared object lands in paper_0810_3203_b200/lib/ (git-ignored, but it
travels to the GPU box with the repository snapshot).
"""
from __future__ import annotations

import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libcftft_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]

SOURCES = ["capi.cu"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    inc = os.path.join(os.path.dirname(PKG), "include")
    for d in (CSRC, inc):
        for f in os.listdir(d):
            if os.path.getmtime(os.path.join(d, f)) > t:
                return True
    return False


def source_sha256() -> str:
    """sha256 over the library's sources (csrc/ and include/, sorted by name):
    identifies a build independently of the .so bytes, which nvcc does not
    reproduce from one run to the next."""
    import hashlib

    h = hashlib.sha256()
    inc = os.path.join(os.path.dirname(PKG), "include")
    for d in (CSRC, inc):
        for f in sorted(os.listdir(d)):
            if f.endswith((".cu", ".cuh", ".hpp", ".h")):
                h.update(f.encode())
                with open(os.path.join(d, f), "rb") as fh:
                    h.update(fh.read())
    return h.hexdigest()


def build_library(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    # CFTFT_BUILD_EXPERIMENTS=1: a build whose experiment knobs (phase clocks,
    # debug skips: csrc/capi.cu env_int) follow the environment
    extra = ["-DCFTFT_EXPERIMENTS"] if os.environ.get("CFTFT_BUILD_EXPERIMENTS") == "1" else []
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-o", LIB + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    if verbose:
        print(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    with open(os.path.join(LIBDIR, "ptxas.log"), "w") as fh:
        fh.write(r.stderr)
    return LIB


if __name__ == "__main__":
    print(build_library(force=True, verbose=True))


API_TEST_SRC = os.path.join(os.path.dirname(PKG), "tests", "cpp", "api_test.cpp")
API_TEST = os.path.join(LIBDIR, "api_test")


def build_api_test(force: bool = False) -> str:
    """The C++ host-API test program (tests/cpp/api_test.cpp), linked against
    the in-tree library with an $ORIGIN rpath."""
    if not force and os.path.exists(API_TEST) and os.path.getmtime(API_TEST) >= max(
            os.path.getmtime(API_TEST_SRC), os.path.getmtime(LIB)):
        return API_TEST
    cmd = [_nvcc(), "-std=c++17", "-O2", "-o", API_TEST + ".tmp", API_TEST_SRC, "-L", LIBDIR, "-lcftft_b200",
           "-Xlinker", "-rpath=$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("api_test build failed:\n" + r.stdout + r.stderr)
    os.replace(API_TEST + ".tmp", API_TEST)
    return API_TEST


CLI_SRC = os.path.join(PKG, "cli", "cftft_cli.cpp")
CLI = os.path.join(LIBDIR, "cftft")


def build_cli(force: bool = False) -> str:
    """The command-line workbench (cli/cftft_cli.cpp: verify / count / bench /
    compare, the reference CLI's contract), linked against the in-tree
    library with an $ORIGIN rpath."""
    if not force and os.path.exists(CLI) and os.path.getmtime(CLI) >= max(os.path.getmtime(CLI_SRC),
                                                                          os.path.getmtime(LIB)):
        return CLI
    cmd = [_nvcc(), "-std=c++17", "-O2", "-o", CLI + ".tmp", CLI_SRC, "-L", LIBDIR, "-lcftft_b200",
           "-Xlinker", "-rpath=$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("cli build failed:\n" + r.stdout + r.stderr)
    os.replace(CLI + ".tmp", CLI)
    return CLI
