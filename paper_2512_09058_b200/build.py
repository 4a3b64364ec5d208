"""Builds libcyqlone_b200.so in-tree for sm_100a with nvcc.

    python -m paper_2512_09058_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libcyqlone_b200.so")
SOURCES = ["riccati.cu", "riccati_warp.cu", "riccati_cta.cu", "riccati_pc.cu", "schur_cr.cu", "schur_tiles.cu", "schur_fused.cu", "schur_big.cu", "backsub.cu", "backsub_warp.cu", "backsub_tile.cu", "forward.cu", "augment.cu", "linesearch.cu", "gradients.cu", "update.cu",
           "capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "cyqlone_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    """One nvcc -c per source (in parallel, into build/), then one link."""
    if not force and not needs_build():
        return OUT
    from concurrent.futures import ThreadPoolExecutor

    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"]

    def compile_one(src: str):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        r = subprocess.run([NVCC, *cflags, "-c", "-o", obj, os.path.join(CSRC, src)],
                           capture_output=True, text=True)
        return obj, r

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    log = "".join(r.stdout + r.stderr for _, r in results)
    if verbose or any(r.returncode for _, r in results):
        sys.stderr.write(log)
    if any(r.returncode for _, r in results):
        raise RuntimeError("nvcc failed building libcyqlone_b200.so")
    r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT,
                        *[o for o, _ in results]], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed for libcyqlone_b200.so")
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as fh:
        fh.write(log)
    return OUT


HOST_SOURCES = ["host/ocp.cpp", "host/kkt_solver.cpp"]
HOST_OUT = os.path.join(HERE, "libcyqlone_b200_host.so")
ROOT = os.path.dirname(HERE)
HOST_TEST_SRC = os.path.join(ROOT, "tests", "cpp", "test_kkt_host.cpp")
HOST_TEST_OUT = os.path.join(ROOT, "tests", "cpp", "test_kkt_host")
CXX = os.environ.get("CXX", "g++")


def build_host(verbose: bool = False) -> str:
    """The C++ mirror of the reference interface (cyqlone::kkt / cyqlone::ocp,
    include/cyqlone_b200/*.hpp) as libcyqlone_b200_host.so over the CUDA
    library, plus the C++ test driver tests/cpp/test_kkt_host. Host-only g++
    (no CUDA headers): the kernels are reached through the C ABI."""
    cmds = [
        [CXX, "-O2", "-std=c++17", "-fPIC", "-shared", "-Wall", "-Wextra", "-o", HOST_OUT,
         *[os.path.join(HERE, s) for s in HOST_SOURCES], "-L" + HERE, "-lcyqlone_b200",
         "-Wl,-rpath,$ORIGIN"],
        [CXX, "-O2", "-std=c++17", "-Wall", "-I" + os.path.join(ROOT, "include"), "-o", HOST_TEST_OUT,
         HOST_TEST_SRC, "-L" + HERE, "-lcyqlone_b200_host", "-lcyqlone_b200",
         "-Wl,-rpath,$ORIGIN/../../paper_2512_09058_b200"],
    ]
    for cmd in cmds:
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError("g++ failed: " + " ".join(cmd[:8]))
    return HOST_OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    print(build_host(verbose=True))
