"""Build libpmagraph_cuda.so in-tree for sm_100a (nvcc, static cudart).

The .so lands next to this file so it travels to the GPU box with the repo
snapshot; nothing is installed into site-packages.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "libpmagraph_cuda.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--extended-lambda",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-I" + os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "pmagraph_cuda.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return OUT
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *FLAGS, "-dc" if False else "-c", src, "-o", obj]
        cmd = [c for c in cmd if c != "-shared"]
        if verbose:
            cmd.append("-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out.decode())
        if p.returncode != 0:
            failed = True
    if failed:
        raise RuntimeError("nvcc failed")
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", *objs, "-o", OUT, "-ldl"]
    subprocess.check_call(link)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))


def build_cpp_tests() -> str:
    """C++ drop-in test (tests/cpp/test_dropin.cpp) against include/pmagraph/*.hpp,
    linked to the in-tree library (rpath $ORIGIN/../../paper_1709_05061_b200)."""
    src = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
    out = os.path.join(ROOT, "tests", "cpp", "test_dropin")
    if os.path.exists(out) and os.path.getmtime(out) > max(os.path.getmtime(src), os.path.getmtime(OUT)) and \
            all(os.path.getmtime(h) < os.path.getmtime(out) for h in glob.glob(os.path.join(ROOT, "include", "pmagraph", "*.hpp"))):
        return out
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), src, "-o", out,
                           "-L" + HERE, "-lpmagraph_cuda", "-Wl,-rpath,$ORIGIN/../../paper_1709_05061_b200"])
    return out


REF_TESTS = "/root/reference/proj/tests"
# the reference's unit-test files whose cases are reusable parity gates
# (SURVEY §4): compiled UNMODIFIED from where they lie, against OUR drop-in
# headers (include/pmagraph) and the Catch2 stand-in (tests/cpp/shim)
REF_SUITE_FILES = ["test_pma.cpp", "test_segment_engine.cpp", "test_graph.cpp", "test_analytics.cpp",
                   "test_primitives.cpp", "test_streaming.cpp"]


def build_ref_suite() -> str | None:
    """tests/cpp/ref_suite: the reference's own unit tests built against the
    drop-in headers and linked to libpmagraph_cuda.so.  Needs /root/reference
    (this container); the binary travels to the GPU box like the .so."""
    out = os.path.join(ROOT, "tests", "cpp", "ref_suite")
    if not os.path.isdir(REF_TESTS):
        return out if os.path.exists(out) else None
    srcs = [os.path.join(REF_TESTS, f) for f in REF_SUITE_FILES] + [os.path.join(ROOT, "tests", "cpp", "shim",
                                                                             "main.cpp")]
    deps = srcs + glob.glob(os.path.join(ROOT, "include", "pmagraph", "*.hpp")) + [OUT] + \
        glob.glob(os.path.join(ROOT, "tests", "cpp", "shim", "catch2", "*.hpp"))
    if os.path.exists(out) and os.path.getmtime(out) > max(os.path.getmtime(d) for d in deps):
        return out
    objdir = os.path.join(HERE, "build", "ref_suite")
    os.makedirs(objdir, exist_ok=True)
    procs, objs = [], []
    for src in srcs:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        procs.append(subprocess.Popen(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "tests", "cpp", "shim"),
                                       "-I" + os.path.join(ROOT, "include"), "-I" + REF_TESTS, "-c", src, "-o", obj]))
    if any(p.wait() for p in procs):
        raise RuntimeError("reference unit tests failed to build against the drop-in headers")
    subprocess.check_call(["g++", *objs, "-o", out, "-L" + HERE, "-lpmagraph_cuda",
                           "-Wl,-rpath,$ORIGIN/../../paper_1709_05061_b200"])
    return out


def build_tools() -> str:
    """tools/cpp/small_batch_latency: the C-ABI small-batch latency probe."""
    src = os.path.join(ROOT, "tools", "cpp", "small_batch_latency.cpp")
    out = os.path.join(ROOT, "tools", "cpp", "small_batch_latency")
    if os.path.exists(out) and os.path.getmtime(out) > max(os.path.getmtime(src), os.path.getmtime(OUT)):
        return out
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"), src, "-o", out,
                           "-L" + HERE, "-lpmagraph_cuda", "-Wl,-rpath,$ORIGIN/../../paper_1709_05061_b200"])
    return out
