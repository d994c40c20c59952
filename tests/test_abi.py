"""CPU: the C-ABI library builds for sm_100a, loads without a GPU, and exports
every symbol the public headers declare (include/pmagraph_cuda.h,
include/pmagraph_stream.h); the ctypes mirror covers the same set."""
import ctypes
import os
import re
import subprocess

from paper_1709_05061_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", "pmagraph_cuda.h"), os.path.join(ROOT, "include", "pmagraph_stream.h")]


def declared():
    names = set()
    for h in HEADERS:
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s+\**\s*([a-z_][a-z0-9_]*)\s*\(", text,
                             re.M):
            names.add(m.group(1))
    return names


def test_library_loads_and_exports_declared_symbols():
    assert os.path.exists(abi.LIB_PATH), "build first: python -c 'import __graft_entry__ as g; g.build()'"
    lib = ctypes.CDLL(abi.LIB_PATH)
    names = declared()
    assert len(names) > 40
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert names <= exported


def test_ctypes_mirror_matches_headers():
    names = declared()
    mirrored = {n for n, _, _ in abi.SIGNATURES}
    assert mirrored <= names, mirrored - names
    assert names <= mirrored, names - mirrored


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", abi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_sizes_match_c_layout():
    assert ctypes.sizeof(abi.pma_stats) == 10 * 8 + 2 * 4 + 64 * 8
    assert ctypes.sizeof(abi.pma_profile) == 4 * 8 + 8
    assert ctypes.sizeof(abi.pma_engine_config) == 4 + 4 + 8 + 8 + 4 + 4
