"""CPU: the C-ABI library builds for sm_100a, loads without a GPU, and exports
every symbol the public headers declare (include/pmagraph_cuda.h,
include/pmagraph_stream.h); the ctypes mirror covers the same set."""
import ctypes
import os
import re
import subprocess
import sys

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


# Every entry point that takes an existing handle first must reject a NULL
# handle with PMA_EINVAL (checked before any CUDA call, so this runs on CPU)
# instead of dereferencing it.  One subprocess for all of them: a crash
# fails the test instead of killing the run.
_NULL_PROBE = r"""
import ctypes as C, sys
sys.path.insert(0, sys.argv[1])
from paper_1709_05061_b200 import abi
lib = abi.load_library()
bad = []
for name, res, args in abi.SIGNATURES:
    if not args or args[0] is not abi._P or res is not C.c_int:
        continue
    if name.endswith(("_destroy", "_create", "last_error")) or name in SKIP:
        continue
    vals = [None]
    for t in args[1:]:
        if t is abi._P or (isinstance(t, type) and issubclass(t, (C._Pointer, C.c_char_p, C.c_void_p))):
            vals.append(None)
        elif t in (C.c_double, C.c_float):
            vals.append(0.0)
        else:
            vals.append(0)
    print(name, flush=True)
    rc = getattr(lib, name)(*vals)
    if rc != abi.PMA_EINVAL:
        bad.append((name, rc))
print("BAD", bad)
"""


def test_null_handles_are_rejected():
    # first argument is not a library handle: an id buffer / a device pointer
    skip = {"gpma_nccl_unique_id", "gpma_ipc_close", "gpma_ipc_free"}
    code = "SKIP = %r\n" % skip + _NULL_PROBE
    p = subprocess.run([sys.executable, "-c", code, ROOT], capture_output=True, text=True, timeout=300)
    last = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else ""
    assert p.returncode == 0, f"crashed after {last!r}: {p.stderr[-500:]}"
    assert last == "BAD []", last


def test_update_stats_csv_rows():
    """UpdateStats.csv_row keeps the reference's schema (update_stats.hpp:27-34);
    csv_row_device appends the device columns SURVEY §5 names (no GPU needed:
    a timing record stands in)."""
    from types import SimpleNamespace

    from paper_1709_05061_b200.pmagraph import UpdateStats
    u = UpdateStats(batch_size=10, rounds=2, slot_writes=40, wall_ns=1234)
    assert UpdateStats.csv_header() == "batch_size,rounds,slot_writes,wall_ns"
    assert u.csv_row() == "10,2,40,1234"
    t = SimpleNamespace(device_ms=1.0, commit_bytes=3_000_000_000)
    assert UpdateStats.csv_header_device().endswith(",gpus,bytes_moved,hbm_frac,nvlink_frac")
    row = u.csv_row_device(t, gpus=2, hbm_peak_gbps=6000.0, nvlink_bytes=450_000_000)
    assert row == "10,2,40,1234,2,3000000000,0.5000,0.5000"
