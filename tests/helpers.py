"""Comparison helpers shared by the parity tests (test infrastructure)."""
import numpy as np

from oracle.oracle import stats_dict

FIXTURE_KEYS = [2, 8, 10, 11, 14, 17, 20, 25, 30, 33, 36, 40, 45, 50, 60, 70, 80, 90]
FIXTURE_SLOTS = [0, 4, 5, 6, 8, 9, 12, 13, 16, 17, 18, 20, 21, 22, 24, 25, 28, 29]


def fixture_arrays():
    """Paper Fig. 3 state (reference tests/support/fixtures.hpp:27-41):
    capacity 32, leaf 4, value = key * 10."""
    k = np.zeros(32, np.uint64)
    v = np.zeros(32, np.uint64)
    s = np.zeros(32, np.uint8)
    for slot, key in zip(FIXTURE_SLOTS, FIXTURE_KEYS):
        k[slot], v[slot], s[slot] = key, key * 10, 1
    return k, v, s


def ref_parity(ref, st):
    d = stats_dict(st)
    d.pop("num_touched_ranges")
    d["touched_ranges"] = ref.touched_ranges()
    return d


def assert_same_slots(a, b, ctx=""):
    ka, va, sa = a
    kb, vb, sb = b
    assert len(sa) == len(sb), f"{ctx}: capacity {len(sa)} vs {len(sb)}"
    bad = np.nonzero((ka != kb) | (va != vb) | (sa != sb))[0]
    assert len(bad) == 0, f"{ctx}: {len(bad)} slots differ, first at {bad[:5]}: " \
                          f"gpu {[(int(ka[i]), int(sa[i])) for i in bad[:3]]} ref {[(int(kb[i]), int(sb[i])) for i in bad[:3]]}"


def assert_same_counters(gpu, ref_layout, ctx=""):
    assert gpu.capacity() == ref_layout.capacity, ctx
    assert gpu.valid_count() == ref_layout.valid_count, ctx
    assert gpu.tombstone_count() == ref_layout.tombstone_count, ctx
    assert gpu.slot_writes() == ref_layout.slot_writes, ctx


def random_batch(rng, size, universe, delete_fraction):
    """TraceRng-style batch (reference tests/support/reference.hpp:252-272)."""
    keys = rng.integers(0, universe, size, dtype=np.uint64)
    ops = (rng.random(size) < delete_fraction).astype(np.uint8)
    vals = rng.integers(0, 2**63, size, dtype=np.uint64)
    vals[ops == 1] = 0
    return keys, vals, ops
