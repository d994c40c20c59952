"""GPU parity of the GPMA+ batch engine and the PMA API against the
UNMODIFIED reference (oracle/_ref/libpmagraph_ref.so): slot arrays (keys,
values, states, gap positions), counters and every UpdateStats field must be
bit-exact after every batch.  Cases mirror the reference's own tests
(proj/tests/test_pma.cpp, test_segment_engine.cpp)."""
import numpy as np
import pytest

from oracle.oracle import RefPMA
from paper_1709_05061_b200.abi import (PMA_EAGER, PMA_LAZY, PMA_STRATEGY_LARGE, PMA_STRATEGY_MEDIUM,
                                       PMA_STRATEGY_SMALL, engine_config)
from paper_1709_05061_b200.pmagraph import (DensityProfile, LogicError, PackedMemoryArray, SegmentEngineConfig,
                                            batch_update)
from tests.helpers import (assert_same_counters, assert_same_slots, fixture_arrays, random_batch, ref_parity)

pytestmark = pytest.mark.gpu


def pair(k, v, s):
    return PackedMemoryArray.from_slots(k, v, s), RefPMA().load_slots(k, v, s)


def run_both(g, r, keys, vals, ops, mode=PMA_LAZY, force=-1, ctx=""):
    cfg = SegmentEngineConfig(deletion_mode=mode, force_strategy=force)
    gs = batch_update(g, keys, vals, ops, cfg)
    rs = r.batch_update(keys, vals, ops, engine_config(deletion_mode=mode, force_strategy=force))
    assert gs.parity() == ref_parity(r, rs), ctx
    assert_same_slots(g.slots(), r.slots(), ctx)
    assert_same_counters(g, r.layout(), ctx)
    return gs


def test_threshold_table_capacity_32():
    # test_pma.cpp:14-41
    g = PackedMemoryArray.from_slots(*fixture_arrays())
    assert (g.capacity(), g.leaf_size(), g.height()) == (32, 4, 3)
    assert [g.min_entries(l) for l in range(4)] == [1, 2, 4, 8]
    assert [g.max_entries(l) for l in range(4)] == [3, 6, 12, 24]
    rho = [0.08, 0.19, 0.29, 0.40]
    tau = [0.92, 0.88, 0.84, 0.80]
    for l in range(4):
        lo, hi = g.thresholds(l)
        assert abs(lo - rho[l]) < 0.005 and abs(hi - tau[l]) < 0.005
    with pytest.raises(IndexError):
        g.thresholds(4)
    with pytest.raises(IndexError):
        g.thresholds(-1)


def test_binary_search_leaf_on_fixture():
    # test_pma.cpp:81-89
    g = PackedMemoryArray.from_slots(*fixture_arrays())
    assert [g.binary_search_leaf(k) for k in (48, 35, 9, 1, 4, 1000)] == [5, 4, 1, 0, 0, 7]


def test_five_insert_batch_three_rounds():
    # test_segment_engine.cpp:53-73
    g, r = pair(*fixture_arrays())
    keys = np.array([1, 4, 9, 35, 48], np.uint64)
    st = run_both(g, r, keys, keys * 10, np.zeros(5, np.uint8))
    assert st.rounds == 3
    assert st.segments_per_level == [1, 0, 2, 0]
    assert st.grow_events == 0
    assert g.valid_count() == 23
    for k in (1, 4, 9, 35, 48):
        assert g.search(k) == k * 10


def test_empty_batch_is_noop():
    g, r = pair(*fixture_arrays())
    before = g.slots()
    st = run_both(g, r, np.zeros(0, np.uint64), np.zeros(0, np.uint64), np.zeros(0, np.uint8))
    assert st.rounds == 0 and st.slot_writes == 0
    assert_same_slots(g.slots(), before)


def test_lazy_deletes_only_tombstone():
    # test_segment_engine.cpp:263-286
    g, r = pair(*fixture_arrays())
    before = g.slots()
    st = run_both(g, r, np.array([30, 45, 999], np.uint64), np.zeros(3, np.uint64), np.ones(3, np.uint8))
    assert st.rounds == 1 and st.tombstones_added == 2 and st.deletes_missed == 1
    assert st.touched_ranges == []
    assert g.tombstone_count() == 2 and g.search(30) is None
    assert (g.slots()[0] == before[0]).all()
    run_both(g, r, np.array([31, 46], np.uint64), np.array([310, 460], np.uint64), np.zeros(2, np.uint8))
    assert g.tombstone_count() == 0 and g.search(31) == 310


def test_growth_exactly_once():
    # test_segment_engine.cpp:250-261: root full at capacity 16 plus 4 inserts
    ref = RefPMA()
    gpu = PackedMemoryArray()
    root_max = gpu.max_entries(gpu.height())
    for i in range(root_max):
        ref.insert(i * 7, i)
        gpu.insert(i * 7, i)
    assert_same_slots(gpu.slots(), ref.slots(), "seq inserts")
    assert gpu.capacity() == 16
    keys = np.array([3, 10, 17, 24], np.uint64)
    st = run_both(gpu, ref, keys, keys * 10, np.zeros(4, np.uint8))
    assert st.grow_events == 1 and st.resized and gpu.capacity() == 32


def test_duplicate_resolution():
    # test_segment_engine.cpp:310-326
    g, r = pair(*fixture_arrays())
    keys = np.array([30, 30, 5, 5, 40, 41, 40], np.uint64)
    vals = np.array([0, 777, 1, 2, 0, 5, 9], np.uint64)
    ops = np.array([1, 0, 0, 0, 1, 0, 0], np.uint8)
    run_both(g, r, keys, vals, ops)
    assert [g.search(k) for k in (30, 5, 40, 41)] == [777, 2, 9, 5]


@pytest.mark.parametrize("mode", [PMA_LAZY, PMA_EAGER])
@pytest.mark.parametrize("force", [-1, PMA_STRATEGY_SMALL, PMA_STRATEGY_MEDIUM, PMA_STRATEGY_LARGE])
def test_random_traces_match_reference(mode, force):
    rng = np.random.default_rng(1000 + 10 * mode + force)
    for trial in range(12):
        universe = int(rng.integers(64, 200000))
        n0 = int(rng.integers(0, 5000))
        keys = np.unique(rng.integers(0, universe, n0, dtype=np.uint64))
        vals = rng.integers(0, 2**63, len(keys), dtype=np.uint64)
        fill = float(rng.uniform(0.1, 0.9))
        g = PackedMemoryArray.from_sorted(keys, vals, fill)
        r = RefPMA().from_sorted(keys, vals, fill)
        assert_same_slots(g.slots(), r.slots(), "from_sorted")
        assert_same_counters(g, r.layout(), "from_sorted")
        for b in range(8):
            nb = int(rng.integers(0, 3000))
            k, v, o = random_batch(rng, nb, universe, float(rng.random()))
            run_both(g, r, k, v, o, mode, force, f"trial {trial} batch {b}")


def test_skewed_batches_escalate_levels():
    """Hot key ranges push groups up the tree (CTA tier, root path, grow)."""
    rng = np.random.default_rng(7)
    for mode in (PMA_LAZY, PMA_EAGER):
        g, r = PackedMemoryArray(), RefPMA()
        base = 0
        for b in range(25):
            n = int(rng.integers(50, 4000))
            keys = (base + np.arange(n, dtype=np.uint64) * int(rng.integers(1, 4))).astype(np.uint64)
            ops = (rng.random(n) < (0.1 if b % 3 else 0.6)).astype(np.uint8)
            vals = rng.integers(0, 2**63, n, dtype=np.uint64)
            st = run_both(g, r, keys, vals, ops, mode, -1, f"mode {mode} batch {b}")
            base += int(rng.integers(0, 3000))
        assert g.capacity() >= 1024


def _sparse_layout(rng, cap, occupancy, tomb_frac):
    """Sorted keys at random slots (runs of empty leaves), some tombstones."""
    n = int(cap * occupancy)
    slots = np.sort(rng.choice(cap, n, replace=False))
    keys = np.sort(rng.choice(2**30, n, replace=False)).astype(np.uint64)
    k = np.zeros(cap, np.uint64)
    v = np.zeros(cap, np.uint64)
    s = np.zeros(cap, np.uint8)
    k[slots], v[slots] = keys, keys * 3
    s[slots] = np.where(rng.random(n) < tomb_frac, 2, 1)
    return k, v, s, keys


@pytest.mark.parametrize("mode", [PMA_LAZY, PMA_EAGER])
def test_empty_leaf_runs_and_header_refresh(mode):
    """Layouts with long runs of empty leaves exercise the backward-filled
    header refresh (left walks, forward scans) against the reference's
    top-down leaf search."""
    rng = np.random.default_rng(17 + mode)
    for trial in range(10):
        cap = int(2 ** rng.integers(8, 15))
        k, v, s, keys = _sparse_layout(rng, cap, float(rng.uniform(0.02, 0.3)), 0.2)
        g, r = pair(k, v, s)
        probe = rng.integers(0, 2**30, 500, dtype=np.uint64)
        assert (g.binary_search_leaf(probe) == r.binary_search_leaf(probe)).all()
        for b in range(6):
            nb = int(rng.integers(1, 400))
            kk = np.where(rng.random(nb) < 0.5, rng.choice(keys, nb), rng.integers(0, 2**30, nb)).astype(np.uint64)
            vv = rng.integers(0, 2**63, nb, dtype=np.uint64)
            oo = (rng.random(nb) < 0.6).astype(np.uint8)
            run_both(g, r, kk, vv, oo, mode, -1, f"trial {trial} batch {b}")
            assert (g.binary_search_leaf(probe) == r.binary_search_leaf(probe)).all(), f"trial {trial} batch {b}"


def test_large_array_and_batch():
    rng = np.random.default_rng(11)
    keys = np.unique(rng.integers(0, 2**40, 300000, dtype=np.uint64))
    vals = rng.integers(0, 2**63, len(keys), dtype=np.uint64)
    g = PackedMemoryArray.from_sorted(keys, vals, 0.5)
    r = RefPMA().from_sorted(keys, vals, 0.5)
    for b in range(4):
        k, v, o = random_batch(rng, 100000, 2**40, 0.5)
        # half the deletes hit existing keys
        hit = rng.random(len(k)) < 0.5
        k[hit & (o == 1)] = rng.choice(keys, int((hit & (o == 1)).sum()))
        run_both(g, r, k, v, o, PMA_LAZY, -1, f"batch {b}")


def test_leaf_search_matches_reference_with_tombstones_and_max_key():
    rng = np.random.default_rng(5)
    for trial in range(20):
        n = int(rng.integers(0, 3000))
        keys = np.unique(rng.integers(0, 500000, n, dtype=np.uint64))
        if trial % 4 == 0 and len(keys):
            keys[-1] = np.uint64(2**64 - 1)
        g = PackedMemoryArray.from_sorted(keys, keys, 0.5)
        r = RefPMA().from_sorted(keys, keys, 0.5)
        tomb = rng.choice(keys, min(20, len(keys)), replace=False) if len(keys) else []
        for t in tomb:
            assert g.mark_tombstone(int(t)) == r.mark_tombstone(int(t))
        probe = np.concatenate([rng.integers(0, 520000, 400, dtype=np.uint64),
                                np.array([0, 2**64 - 1], np.uint64)])
        assert (g.binary_search_leaf(probe) == r.binary_search_leaf(probe)).all()


def test_from_sorted_rejects_unsorted_or_duplicate():
    with pytest.raises(ValueError, match="strictly increasing"):
        PackedMemoryArray.from_sorted(np.array([1, 1], np.uint64), np.zeros(2, np.uint64), 0.5)
    with pytest.raises(ValueError, match="index 1"):
        PackedMemoryArray.from_sorted(np.array([5, 3], np.uint64), np.zeros(2, np.uint64), 0.5)
    with pytest.raises(ValueError):
        PackedMemoryArray.from_sorted(np.zeros(0, np.uint64), np.zeros(0, np.uint64), 0.0)
    g = PackedMemoryArray.from_sorted(np.zeros(0, np.uint64), np.zeros(0, np.uint64), 0.5)
    assert g.capacity() == 16 and g.valid_count() == 0


def test_sequential_ops_match_reference():
    # test_pma.cpp random insert / alternating insert-erase traces
    rng = np.random.default_rng(31)
    g, r = PackedMemoryArray(), RefPMA()
    for i in range(1500):
        key = int(rng.integers(0, 600))
        if rng.random() < 0.55:
            val = int(rng.integers(0, 2**63))
            g.insert(key, val)
            r.insert(key, val)
        elif rng.random() < 0.8:
            assert g.erase(key) == r.erase(key)
        else:
            assert g.mark_tombstone(key) == r.mark_tombstone(key)
        if i % 50 == 0:
            assert_same_slots(g.slots(), r.slots(), f"op {i}")
            assert_same_counters(g, r.layout(), f"op {i}")
    assert_same_slots(g.slots(), r.slots(), "end")


def test_fixture_insert_48_and_redispatch():
    # test_pma.cpp:132-153, 249-260
    g, r = pair(*fixture_arrays())
    g.insert(48, 480)
    r.insert(48, 480)
    assert_same_slots(g.slots(), r.slots())
    k, v, s = g.slots()
    want = {16: 30, 17: 33, 18: 36, 20: 40, 21: 45, 23: 48, 24: 50, 26: 60, 27: 70, 29: 80, 30: 90}
    for slot, key in want.items():
        assert s[slot] == 1 and k[slot] == key
    g2, r2 = pair(*fixture_arrays())
    g2.redispatch(2, 1, [48], [480])
    r2.redispatch(2, 1, np.array([48], np.uint64), np.array([480], np.uint64))
    assert_same_slots(g2.slots(), r2.slots())
    with pytest.raises(LogicError):
        g2.redispatch(2, 1, list(range(200, 213)), [0] * 13)


def test_shrink_disabled_profile():
    prof = DensityProfile(allow_shrink=False)
    g = PackedMemoryArray(prof)
    for i in range(40):
        g.insert(i, i)
    grown = g.capacity()
    for i in range(40):
        g.erase(i)
    assert g.capacity() == grown and g.valid_count() == 0


@pytest.mark.parametrize("mode", [PMA_LAZY, PMA_EAGER])
@pytest.mark.parametrize("force", [-1, PMA_STRATEGY_LARGE])
def test_grid_tier_matches_reference(mode, force):
    """The grid tier (pma_set_grid_segment): segments from 64 slots up are
    merged by device-wide kernels instead of one CTA each — slot arrays,
    counters and every UpdateStats field (incl. commit_in_place's slot_writes
    under the large tier) must stay bit-exact."""
    rng = np.random.default_rng(2024 + 10 * mode + force)
    grid_merges = 0
    for trial in range(6):
        universe = int(rng.integers(2000, 200000))
        keys = np.unique(rng.integers(0, universe, int(rng.integers(500, 6000)), dtype=np.uint64))
        vals = rng.integers(0, 2**63, len(keys), dtype=np.uint64)
        g = PackedMemoryArray.from_sorted(keys, vals, 0.5)
        g.set_grid_segment(64)
        r = RefPMA().from_sorted(keys, vals, 0.5)
        base = 0
        for b in range(10):
            if b % 2:  # hot key runs: groups escalate to large segments
                n = int(rng.integers(200, 3000))
                k = (base + np.arange(n, dtype=np.uint64) * int(rng.integers(1, 3))).astype(np.uint64)
                o = (rng.random(n) < 0.3).astype(np.uint8)
                v = rng.integers(0, 2**63, n, dtype=np.uint64)
                base += int(rng.integers(0, 5000))
            else:
                k, v, o = random_batch(rng, int(rng.integers(0, 3000)), universe, float(rng.random()))
            run_both(g, r, k, v, o, mode, force, f"grid tier trial {trial} batch {b}")
            grid_merges += int(g.last_timing().grid_merges)
    assert grid_merges > 0, "the batches never reached the grid tier"
