"""Stream generators (CPU) and the device sliding window (GPU) against the
reference generators.hpp / streaming.hpp through the oracle."""
import numpy as np
import pytest

from oracle.oracle import RefRng, RefStream, RefWindow, draw_below_sequence as ref_draw
from paper_1709_05061_b200.pmagraph import EdgeStream, Mt19937_64, SlidingWindow, draw_below_sequence


@pytest.mark.parametrize("kind", ["rmat", "er", "rmat_params"])
def test_generators_match_reference(kind):
    if kind == "rmat":
        a, b = EdgeStream.rmat(2**12, 40000, seed=1), RefStream.rmat(2**12, 40000, seed=1)
    elif kind == "rmat_params":
        a = EdgeStream.rmat(2**10, 20000, seed=5, a=0.45, b=0.15, c=0.15, d=0.25)
        b = RefStream.rmat(2**10, 20000, seed=5, a=0.45, b=0.15, c=0.15, d=0.25)
    else:
        a, b = EdgeStream.erdos_renyi(5000, 0.003, seed=3), RefStream.erdos_renyi(5000, 0.003, seed=3)
    a.shuffle(2)
    b.shuffle(2)
    s, d = a.arrays()
    rs, rd, _, _ = b.arrays()
    assert len(s) == len(rs) and (s == rs).all() and (d == rd).all()


def test_draw_below_matches_reference():
    assert (draw_below_sequence(7, 2**21, 50) == ref_draw(7, 2**21, 50)).all()


def test_generator_rejects_bad_params():
    with pytest.raises(ValueError):
        EdgeStream.rmat(1000, 10)
    with pytest.raises(ValueError):
        EdgeStream.rmat(1024, 10, a=0.5, b=0.5, c=0.5, d=0.5)
    with pytest.raises(ValueError):
        EdgeStream.erdos_renyi(10, 1.0)


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [1, 7, 250, 4096])
def test_device_window_matches_reference(batch):
    # test_streaming.cpp:96-135: duplicates in the stream are not deleted
    # while another arrival of the same edge is still in the window
    a = EdgeStream.rmat(2**8, 20000, seed=4)      # many duplicate arrivals
    b = RefStream.rmat(2**8, 20000, seed=4)
    w, rw = SlidingWindow(a, 0), RefWindow(b)
    s, d = a.arrays()
    for _ in range(12 if batch > 100 else 40):
        sl = w.slide(batch)
        ra, rb, _, rc, rd = rw.slide(batch)
        assert (s[sl.ins_offset:sl.ins_offset + sl.n_ins] == ra).all()
        assert (d[sl.ins_offset:sl.ins_offset + sl.n_ins] == rb).all()
        c, dd = w.deletions_host(sl.del_offset, sl.n_del)
        assert (c == rc).all() and (dd == rd).all()


def _same_slide(w, sl, s, d, ref):
    ra, rb, _, rc, rd = ref
    assert (s[sl.ins_offset:sl.ins_offset + sl.n_ins] == ra).all()
    assert (d[sl.ins_offset:sl.ins_offset + sl.n_ins] == rb).all()
    c, dd = w.deletions_host(sl.del_offset, sl.n_del)
    assert len(c) == len(rc) and (c == rc).all() and (dd == rd).all()


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [1, 16, 300, 5000])
def test_device_explicit_random_slides_match_reference(batch):
    """slide_explicit_random (streaming.hpp:129-158; test_streaming.cpp:137-190):
    the drawn evictions, the multiplicity-filtered deletions (in window order)
    and the arrivals equal the reference's for the same engine seed — also
    when FIFO and explicit slides are mixed on one window."""
    a = EdgeStream.rmat(2**8, 20000, seed=6)      # many duplicate arrivals
    b = RefStream.rmat(2**8, 20000, seed=6)
    w, rw = SlidingWindow(a, 0), RefWindow(b)
    rng, rrng = Mt19937_64(11), RefRng(11)
    s, d = a.arrays()
    for i in range(14 if batch > 100 else 30):
        if i % 3 == 2:
            sl, ref = w.slide(batch), rw.slide(batch)
        else:
            sl, ref = w.slide_explicit_random(batch, rng), rw.slide_explicit_random(batch, rrng)
        _same_slide(w, sl, s, d, ref)
    assert w.window_size() == int(__import__("oracle").oracle.ref_lib().ref_window_size(rw.h))


@pytest.mark.gpu
def test_explicit_random_full_batch_replaces_window():
    """test_streaming.cpp:137-150: a full-window batch evicts every old edge."""
    a = EdgeStream.erdos_renyi(64, 0.5, seed=2)
    b = RefStream.erdos_renyi(64, 0.5, seed=2)
    w, rw = SlidingWindow(a, 0), RefWindow(b)
    n0 = w.window_size()
    s, d = a.arrays()
    sl = w.slide_explicit_random(n0, Mt19937_64(5))
    _same_slide(w, sl, s, d, rw.slide_explicit_random(n0, RefRng(5)))
    assert w.window_size() == sl.n_ins
