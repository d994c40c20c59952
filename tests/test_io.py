"""CPU: the file formats (io.hpp) — files written here are byte-identical to
the reference's, and each side parses the other's files to the same data."""
import struct

import numpy as np
import pytest

from oracle import oracle
from oracle.oracle import RefIO, RefStream
from paper_1709_05061_b200 import io as pio
from paper_1709_05061_b200.pmagraph import EdgeStream

pytestmark = pytest.mark.skipif(not oracle.have_ref(), reason="reference oracle not built")


def _bytes(p):
    with open(p, "rb") as f:
        return f.read()


def test_format_double_matches_to_chars():
    rng = np.random.default_rng(3)
    vals = [0.0, -0.0, 1.0, -1.0, 0.5, 1e5, 1e16, 1e15, 123456.789, 1e-7, 1e-4, 1e23, 5e-324, 1.7976931348623157e308,
            0.1, 1 / 3, 2.0**60, -(2.0**70), float("inf"), -float("inf"), float("nan")]
    vals += list(rng.standard_normal(2000) * 10.0 ** rng.integers(-30, 30, 2000))
    vals += [struct.unpack("d", struct.pack("Q", int(x)))[0] for x in rng.integers(0, 2**64 - 1, 3000, np.uint64)]
    vals += [x / 1000 for x in range(1000)] + [10.0**k for k in range(-300, 300, 7)]
    for v in vals:
        assert pio.format_double(v) == RefIO.format_double(v), v


@pytest.mark.parametrize("text", [False, True])
def test_pairs_round_trip(tmp_path, text):
    rng = np.random.default_rng(5)
    k = np.sort(rng.integers(0, 2**64 - 1, 3000, np.uint64, endpoint=True))
    v = rng.integers(0, 2**64 - 1, 3000, np.uint64, endpoint=True)
    ours, ref = tmp_path / "ours", tmp_path / "ref"
    (pio.write_pairs_text if text else pio.write_pairs_binary)(ours, k, v)
    RefIO.write_pairs(ref, k, v, text)
    assert _bytes(ours) == _bytes(ref)
    rk, rv = (pio.read_pairs_text if text else pio.read_pairs_binary)(ref)
    assert (rk == k).all() and (rv == v).all()
    qk, qv = RefIO.read_pairs(ours, text)
    assert (qk == k).all() and (qv == v).all()


def _stream(seed=1):
    st = RefStream.rmat(2**10, 6000, seed)
    st.shuffle(2)
    s, d, w, ts = st.arrays()
    rng = np.random.default_rng(seed)
    w = np.where(rng.random(len(s)) < 0.3, rng.standard_normal(len(s)) * 10.0 ** rng.integers(-8, 8, len(s)), w)
    ts = np.cumsum(rng.integers(0, 3, len(s))).astype(np.uint64)
    return pio.StreamData(2**10, s, d, w, ts)


@pytest.mark.parametrize("text", [False, True])
def test_stream_files_match_reference(tmp_path, text):
    sd = _stream()
    ours, ref = tmp_path / "ours", tmp_path / "ref"
    (pio.write_stream_text if text else pio.write_stream_binary)(ours, sd)
    RefIO.write_stream(ref, sd.num_vertices, sd.src, sd.dst, sd.weight, sd.ts, text)
    assert _bytes(ours) == _bytes(ref)
    for mode, fn in ((0, pio.read_stream), (2 - int(text), pio.read_stream_text if text else pio.read_stream_binary)):
        got = fn(ref)
        nv, s, d, w, ts = RefIO.read_stream(ours, mode)
        assert got.num_vertices == nv == sd.num_vertices
        for a, b, c in ((got.src, s, sd.src), (got.dst, d, sd.dst), (got.ts, ts, sd.ts)):
            assert (a == b).all() and (a == c).all()
        assert (got.weight.view(np.uint64) == w.view(np.uint64)).all()
        assert (w.view(np.uint64) == sd.weight.view(np.uint64)).all()
    got.validate()


def test_stream_text_defaults_and_errors(tmp_path):
    p = tmp_path / "s.txt"
    p.write_text("# a comment\n0 1\n\n2 3 0.25\n4 5 2 9\n7 1 1.5e3 11\n6 6 abc\n")
    got = pio.read_stream_text(p)
    nv, s, d, w, ts = RefIO.read_stream(p, 1)
    assert got.num_vertices == nv == 8  # max id + 1 without a header
    assert (got.src == s).all() and (got.dst == d).all() and (got.ts == ts).all()
    assert (got.weight == w).all() and list(w) == [1.0, 0.25, 2.0, 1500.0, 0.0]
    p.write_text("# vertices 100\n1 2\n")
    assert pio.read_stream(p).num_vertices == RefIO.read_stream(p)[0] == 100
    p.write_text("1 2\nbad\n")
    with pytest.raises(RuntimeError, match="bad edge line: bad"):
        pio.read_stream_text(p)
    with pytest.raises(oracle.OracleError, match="bad edge line"):
        RefIO.read_stream(p, 1)
    p.write_bytes(b"\x00" * 24)
    with pytest.raises(RuntimeError, match="is not an edge-stream file"):
        pio.read_stream_binary(p)
    with pytest.raises(oracle.OracleError, match="is not an edge-stream file"):
        RefIO.read_stream(p, 2)
    with pytest.raises(RuntimeError, match="cannot open"):
        pio.read_stream(tmp_path / "missing")


def test_generated_stream_export(tmp_path):
    """A library-generated stream exports as the reference's generator output."""
    a = EdgeStream.rmat(2**9, 3000, seed=4).shuffle(2)
    b = RefStream.rmat(2**9, 3000, 4)
    b.shuffle(2)
    ours, ref = tmp_path / "ours", tmp_path / "ref"
    sd = pio.StreamData.from_edge_stream(a)
    pio.write_stream_binary(ours, sd)
    s, d, w, ts = b.arrays()
    RefIO.write_stream(ref, 2**9, s, d, w, ts)
    assert _bytes(ours) == _bytes(ref)
    back = pio.read_stream(ours).to_edge_stream()
    s2, d2 = back.arrays()
    assert (s2 == s).all() and (d2 == d).all()


@pytest.mark.parametrize("text", [False, True])
@pytest.mark.parametrize("dtype", [np.float64, np.uint32, np.uint64])
def test_vectors_match_reference(tmp_path, text, dtype):
    rng = np.random.default_rng(9)
    v = (rng.standard_normal(500) * 1e3 if dtype == np.float64
         else rng.integers(0, np.iinfo(dtype).max, 500, dtype, endpoint=True)).astype(dtype)
    ours, ref = tmp_path / "ours", tmp_path / "ref"
    (pio.write_vector_text if text else pio.write_vector_binary)(ours, v)
    RefIO.write_vector(ref, v, text)
    assert _bytes(ours) == _bytes(ref)
