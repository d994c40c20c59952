"""GPU parity of the hand-written data-parallel primitives (csrc/radix.cuh)
against the reference's sort_by_key / exclusive_scan contract
(primitives.hpp:21-84): a STABLE ascending sort by the key bits, payloads
moving with their keys (equal keys keep input order), and out[i] = sum of
in[0..i).  The checker is numpy's stable sort / cumsum on the same inputs.

Sizes cover the one-CTA path (n <= 4096), partial tiles, the multi-tile
onesweep path with look-back across hundreds of tiles, constant digits (the
reference skips them, primitives.hpp:38-46), heavy duplicates (RMAT-like),
and sub-ranges of key bits (the batch pipeline sorts packed words by their
key bits only)."""
import numpy as np
import pytest

from paper_1709_05061_b200 import pmagraph as pg

pytestmark = pytest.mark.gpu


def np_sort(keys, pay, b, e):
    m = np.uint64((1 << (e - b)) - 1) if e - b < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    d = (keys >> np.uint64(b)) & m
    order = np.argsort(d, kind="stable")
    return keys[order], (None if pay is None else pay[order])


def gen(n, kind, rng):
    if kind == "uniform":
        return rng.integers(0, 2 ** 63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
    if kind == "dups":  # few distinct keys: long equal runs, stability visible
        return rng.integers(0, 17, n, dtype=np.uint64) << np.uint64(29)
    if kind == "edges":  # src << 32 | dst with 21-bit ids, skewed sources
        src = (rng.zipf(1.3, n) % (1 << 21)).astype(np.uint64)
        dst = rng.integers(0, 1 << 21, n, dtype=np.uint64)
        return (src << np.uint64(32)) | dst
    if kind == "const_high":  # upper digits constant everywhere
        return np.uint64(0xAB00000000000000) | rng.integers(0, 1 << 20, n, dtype=np.uint64)
    raise ValueError(kind)


@pytest.mark.parametrize("n", [0, 1, 2, 63, 64, 100, 1000, 4095, 4096, 4097, 8192 + 17, 100_003, 1_500_000])
@pytest.mark.parametrize("kind", ["uniform", "dups", "edges"])
def test_sort_by_key_pairs(n, kind):
    rng = np.random.default_rng(n * 7 + len(kind))
    k = gen(n, kind, rng)
    p = np.arange(n, dtype=np.uint32)
    gk, gp = pg.sort_by_key(k, p)
    rk, rp = np_sort(k, p, 0, 64)
    assert (gk == rk).all() and (gp == rp).all()


@pytest.mark.parametrize("n", [3000, 50_000, 2_000_000])
@pytest.mark.parametrize("bits", [(0, 64), (0, 53), (20, 61), (7, 8), (32, 53), (0, 0)])
def test_sort_by_key_bit_ranges_keys_only(n, bits):
    rng = np.random.default_rng(n + bits[0] * 100 + bits[1])
    k = gen(n, "edges", rng)
    gk, _ = pg.sort_by_key(k, None, *bits)
    rk, _ = np_sort(k, None, *bits) if bits[1] > bits[0] else (k, None)
    assert (gk == rk).all()


@pytest.mark.parametrize("n", [4000, 300_000])
def test_sort_constant_digits_skipped(n):
    rng = np.random.default_rng(5)
    k = gen(n, "const_high", rng)
    p = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    gk, gp = pg.sort_by_key(k, p)
    rk, rp = np_sort(k, p, 0, 64)
    assert (gk == rk).all() and (gp == rp).all()


def test_sort_all_equal_keeps_input_order():
    n = 123_457
    k = np.full(n, 42, np.uint64)
    p = np.arange(n, dtype=np.uint32)[::-1].copy()
    gk, gp = pg.sort_by_key(k, p)
    assert (gk == k).all() and (gp == p).all()


def test_sort_device_in_place():
    import torch
    rng = np.random.default_rng(11)
    n = 777_777
    k = gen(n, "edges", rng)
    p = np.arange(n, dtype=np.uint32)
    dk = torch.from_numpy(k.view(np.int64)).cuda()
    dp = torch.from_numpy(p.view(np.int32)).cuda()
    pg.sort_by_key_device(dk.data_ptr(), dp.data_ptr(), n, 0, 64)
    rk, rp = np_sort(k, p, 0, 64)
    assert (dk.cpu().numpy().view(np.uint64) == rk).all()
    assert (dp.cpu().numpy().view(np.uint32) == rp).all()


def test_sort_rejects_bad_bits():
    with pytest.raises(ValueError):
        pg.sort_by_key(np.arange(10, dtype=np.uint64), None, 3, 65)


@pytest.mark.parametrize("n", [1, 7, 2048, 2049, 100_000, 4_194_306])
def test_exclusive_scan(n):
    import torch
    rng = np.random.default_rng(n)
    x = rng.integers(0, 300, n, dtype=np.uint64).astype(np.uint32)
    dx = torch.from_numpy(x.view(np.int32)).cuda()
    dy = torch.empty_like(dx)
    pg.exclusive_scan_device(dx.data_ptr(), dy.data_ptr(), n)
    ref = np.concatenate([[0], np.cumsum(x.astype(np.uint64))[:-1]]).astype(np.uint32)
    assert (dy.cpu().numpy().view(np.uint32) == ref).all()
