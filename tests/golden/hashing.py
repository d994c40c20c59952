"""Parity digests shared by the fixture generator and the GPU tests.

slot_chunk_hashes restates the device digest pma_slot_hash (csrc/pma.cu
k_slot_hash) in numpy: slot i contributes
    mix(key + mix(value ^ (i * 0x9E3779B97F4A7C15 + state)))
(mix = the splitmix64 finaliser, all arithmetic mod 2^64) and a chunk's hash
is the wrapping sum over its slots.  vec_hash digests any integer vector
(row offsets, BFS distances, CC labels, touched ranges) the same way.
"""
from __future__ import annotations

import numpy as np

PHI = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def mix(x):
    with np.errstate(over="ignore"):
        x = (x ^ (x >> np.uint64(30))) * M1
        x = (x ^ (x >> np.uint64(27))) * M2
        return x ^ (x >> np.uint64(31))


def slot_chunk_hashes(keys, vals, states, chunk: int, block: int = 1 << 22):
    """Per-chunk digest of a slot array (chunk a power of two)."""
    cap = len(keys)
    out = np.zeros(cap // chunk, np.uint64)
    with np.errstate(over="ignore"):
        for b in range(0, cap, block):  # bounded temporaries at C4's 2^29 slots
            e = min(cap, b + block)
            i = np.arange(b, e, dtype=np.uint64)
            a = i * PHI + states[b:e].astype(np.uint64)
            h = mix(keys[b:e].astype(np.uint64) + mix(vals[b:e].astype(np.uint64) ^ a))
            if chunk >= e - b:
                out[b // chunk] += h.sum(dtype=np.uint64)
            else:
                out[b // chunk:e // chunk] += h.reshape(-1, chunk).sum(axis=1, dtype=np.uint64)
    return out


def vec_hash(x) -> str:
    """Order-dependent digest of an integer vector, as 16 hex digits."""
    x = np.ascontiguousarray(x).astype(np.uint64).ravel()
    with np.errstate(over="ignore"):
        i = np.arange(len(x), dtype=np.uint64)
        h = mix(x + mix(i * PHI + np.uint64(len(x))))
        return f"{int(h.sum(dtype=np.uint64)):016x}"
