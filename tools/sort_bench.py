#!/usr/bin/env python
"""Onesweep radix sort (gpma_sort_by_key_device) timing vs torch.sort (CUB)
on the pipeline's shapes: packed update words (2M keys, 43 + 21 bits; C4:
5.4M keys, 49 bits), and a bulk load (32M (key, index) pairs, 64 bits)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_1709_05061_b200 import pmagraph as pg
    rng = np.random.default_rng(1)
    for n, lo, hi, pay in [(2_000_000, 21, 64, False), (5_400_000, 1, 50, False), (2_000_000, 0, 43, True),
                           (32_000_000, 0, 64, True)]:
        width = min(hi - lo, 63)
        k = rng.integers(0, 2 ** width, n, dtype=np.uint64) << np.uint64(lo)
        dk = torch.from_numpy(k.view(np.int64)).cuda()
        dp = torch.arange(n, dtype=torch.int32, device="cuda") if pay else None
        work = dk.clone()
        wp = dp.clone() if pay else None
        for rep in range(6):
            work.copy_(dk)
            if pay:
                wp.copy_(dp)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pg.sort_by_key_device(work.data_ptr(), wp.data_ptr() if pay else None, n, lo, hi)
            e1.record()
            torch.cuda.synchronize()
            ours = e0.elapsed_time(e1)
        e0.record()
        for _ in range(5):
            torch.sort(dk, stable=True)
        e1.record()
        torch.cuda.synchronize()
        cub = e0.elapsed_time(e1) / 5
        print(f"n={n} bits [{lo},{hi}) payload={pay}: ours {ours * 1e3:.1f} us (incl. sync + copy back), "
              f"torch.sort (CUB, all 64 bits) {cub * 1e3:.1f} us", flush=True)


if __name__ == "__main__":
    main()
