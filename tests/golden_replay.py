"""Replay the committed golden fixtures (tests/golden/*.npz, generated from
the unmodified reference by tests/golden/make_golden.py) through any
implementation that offers the reference interface."""
import hashlib
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
STAT_FIELDS = ["batch_size", "rounds", "slot_writes", "grow_events", "shrink_events", "deletes_missed",
               "tombstones_added", "num_touched_ranges", "resized"]


def load(name):
    return np.load(os.path.join(GOLDEN, name))


def slot_hash(k, v, s):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(k, np.uint64).tobytes())
    h.update(np.ascontiguousarray(v, np.uint64).tobytes())
    h.update(np.ascontiguousarray(s, np.uint8).tobytes())
    return h.hexdigest()


def stats_vector(d):
    return np.array([d["batch_size"], d["rounds"], d["slot_writes"], d["grow_events"], d["shrink_events"],
                     d["deletes_missed"], d["tombstones_added"], d["num_touched_ranges"], int(d["resized"])],
                    np.uint64)


def window_slides(z):
    """Yield (index, ins_src, ins_dst, del_src, del_dst) of the stored slides."""
    s = z["stream_src"].astype(np.uint32)
    d = z["stream_dst"].astype(np.uint32)
    cursor = (len(s) + 1) // 2
    i = 0
    while f"s{i}_stats" in z:
        n = int(z[f"s{i}_n_ins"])
        yield i, s[cursor:cursor + n], d[cursor:cursor + n], z[f"s{i}_del_src"].astype(np.uint32), \
            z[f"s{i}_del_dst"].astype(np.uint32)
        cursor += n
        i += 1
