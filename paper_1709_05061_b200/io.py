"""File formats of the reference (io.hpp:24-181), host side, vectorised.

* key/value pairs: binary little-endian (u64 key, u64 value) records, or
  "key value" text lines (io.hpp:34-67);
* edge streams: "src dst weight ts" text lines under a "# vertices N" header,
  or packed 24-byte binary records (u64 edge key, u64 weight bits, u64 ts)
  after a (magic "pgma1", u64 |V|) header (io.hpp:71-153);
* result vectors: one value per line, or raw binary (io.hpp:157-177).

Doubles render as std::to_chars does (shortest round-trip, fixed or
scientific whichever is shorter, fixed on ties — io.hpp:26-30), so files are
byte-identical to the reference's.  Streams are plain arrays
(:class:`StreamData`); ``EdgeStream`` (the library's generator handle) and
the device window consume them through ``StreamData.to_edge_stream``.
"""
from __future__ import annotations

import math
import re
from dataclasses import dataclass
from decimal import Decimal

import numpy as np

STREAM_MAGIC = 0x70676D6131  # "pgma1" (io.hpp:115)

__all__ = ["StreamData", "format_double", "write_pairs_binary", "read_pairs_binary", "write_pairs_text",
           "read_pairs_text", "write_stream_text", "read_stream_text", "write_stream_binary", "read_stream_binary",
           "read_stream", "write_vector_text", "write_vector_binary"]


@dataclass
class StreamData:
    """EdgeStream (streaming.hpp:27-38): arrival-ordered (src, dst, weight, ts)."""
    num_vertices: int
    src: np.ndarray
    dst: np.ndarray
    weight: np.ndarray
    ts: np.ndarray

    def __len__(self):
        return len(self.src)

    def validate(self):
        """streaming.hpp:31-37"""
        if len(self.ts) > 1 and np.any(self.ts[1:] < self.ts[:-1]):
            raise ValueError("EdgeStream: timestamps must be non-decreasing")

    @classmethod
    def from_edge_stream(cls, stream) -> "StreamData":
        """A generated stream: weights 1.0 (generators.hpp:60,86), ts = arrival index."""
        s, d = stream.arrays()
        return cls(stream.num_vertices, s, d, np.ones(len(s)), np.arange(len(s), dtype=np.uint64))

    def to_edge_stream(self):
        from .pmagraph import EdgeStream
        return EdgeStream.from_arrays(self.num_vertices, self.src, self.dst)


def _open(path, mode):
    # std::runtime_error("cannot open ...") in the reference (io.hpp:35,44,...)
    try:
        return open(path, mode, newline="\n") if "b" not in mode else open(path, mode)
    except OSError:
        raise RuntimeError(f"cannot open {path}" + (" for writing" if "w" in mode else "")) from None


# ---------------------------------------------------------------- doubles
def format_double(v: float) -> str:
    """std::to_chars(double) (io.hpp:26-30): the shortest representation that
    parses back exactly, printf-%f or printf-%e style, %f on a tie."""
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0.0:
        return sign + "0"
    # shortest round-trip digits (Python's repr is shortest round-trip too)
    t = Decimal(repr(abs(v))).normalize().as_tuple()
    digits = "".join(map(str, t.digits))
    e = t.exponent  # value = int(digits) * 10^e
    n = len(digits)
    # %e with precision n - 1
    x = n - 1 + e  # decimal exponent of the leading digit
    mant = digits[0] + ("." + digits[1:] if n > 1 else "")
    sci = f"{mant}e{'-' if x < 0 else '+'}{abs(x):02d}"
    # %f with the fewest fractional digits
    if e >= 0:
        fixed = str(int(abs(v)))  # an integral double prints exactly in %f form
    else:
        frac = -e
        if n > frac:
            fixed = digits[:n - frac] + "." + digits[n - frac:]
        else:
            fixed = "0." + "0" * (frac - n) + digits
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def _fmt_doubles(w: np.ndarray):
    # the generated streams are all 1.0: format each distinct value once
    u, inv = np.unique(w.view(np.uint64), return_inverse=True)
    table = np.array([format_double(x) for x in u.view(np.float64)], dtype=object)
    return table[inv]


# ---------------------------------------------------------------- key/value pairs
def write_pairs_binary(path, keys, values):
    """io.hpp:34-41"""
    rec = np.empty((len(keys), 2), np.uint64)
    rec[:, 0] = keys
    rec[:, 1] = values
    with _open(path, "wb") as f:
        f.write(rec.astype("<u8").tobytes())


def read_pairs_binary(path):
    """io.hpp:43-52: whole 16-byte records; a trailing partial record is ignored."""
    with _open(path, "rb") as f:
        b = f.read()
    n = len(b) // 16
    rec = np.frombuffer(b[:16 * n], dtype="<u8").reshape(n, 2).astype(np.uint64)
    return rec[:, 0].copy(), rec[:, 1].copy()


def write_pairs_text(path, keys, values):
    """io.hpp:54-58"""
    with _open(path, "w") as f:
        f.write("".join(f"{int(k)} {int(v)}\n" for k, v in zip(np.asarray(keys, np.uint64),
                                                              np.asarray(values, np.uint64))))


_U64 = re.compile(r"\+?[0-9]+")


def read_pairs_text(path):
    """io.hpp:60-67: whitespace-separated u64 pairs until the first token that
    is not one (or an odd trailing token)."""
    with _open(path, "r") as f:
        toks = f.read().split()
    vals = []
    for t in toks:
        if not _U64.fullmatch(t) or int(t) >= 1 << 64:
            break
        vals.append(int(t))
    n = len(vals) // 2
    a = np.array(vals[:2 * n], dtype=np.uint64).reshape(n, 2)
    return a[:, 0].copy(), a[:, 1].copy()


# ---------------------------------------------------------------- edge streams
def write_stream_text(path, stream: StreamData):
    """io.hpp:71-78"""
    w = _fmt_doubles(np.ascontiguousarray(stream.weight, np.float64))
    lines = [f"# vertices {int(stream.num_vertices)}\n"]
    lines += [f"{s} {d} {x} {t}\n" for s, d, x, t in zip(stream.src.tolist(), stream.dst.tolist(), w,
                                                          np.asarray(stream.ts, np.uint64).tolist())]
    with _open(path, "w") as f:
        f.write("".join(lines))


_NUM = re.compile(r"[+-]?(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?")


def read_stream_text(path) -> StreamData:
    """io.hpp:80-110: lines "src dst [weight] [ts]" — weight defaults to 1,
    ts to the edge-line index; "# vertices N" pins |V|, else max id + 1;
    other '#' lines and empty lines are skipped."""
    src, dst, wt, ts = [], [], [], []
    nv = None
    with _open(path, "r") as f:
        for line in f.read().split("\n"):
            if not line:
                continue
            if line[0] == "#":
                h = line[1:].split()
                if len(h) >= 2 and h[0] == "vertices" and _U64.fullmatch(h[1]):
                    nv = int(h[1])
                continue
            tok = line.split()
            if len(tok) < 2 or not all(_U64.fullmatch(x) and int(x) < 1 << 32 for x in tok[:2]):
                raise RuntimeError("bad edge line: " + line)
            # istream semantics: a failed extraction stores 0 and stops the
            # line; a numeric prefix is taken and the rest feeds the next one
            w, t = 1.0, len(src)
            if len(tok) >= 3:
                m = _NUM.match(tok[2])
                if not m:
                    w = 0.0
                else:
                    w = float(m.group(0))
                    rest = tok[2][m.end():]
                    nxt = rest if rest else (tok[3] if len(tok) >= 4 else None)
                    if nxt is not None:
                        mt = _U64.match(nxt)
                        t = min(int(mt.group(0)), (1 << 64) - 1) if mt else 0
            src.append(int(tok[0]))
            dst.append(int(tok[1]))
            wt.append(w)
            ts.append(t)
    s = np.array(src, np.uint32)
    d = np.array(dst, np.uint32)
    if nv is None:
        nv = 0 if len(s) == 0 else int(max(s.max(), d.max())) + 1
    return StreamData(nv, s, d, np.array(wt, np.float64), np.array(ts, np.uint64))


def write_stream_binary(path, stream: StreamData):
    """io.hpp:113-127: header (magic, |V|), then (key, weight bits, ts) records."""
    n = len(stream.src)
    rec = np.empty((n, 3), np.uint64)
    rec[:, 0] = (np.asarray(stream.src, np.uint64) << np.uint64(32)) | np.asarray(stream.dst, np.uint64)
    rec[:, 1] = np.ascontiguousarray(stream.weight, np.float64).view(np.uint64)
    rec[:, 2] = stream.ts
    with _open(path, "wb") as f:
        f.write(np.array([STREAM_MAGIC, stream.num_vertices], "<u8").tobytes())
        f.write(rec.astype("<u8").tobytes())


def read_stream_binary(path) -> StreamData:
    """io.hpp:129-146"""
    with _open(path, "rb") as f:
        b = f.read()
    if len(b) < 16 or int.from_bytes(b[:8], "little") != STREAM_MAGIC:
        raise RuntimeError(f"{path} is not an edge-stream file")
    nv = int.from_bytes(b[8:16], "little")
    n = (len(b) - 16) // 24
    rec = np.frombuffer(b[16:16 + 24 * n], dtype="<u8").reshape(n, 3).astype(np.uint64)
    key = rec[:, 0]
    return StreamData(nv, (key >> np.uint64(32)).astype(np.uint32), (key & np.uint64(0xFFFFFFFF)).astype(np.uint32),
                      rec[:, 1].copy().view(np.float64), rec[:, 2].copy())


def read_stream(path) -> StreamData:
    """io.hpp:148-153: binary when the file starts with the magic, else text."""
    with _open(path, "rb") as f:
        head = f.read(8)
    if len(head) == 8 and int.from_bytes(head, "little") == STREAM_MAGIC:
        return read_stream_binary(path)
    return read_stream_text(path)


# ---------------------------------------------------------------- result vectors
def write_vector_text(path, v):
    """io.hpp:157-165: one value per line (doubles via format_double)."""
    a = np.asarray(v)
    if a.dtype.kind == "f":
        body = "".join(x + "\n" for x in _fmt_doubles(a.astype(np.float64)))
    else:
        body = "".join(f"{int(x)}\n" for x in a.tolist())
    with _open(path, "w") as f:
        f.write(body)


def write_vector_binary(path, v):
    """io.hpp:167-172: the raw little-endian array."""
    a = np.ascontiguousarray(v)
    with _open(path, "wb") as f:
        f.write(a.astype(a.dtype.newbyteorder("<")).tobytes())
