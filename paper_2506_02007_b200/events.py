"""Columnar event ingest: the canonical JSON-lines trace
(read_trace) converted once into a columnar binary file, read back
without parsing (memory-mapped columns), and turned into a feature matrix on the device
(es_events_extract: validate_event's invariants, the layer filter, log10 transforms —
SPEC.md:32-70) so that the JSON parser is off the pipeline's path.

Columnar file "ESCOL1" (little endian, every block padded to 8 bytes):
    magic b"ESCOL1\\0\\0" | u64 n | u32 version (1) | u32 n_kinds | kinds: u16 length + utf-8
    columns: layer u8[n] | kind u16[n] | ts_start i64[n] | duration_ns i64[n] | pid i32[n] |
             tid i32[n] | device i32[n] (-1: none) | message_bytes, util_pct, mem_used_mb,
             temp_c, power_w f64[n] (NaN: attribute absent)
Attributes other than these five are not carried by the columnar form.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

LAYERS = {"Cuda": 0, "Python": 1, "Torch": 2, "Nccl": 3, "GpuSample": 4}
LAYER_NAMES = {v: k for k, v in LAYERS.items()}
ATTRS = ("message_bytes", "util_pct", "mem_used_mb", "temp_c", "power_w")
MAGIC = b"ESCOL1\0\0"


@dataclass
class EventColumns:
    """TraceEvent fields as columns; attrs restricted to ATTRS (NaN: absent)."""
    layer: np.ndarray
    kind: np.ndarray
    kinds: List[str]
    ts_start: np.ndarray
    duration_ns: np.ndarray
    pid: np.ndarray
    tid: np.ndarray
    device: np.ndarray
    attrs: Dict[str, np.ndarray] = field(default_factory=dict)

    def __len__(self) -> int:
        return int(self.layer.shape[0])


def _err(name: str, msg: str):
    from . import EventscopeError
    return EventscopeError("Data", name, msg)


def _validate(rec: dict, line: int) -> dict:
    """validate_event: the first violated field, with the line number."""
    for k in ("layer", "kind", "ts_start", "duration_ns", "pid", "tid"):
        if k not in rec:
            raise _err("MissingField", f"line {line}: {k}")
    if rec["layer"] not in LAYERS:
        raise _err("UnknownLayer", f"line {line}: {rec['layer']}")
    if not (isinstance(rec["duration_ns"], int) and rec["duration_ns"] >= 0):
        raise _err("RangeViolation", f"line {line}: duration_ns {rec['duration_ns']}")
    if not (isinstance(rec["ts_start"], int) and rec["ts_start"] > 0):
        raise _err("RangeViolation", f"line {line}: ts_start {rec['ts_start']}")
    a = rec.get("attrs", {}) or {}
    if rec["layer"] == "Nccl":
        if "message_bytes" not in a:
            raise _err("MissingField", f"line {line}: message_bytes")
        if not a["message_bytes"] >= 0:
            raise _err("RangeViolation", f"line {line}: message_bytes {a['message_bytes']}")
    if rec["layer"] == "GpuSample":
        for k, lo, hi, lo_open in (("util_pct", 0, 100, False), ("mem_used_mb", 0, float("inf"), False),
                                   ("temp_c", -50, 150, True)):
            if k not in a:
                raise _err("MissingField", f"line {line}: {k}")
            v = a[k]
            ok = (lo < v < hi) if lo_open else (lo <= v <= hi)
            if not ok:
                raise _err("RangeViolation", f"line {line}: {k} {v}")
    return rec


def read_trace_jsonl(path: str) -> EventColumns:
    """read_trace: one JSON object per line, validated, in file order;
    ParseError / validation errors name the (1-based) line."""
    recs = []
    with open(path, "r", encoding="utf-8") as fh:
        for ln, text in enumerate(fh, 1):
            if not text.strip():
                continue
            try:
                rec = json.loads(text)
            except json.JSONDecodeError as e:
                raise _err("ParseError", f"line {ln}: {e.msg}") from None
            if not isinstance(rec, dict):
                raise _err("ParseError", f"line {ln}: not an object")
            recs.append(_validate(rec, ln))
    return from_records(recs)


def from_records(recs) -> EventColumns:
    n = len(recs)
    kinds: List[str] = []
    kid: Dict[str, int] = {}
    kind = np.empty(n, np.uint16)
    for i, r in enumerate(recs):
        k = r["kind"]
        if k not in kid:
            kid[k] = len(kinds)
            kinds.append(k)
        kind[i] = kid[k]
    attrs = {a: np.array([float((r.get("attrs") or {}).get(a, np.nan)) for r in recs], np.float64) for a in ATTRS}
    return EventColumns(
        layer=np.array([LAYERS[r["layer"]] for r in recs], np.uint8), kind=kind, kinds=kinds,
        ts_start=np.array([r["ts_start"] for r in recs], np.int64),
        duration_ns=np.array([r["duration_ns"] for r in recs], np.int64),
        pid=np.array([r["pid"] for r in recs], np.int32), tid=np.array([r["tid"] for r in recs], np.int32),
        device=np.array([r.get("device", -1) if r.get("device") is not None else -1 for r in recs], np.int32),
        attrs=attrs)


def _pad8(n: int) -> int:
    return (n + 7) & ~7


def write_columnar(cols: EventColumns, path: str) -> None:
    n = len(cols)
    with open(path, "wb") as fh:
        head = bytearray(MAGIC + np.uint64(n).tobytes() + np.uint32(1).tobytes() +
                         np.uint32(len(cols.kinds)).tobytes())
        for k in cols.kinds:
            b = k.encode("utf-8")
            head += np.uint16(len(b)).tobytes() + b
        head += b"\0" * (_pad8(len(head)) - len(head))
        fh.write(head)
        for arr, dt in ((cols.layer, np.uint8), (cols.kind, np.uint16), (cols.ts_start, np.int64),
                        (cols.duration_ns, np.int64), (cols.pid, np.int32), (cols.tid, np.int32),
                        (cols.device, np.int32)) + tuple((cols.attrs.get(a, np.full(n, np.nan)), np.float64)
                                                         for a in ATTRS):
            b = np.ascontiguousarray(arr, dt).tobytes()
            fh.write(b + b"\0" * (_pad8(len(b)) - len(b)))


def read_columnar(path: str) -> EventColumns:
    """Memory-mapped columns of an ESCOL1 file (no parsing; pages are read on first use)."""
    mm = np.memmap(path, dtype=np.uint8, mode="r")
    if bytes(mm[:8]) != MAGIC:
        raise _err("ParseError", f"{path}: not an ESCOL1 file")
    n = int(np.frombuffer(mm[8:16], np.uint64)[0])
    nk = int(np.frombuffer(mm[20:24], np.uint32)[0])
    off = 24
    kinds = []
    for _ in range(nk):
        ln = int(np.frombuffer(mm[off:off + 2], np.uint16)[0])
        kinds.append(bytes(mm[off + 2:off + 2 + ln]).decode("utf-8"))
        off += 2 + ln
    off = _pad8(off)
    out = []
    for dt in (np.uint8, np.uint16, np.int64, np.int64, np.int32, np.int32, np.int32) + (np.float64,) * len(ATTRS):
        size = n * np.dtype(dt).itemsize
        out.append(np.frombuffer(mm, dtype=dt, count=n, offset=off))
        off += _pad8(size)
    if off > mm.shape[0]:
        raise _err("ParseError", f"{path}: truncated")
    return EventColumns(out[0], out[1], kinds, out[2], out[3], out[4], out[5], out[6],
                        dict(zip(ATTRS, out[7:])))


class _EventCols(C.Structure):
    _fields_ = [("layer", C.c_void_p), ("ts_start", C.c_void_p), ("duration_ns", C.c_void_p),
                ("message_bytes", C.c_void_p), ("util_pct", C.c_void_p), ("mem_used_mb", C.c_void_p),
                ("temp_c", C.c_void_p)]


def extract_features(cols: EventColumns, layer: str, ctx=None):
    """extract_features on the device (es_events_extract): returns the
    feature Dataset of `layer` (rows in event order) and the source event of each row.
    Standardization is run_pipeline's (train-split statistics)."""
    from . import Dataset, _check, default_context
    c = ctx or default_context()
    n = len(cols)

    def p(a):
        if a is None:
            return None
        a = np.ascontiguousarray(a)
        keep.append(a)
        return a.ctypes.data

    keep: list = []
    ec = _EventCols(p(cols.layer), p(cols.ts_start), p(cols.duration_ns), p(cols.attrs.get("message_bytes")),
                    p(cols.attrs.get("util_pct")), p(cols.attrs.get("mem_used_mb")), p(cols.attrs.get("temp_c")))
    h = C.c_void_p()
    idx = np.empty(max(n, 1), np.int64)
    bad = C.c_int64(-1)
    _check(c._lib.es_events_extract(c.handle, C.byref(ec), C.c_int64(n), C.c_int32(LAYERS[layer]), C.byref(h),
                                    C.c_void_p(idx.ctypes.data), C.byref(bad)))
    ds = Dataset(c, h)
    return ds, idx[:ds.n_local].copy()
