"""PATARR01 array files and streamed multi-frame reconstruction.

The reference's SPEC defines the container its CLI would exchange arrays in
(``[TYPE] ArrayFile``; invariants at
SPEC.md:486 "array files round-trip bit-exactly", exit codes at 487); the
reference package itself never implemented it.  Layout,
all integers little-endian:

    offset 0   8 bytes   magic b"PATARR01"
    offset 8   8 bytes   uint64 n = byte length of the JSON header
    offset 16  n bytes   UTF-8 JSON object:
                         {"dtype": "f64", "byte_order": "LE", "layout": "C",
                          "dims": [...], "spacing": [...], "axes": [...]}
                         plus optional free-form keys (kept verbatim in "meta")
    offset 16+n          prod(dims) * 8 bytes of float64 LE payload, C order

Reading validates every invariant (magic, dtype/byte order/layout, payload
size == prod(dims) * 8) and raises ``DataValidationError`` otherwise.

``reconstruct_frames_file`` is the config-5 ingest path: a file of shape
(frames, M, N_t) sharing one sensor layout is memory-mapped and streamed
frame by frame through one ``NedNerPlan`` (the C ABI releases the GIL, so a
reader thread fetches frame k+1 from disk while the GPU reconstructs frame
k), and the volumes are written to an output PATARR01 file of shape
(frames, *volume).
"""

from __future__ import annotations

import json
import os
import struct
import threading
from dataclasses import dataclass, field

import numpy as np

from .errors import DataValidationError, ParameterError

__all__ = ["MAGIC", "ArrayHeader", "write_array", "read_array", "open_array", "reconstruct_frames_file"]

MAGIC = b"PATARR01"
_PREFIX = struct.Struct("<8sQ")
_REQUIRED = {"dtype": "f64", "byte_order": "LE", "layout": "C"}


@dataclass
class ArrayHeader:
    dims: tuple
    spacing: tuple
    axes: tuple
    meta: dict = field(default_factory=dict)
    data_offset: int = 0

    def to_json(self) -> bytes:
        doc = dict(_REQUIRED)
        doc.update(dims=[int(n) for n in self.dims], spacing=[float(s) for s in self.spacing],
                   axes=[str(a) for a in self.axes])
        for k, v in self.meta.items():
            if k not in doc:
                doc[k] = v
        return json.dumps(doc, separators=(",", ":"), sort_keys=True).encode("utf-8")


def _header(dims, spacing, axes, meta) -> ArrayHeader:
    dims = tuple(int(n) for n in dims)
    if any(n < 0 for n in dims):
        raise ParameterError("array dims must be non-negative")
    spacing = tuple(float(s) for s in (spacing if spacing is not None else (1.0,) * len(dims)))
    axes = tuple(str(a) for a in (axes if axes is not None else (f"axis{i}" for i in range(len(dims)))))
    if len(spacing) != len(dims) or len(axes) != len(dims):
        raise ParameterError("spacing and axes must have one entry per dimension")
    return ArrayHeader(dims, spacing, axes, dict(meta or {}))


def write_array(path, values, spacing=None, axes=None, meta=None) -> ArrayHeader:
    """Write ``values`` (cast to float64 LE, C order) as a PATARR01 file."""
    arr = np.ascontiguousarray(values, dtype="<f8")
    h = _header(arr.shape, spacing, axes, meta)
    js = h.to_json()
    with open(path, "wb") as f:
        f.write(_PREFIX.pack(MAGIC, len(js)))
        f.write(js)
        f.write(arr.tobytes(order="C"))
    h.data_offset = _PREFIX.size + len(js)
    return h


def read_header(path) -> ArrayHeader:
    """Parse and validate the header (SPEC.md:449-451 invariants)."""
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        pre = f.read(_PREFIX.size)
        if len(pre) != _PREFIX.size:
            raise DataValidationError("truncated PATARR01 file")
        magic, n = _PREFIX.unpack(pre)
        if magic != MAGIC:
            raise DataValidationError("not a PATARR01 file (bad magic)")
        if n > size - _PREFIX.size:
            raise DataValidationError("PATARR01 header length exceeds the file")
        try:
            doc = json.loads(f.read(n).decode("utf-8"))
        except (UnicodeDecodeError, json.JSONDecodeError) as e:
            raise DataValidationError(f"PATARR01 header is not valid JSON: {e}") from None
    if not isinstance(doc, dict):
        raise DataValidationError("PATARR01 header must be a JSON object")
    for k, v in _REQUIRED.items():
        if doc.get(k) != v:
            raise DataValidationError(f"PATARR01 header {k!r} must be {v!r}, got {doc.get(k)!r}")
    try:
        h = _header(doc["dims"], doc.get("spacing"), doc.get("axes"),
                    {k: v for k, v in doc.items() if k not in ("dims", "spacing", "axes", *_REQUIRED)})
    except (KeyError, TypeError, ValueError, ParameterError) as e:
        raise DataValidationError(f"bad PATARR01 header: {e}") from None
    h.data_offset = _PREFIX.size + n
    if size - h.data_offset != int(np.prod(h.dims, dtype=np.int64)) * 8:
        raise DataValidationError("PATARR01 payload size does not match prod(dims) * 8")
    return h


def open_array(path):
    """(read-only float64 memmap of the payload, header) -- no copy."""
    h = read_header(path)
    if int(np.prod(h.dims, dtype=np.int64)) == 0:
        return np.zeros(h.dims), h
    return np.memmap(path, dtype="<f8", mode="r", offset=h.data_offset, shape=h.dims, order="C"), h


def read_array(path):
    """(float64 array, header), fully loaded."""
    mm, h = open_array(path)
    return np.array(mm, dtype=np.float64), h


def reconstruct_frames_file(plan, in_path, out_path, frames: slice | None = None) -> ArrayHeader:
    """Stream the frames of a (frames, M, N_t) PATARR01 file through ``plan``.

    ``plan`` is a :class:`~paper_1501_02946_b200.recon.NedNerPlan` built for
    the file's sensor layout.  Output: PATARR01 (frames, *volume) float64.
    Disk reads of frame k+1 overlap the GPU reconstruction of frame k.
    """
    data, h = open_array(in_path)
    if len(h.dims) != 3:
        raise DataValidationError("frame file must have dims (frames, sensors, time)")
    n_frames, m, nt = h.dims
    if (m, nt) != (plan.n_sensors, plan.n_time):
        raise ParameterError(f"plan built for {(plan.n_sensors, plan.n_time)} samples, file has {(m, nt)}")
    idx = range(n_frames)[frames] if frames is not None else range(n_frames)
    shape = tuple(int(n) for n in plan.out_shape)
    meta = {"source": os.path.basename(str(in_path)), "frames": [int(i) for i in idx]}
    oh = _header((len(idx),) + shape, (1.0,) + tuple(plan.spacing),
                 ("frame",) + tuple(f"x{i}" for i in range(len(shape) - 1)) + ("z",), meta)
    js = oh.to_json()
    out = np.empty(shape, dtype=np.float64)
    nxt = [None]

    def fetch(k):
        nxt[0] = np.array(data[k], dtype=np.float64) if k is not None else None

    with open(out_path, "wb") as f:
        f.write(_PREFIX.pack(MAGIC, len(js)))
        f.write(js)
        order = list(idx)
        fetch(order[0] if order else None)
        for i in range(len(order)):
            cur = nxt[0]
            th = threading.Thread(target=fetch, args=(order[i + 1] if i + 1 < len(order) else None,))
            th.start()
            _, _, nonfinite = plan.execute_checked(cur, out=out)
            th.join()
            if nonfinite:  # the ScalarField finiteness rule (recon.py:62-63), per frame
                raise DataValidationError(f"frame {order[i]}: field values must be finite "
                                          f"({nonfinite} non-finite voxels)")
            f.write(np.ascontiguousarray(out, dtype="<f8").tobytes(order="C"))
    oh.data_offset = _PREFIX.size + len(js)
    return oh
