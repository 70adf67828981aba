"""PATARR01 ArrayFile: layout, invariants, bit-exact round trips.

The reference never implemented the container, so the oracle here is the
SPEC text itself: the expected bytes are assembled by hand with ``struct``.
"""

import json
import os
import struct

import numpy as np
import pytest

from paper_1501_02946_b200 import DataValidationError, ParameterError
from paper_1501_02946_b200 import arrayfile as af


def _hand_made(values, spacing, axes):
    hdr = {"axes": list(axes), "byte_order": "LE", "dims": list(values.shape), "dtype": "f64", "layout": "C",
           "spacing": [float(s) for s in spacing]}
    js = json.dumps(hdr, separators=(",", ":"), sort_keys=True).encode()
    return b"PATARR01" + struct.pack("<Q", len(js)) + js + values.astype("<f8").tobytes()


def test_writer_emits_the_specified_bytes(tmp_path):
    v = np.arange(24, dtype=np.float64).reshape(2, 3, 4) * 0.25 - 1.0
    p = tmp_path / "a.patarr"
    af.write_array(p, v, spacing=(1e-4, 2e-4, 3e-8), axes=("x", "y", "t"))
    assert p.read_bytes() == _hand_made(v, (1e-4, 2e-4, 3e-8), ("x", "y", "t"))


def test_round_trip_is_bit_exact(tmp_path):
    rng = np.random.default_rng(3)
    v = rng.standard_normal((5, 7, 9))
    v[0, 0, :3] = [np.inf, -0.0, 5e-324]
    p1, p2 = tmp_path / "1.patarr", tmp_path / "2.patarr"
    af.write_array(p1, v, spacing=(1, 2, 3), axes=("a", "b", "c"), meta={"seed": 3})
    got, h = af.read_array(p1)
    assert got.tobytes() == v.tobytes()
    assert h.dims == (5, 7, 9) and h.spacing == (1.0, 2.0, 3.0) and h.axes == ("a", "b", "c")
    assert h.meta == {"seed": 3}
    af.write_array(p2, got, spacing=h.spacing, axes=h.axes, meta=h.meta)   # write -> read -> write
    assert p1.read_bytes() == p2.read_bytes()


def test_memmap_reader_and_empty_arrays(tmp_path):
    v = np.linspace(0, 1, 60).reshape(3, 4, 5)
    p = tmp_path / "m.patarr"
    af.write_array(p, v)
    mm, h = af.open_array(p)
    assert h.axes == ("axis0", "axis1", "axis2")
    np.testing.assert_array_equal(mm[2], v[2])
    af.write_array(tmp_path / "e.patarr", np.zeros((0, 4)))
    e, h = af.read_array(tmp_path / "e.patarr")
    assert e.shape == (0, 4)


@pytest.mark.parametrize("corrupt, msg", [
    (lambda b: b"PATARR02" + b[8:], "magic"),
    (lambda b: b[:-8], "payload size"),
    (lambda b: b + b"\0" * 8, "payload size"),
    (lambda b: b[:5], "truncated"),
    (lambda b: b.replace(b'"LE"', b'"BE"'), "byte_order"),
    (lambda b: b.replace(b'"f64"', b'"f32"'), "dtype"),
    (lambda b: b.replace(b'"layout":"C"', b'"layout":"F"'), "layout"),
    (lambda b: b[:8] + struct.pack("<Q", 1 << 40) + b[16:], "exceeds"),
    (lambda b: b.replace(b'{"axes"', b'["axes"'), "JSON"),
])
def test_invariant_violations_raise_data_validation_error(tmp_path, corrupt, msg):
    v = np.ones((2, 3))
    p = tmp_path / "c.patarr"
    p.write_bytes(corrupt(_hand_made(v, (1, 1), ("x", "t"))))
    with pytest.raises(DataValidationError, match=msg):
        af.read_array(p)


def test_writer_validates_arguments(tmp_path):
    with pytest.raises(ParameterError):
        af.write_array(tmp_path / "x.patarr", np.ones((2, 3)), spacing=(1.0,))
