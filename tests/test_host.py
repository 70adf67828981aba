"""Host-side logic of the drop-in boundary (no GPU compute)."""

import ctypes
import os

import numpy as np
import pytest

import paper_1501_02946_b200 as pb
from paper_1501_02946_b200 import _lib, synth


def _lib_or_skip():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("CUDA library not built (run __graft_entry__.build())")
    return _lib.load()


def test_library_exports_every_header_symbol():
    lib = _lib_or_skip()
    syms = _lib.header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing
    # every exported symbol has a ctypes signature in the shim
    assert set(syms) == set(_lib._SIGS)


def test_library_metadata_calls():
    lib = _lib_or_skip()
    assert b"sm_100a" in lib.patfft_version()
    assert lib.patfft_nedner_stage_name(0) == b"spread"
    assert lib.patfft_nedner_stage_name(4) == b"inverse"


def test_window_spec_mirrors_reference_validation():
    with pytest.raises(pb.ParameterError):
        pb.WindowSpec(c=1.0)
    with pytest.raises(pb.ParameterError):
        pb.WindowSpec(K=0)
    with pytest.raises(pb.ParameterError):
        pb.WindowSpec(K=2.5)
    with pytest.raises(pb.ParameterError):
        pb.WindowSpec(alpha=3.0)      # <= pi
    with pytest.raises(pb.ParameterError):
        pb.WindowSpec(alpha=20.0)     # >= pi(2c-1)
    with pytest.raises(pb.ParameterError):
        pb.WindowSpec(beta=-1.0)
    r = pb.WindowSpec().resolved(2.0)
    assert r.alpha == pytest.approx(9.41535318280861)
    assert r.beta == pytest.approx(2.9813866459901393)
    assert isinstance(pb.ParameterError("x"), ValueError)
    assert isinstance(pb.DataValidationError("x"), ValueError)


def _rec(**over):
    s = synth.make_3d(3, 8, 16, 20e-9, "jittered", 1)
    kw = dict(positions=s.positions, weights=s.weights, samples=s.samples, dt=s.dt,
              sound_speed=s.sound_speed, dx=s.dx, n_lateral=s.n_lateral)
    kw.update(over)
    return kw


def test_sensor_record_validation_mirrors_reference():
    pb.SensorRecord(**_rec())
    with pytest.raises(pb.DataValidationError, match="weights sum"):
        kw = _rec()
        pb.SensorRecord(**_rec(weights=kw["weights"] * 1.01))
    with pytest.raises(pb.DataValidationError, match="even N_t"):
        kw = _rec()
        pb.SensorRecord(**_rec(samples=kw["samples"][:, :15]))
    with pytest.raises(pb.DataValidationError, match="aperture"):
        kw = _rec()
        p = kw["positions"].copy()
        p[0, 0] = 10 * kw["dx"] * 8
        pb.SensorRecord(**_rec(positions=p))
    with pytest.raises(pb.DataValidationError, match="positive"):
        pb.SensorRecord(**_rec(dt=0.0))
    with pytest.raises(pb.DataValidationError, match="even"):
        pb.SensorRecord(**_rec(n_lateral=(7, 8)))
    with pytest.raises(pb.DataValidationError, match="sensor count"):
        kw = _rec()
        pb.SensorRecord(**_rec(weights=kw["weights"][:-1]))


def test_reconstruct_argument_errors_precede_device():
    rec = pb.SensorRecord(**_rec())
    with pytest.raises(pb.ParameterError):
        pb.reconstruct_nedner(rec, upsample=0)
    with pytest.raises(pb.ParameterError):
        pb.reconstruct_nedner(rec, upsample=1.5)
    with pytest.raises(pb.ParameterError):
        pb.reconstruct_nedner(rec, out_dims=(7, 8))
    with pytest.raises(pb.ParameterError):
        pb.reconstruct_nedner(rec, out_dims=(8,))


def test_kappa_and_amplitude_known_answers():
    # SPEC.md:147-158
    assert pb.kappa(0.0, 5.0) == 5.0
    assert pb.kappa(np.array([3.0, 0.0]), 4.0) == 5.0
    assert pb.kappa(np.array([3.0, 0.0]), -4.0) == -5.0
    assert pb.amplitude_factor(0.0, 3.0) == 2.0
    assert pb.amplitude_factor(2.0, 0.0) == 0.0
    assert pb.amplitude_factor(3.0, 4.0) == pytest.approx(1.6)


def test_no_cpu_fallback_without_gpu(gpu_available):
    if gpu_available:
        pytest.skip("GPU present")
    _lib_or_skip()
    rec = pb.SensorRecord(**_rec())
    with pytest.raises(pb.DeviceError):
        pb.reconstruct_nedner(rec)


def test_product_package_never_imports_oracle():
    root = os.path.dirname(pb.__file__)
    for dirpath, _, files in os.walk(root):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f


def test_desc_struct_layout_matches_header():
    # int32 n_lat, int32[2], int32 x3, double[2], double, int32, double, double
    d = _lib.NednerDesc
    assert d.lat_ratio.offset == 24
    assert d.spec_c.offset == 40
    assert d.spec_K.offset == 48
    assert d.spec_alpha.offset == 56
    assert ctypes.sizeof(d) == 72


def test_output_pool_never_hands_out_a_reachable_volume():
    """NedNerPlan._fresh_out recycles an output buffer only after the caller
    dropped the array AND every view of it (lease lifetime via weakref.finalize,
    no reference-count heuristics)."""
    import gc

    from paper_1501_02946_b200.recon import NedNerPlan

    class FakePlan:
        out_shape = (3, 4, 5)
        _OUT_POOL_SIZE = 2

    p = FakePlan()
    fresh = NedNerPlan._fresh_out.__get__(p)
    a = fresh()
    assert a.flags.writeable and a.flags.c_contiguous and a.shape == p.out_shape
    a[...] = 1.0
    view = a[1]                      # a view keeps the buffer reachable
    del a
    gc.collect()
    b = fresh()
    c = fresh()                      # pool full of live results: an unpooled array
    for x in (b, c):
        assert not np.shares_memory(x, view)
    b[...] = 2.0
    assert np.all(view == 1.0)
    held = {"field": pb.ScalarField(b, (1.0, 1.0, 1.0))}  # a ScalarField holding the result also counts
    del b
    gc.collect()
    d = fresh()
    assert not np.shares_memory(d, held["field"].values) and not np.shares_memory(d, view)
    del d, view, c
    gc.collect()
    e = fresh()                      # everything dropped: a pooled buffer comes back
    assert any(np.shares_memory(e, s[0]) for s in p._out_pool)
