"""GPU parity: the sm_100a path through the C ABI vs the reference's outputs.

Bar (BASELINE.json north_star): relative L2 <= 1e-4 on the reconstructed
volume (float32/complex64 compute vs the float64 reference).
"""

import os

import numpy as np
import pytest

import paper_1501_02946_b200 as pb
from conftest import GOLDEN, golden_recon_files, golden_spec, rel_l2
from oracle import nedner_oracle as O
from paper_1501_02946_b200 import synth

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _record(g):
    return pb.SensorRecord(g["positions"], g["weights"], g["samples"], float(g["dt"]), float(g["sound_speed"]),
                           float(g["dx"]), tuple(int(n) for n in g["n_lateral"]))


@pytest.mark.parametrize("path", golden_recon_files(), ids=os.path.basename)
def test_gpu_matches_reference_golden(path):
    # recon_3d_spec_c25 (c = 2.5, explicit alpha = 12, beta = 2.3) loses accuracy
    # at the GPU's power-of-two oversampled lengths; it is accurate at the
    # reference's own lengths, so the plan resolves the window for its own
    # oversampling and must still match the reference golden
    g = np.load(path)
    c, K, a, b = golden_spec(g)
    spec = pb.WindowSpec(c=c, K=K, alpha=a, beta=b)
    f = pb.reconstruct_nedner(_record(g), out_dims=tuple(int(n) for n in g["out_dims"]),
                              upsample=int(g["upsample"]), spec=spec)
    assert f.values.shape == g["values"].shape
    assert f.values.dtype == np.float64
    np.testing.assert_allclose(f.spacing, g["spacing"], rtol=1e-15)
    err = rel_l2(f.values, g["values"])
    print(f"{os.path.basename(path)}: rel-L2 {err:.3e}")
    assert err <= TOL
    assert f.meta["imag_residual"] <= 1e-9


def test_gpu_inaccurate_window_runs_on_reference_lengths():
    """alpha = 12, beta = 0.5 at c = 2.5 is admissible (nufft.py:119-131) but inaccurate: the
    reference's own answer is 1e-3 off the exact transform and depends on its oversampled grid
    length (40 here; the GPU's power of two would be 64).  The plan therefore runs on the
    reference's lengths (csrc/reflen.cu) and reproduces that answer; it used to be refused."""
    g = np.load(os.path.join(GOLDEN, "recon_3d_badwin_c25.npz"))
    spec = pb.WindowSpec(c=2.5, K=6, alpha=12.0, beta=0.5)
    s = _record(g)
    plan = pb.NedNerPlan(s.positions, s.weights, s.samples.shape[1], s.dt, s.sound_speed, s.dx, s.n_lateral, spec=spec)
    info = plan.window_info()
    assert info["lateral"]["c_eff"] == 2.5 and info["lateral"]["alpha"] == 12.0 and info["lateral"]["beta"] == 0.5
    assert info["ner"]["c_eff"] == 2.5  # 2 N_t = 64 -> 160, not 256
    got, _ = plan.execute(s.samples)
    err = rel_l2(got, g["values"])
    exact, _ = O.reconstruct_nedner(g["positions"], g["weights"], g["samples"], float(g["dt"]), float(g["sound_speed"]),
                                    float(g["dx"]), tuple(int(n) for n in g["n_lateral"]))
    off = rel_l2(g["values"], exact)
    print(f"inaccurate window on the reference's lengths: rel-L2 vs reference {err:.3e} "
          f"(the reference is {off:.3e} from the exact transform)")
    assert err <= TOL and off > 5 * TOL


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_gpu_matches_oracle_on_baseline_configs(name):
    s = synth.CONFIGS[name]()
    f = pb.reconstruct_nedner(s.as_record())
    want, _ = O.reconstruct_nedner(s.positions, s.weights, s.samples, s.dt, s.sound_speed, s.dx, s.n_lateral)
    err = rel_l2(f.values, want)
    print(f"{name}: rel-L2 {err:.3e}")
    assert err <= TOL


def test_gpu_zero_data_zero_image():
    s = synth.make_3d(5, 32, 64, 20e-9, "uniform", 2)
    r = s.as_record()
    r.samples = np.zeros_like(r.samples)
    f = pb.reconstruct_nedner(r)
    assert not np.any(f.values)


def test_gpu_bit_identical_reruns():
    s = synth.make_3d(6, 48, 96, 20e-9, "clustered", 3, sigma=2e-3)
    r = s.as_record()
    a = pb.reconstruct_nedner(r).values
    b = pb.reconstruct_nedner(r).values
    assert np.array_equal(a, b)


def test_gpu_linearity():
    s1 = synth.make_3d(8, 32, 64, 20e-9, "jittered", 2)
    s2 = synth.make_3d(8, 32, 64, 20e-9, "jittered", 2)
    rng = np.random.default_rng(0)
    s2.samples = rng.standard_normal(s2.samples.shape)
    r1, r2 = s1.as_record(), s2.as_record()
    a, b = 0.7, -1.3
    r3 = s1.as_record()
    r3.samples = a * r1.samples + b * r2.samples
    f1 = pb.reconstruct_nedner(r1).values
    f2 = pb.reconstruct_nedner(r2).values
    f3 = pb.reconstruct_nedner(r3).values
    assert rel_l2(f3, a * f1 + b * f2) <= 1e-5


def test_gpu_full_grid_equals_equispaced_reduction():
    # on a complete grid with uniform weights NEDNER reduces to
    # the equispaced reconstruction; compare against the oracle on that grid.
    n, nt = 32, 64
    dx = synth.PITCH
    axes = [(np.arange(n) - n // 2) * dx] * 2
    mesh = np.meshgrid(*axes, indexing="ij")
    pos = np.stack([m.ravel() for m in mesh], axis=-1)
    balls = [(0.5e-3, -0.3e-3, 2.5e-3, 0.8e-3, 1.0)]
    samples = synth.ball_traces(pos, nt, 20e-9, synth.SOUND_SPEED, balls)
    w = np.full(n * n, dx * dx)
    r = pb.SensorRecord(pos, w, samples, 20e-9, synth.SOUND_SPEED, dx, (n, n))
    f = pb.reconstruct_nedner(r)
    want, _ = O.reconstruct_nedner(pos, w, samples, 20e-9, synth.SOUND_SPEED, dx, (n, n))
    assert rel_l2(f.values, want) <= TOL


def test_gpu_accepts_reference_style_record_object():
    class Rec:  # duck-typed stand-in for patfft.recon.SensorRecord
        pass

    s = synth.make_2d(seed=4, n=64, nt=128)
    r = Rec()
    for k in ("positions", "weights", "samples", "dt", "sound_speed", "dx", "n_lateral"):
        setattr(r, k, getattr(s, k))
    f = pb.reconstruct_nedner(r)
    want, _ = O.reconstruct_nedner(s.positions, s.weights, s.samples, s.dt, s.sound_speed, s.dx, s.n_lateral)
    assert rel_l2(f.values, want) <= TOL


def test_gpu_full_size_cfg3_matches_oracle():
    # BASELINE config 3 at full size (128^2 sensors x 512): the oracle takes ~10-20 s
    s = synth.CONFIGS["cfg3"]()
    f = pb.reconstruct_nedner(s.as_record())
    want, _ = O.reconstruct_nedner(s.positions, s.weights, s.samples, s.dt, s.sound_speed, s.dx, s.n_lateral)
    err = rel_l2(f.values, want)
    print(f"cfg3 full size: rel-L2 {err:.3e}")
    assert err <= TOL


def test_gpu_full_size_cfg4_properties():
    # BASELINE config 4 (256^2 clustered x 1024): size-independent properties --
    # linearity, bit-determinism and finite output (the oracle needs ~2 min here)
    s = synth.CONFIGS["cfg4"]()
    r1 = s.as_record()
    rng = np.random.default_rng(1)
    noise = rng.standard_normal(r1.samples.shape)
    r2 = s.as_record()
    r2.samples = noise
    r3 = s.as_record()
    r3.samples = 0.5 * r1.samples - 2.0 * noise
    f1 = pb.reconstruct_nedner(r1).values
    f1b = pb.reconstruct_nedner(r1).values
    f2 = pb.reconstruct_nedner(r2).values
    f3 = pb.reconstruct_nedner(r3).values
    assert f1.shape == (256, 256, 1024)
    assert np.array_equal(f1, f1b)
    assert np.all(np.isfinite(f1))
    assert rel_l2(f3, 0.5 * f1 - 2.0 * f2) <= 1e-5


@pytest.mark.parametrize("name", ["grid_3d_16x16x64", "grid_3d_8x16x32_up2", "grid_2d_64x128"])
def test_gpu_equispaced_and_interp_match_reference(name):
    from conftest import GOLDEN

    g = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    rec = pb.SensorRecord(g["positions"], g["weights"], g["samples"], float(g["dt"]), float(g["sound_speed"]),
                          float(g["dx"]), tuple(int(n) for n in g["n_lateral"]))
    up = int(g["upsample"])
    eq = pb.reconstruct_equispaced(rec, upsample=up)
    ip = pb.reconstruct_interp_fft(rec, upsample=up)
    e1, e2 = rel_l2(eq.values, g["values_equispaced"]), rel_l2(ip.values, g["values_interp"])
    print(f"{name}: equispaced rel-L2 {e1:.3e}, interp rel-L2 {e2:.3e}")
    assert eq.values.shape == g["values_equispaced"].shape
    np.testing.assert_allclose(eq.spacing, g["spacing"], rtol=1e-15)
    assert e1 <= TOL and e2 <= TOL


def test_gpu_equispaced_rejects_incomplete_grid():
    s = synth.make_3d(9, 16, 32, 20e-9, "jittered", 1)
    with pytest.raises(pb.ParameterError, match="complete sensor grid"):
        pb.reconstruct_equispaced(s.as_record())


def test_gpu_nerplan_matches_reference_golden():
    from conftest import GOLDEN

    g = np.load(os.path.join(GOLDEN, "ner_rows.npz"))
    plan = pb.NerPlan(g["u"].shape[-1])
    out = plan.execute(g["u"], g["kappas"])
    assert out.shape == g["out"].shape and out.dtype == np.complex128
    e1 = rel_l2(out, g["out"])
    e2 = rel_l2(plan.execute(g["u"], g["kappas_shared"]), g["out_shared"])
    e3 = rel_l2(out, g["direct"])
    print(f"NerPlan rows {e1:.2e} shared {e2:.2e} vs direct {e3:.2e}")
    assert e1 <= 1e-5 and e2 <= 1e-5 and e3 <= 1e-5


def test_gpu_nerplan_validation_and_larger_sizes():
    rng = np.random.default_rng(3)
    with pytest.raises(pb.ParameterError):
        pb.NerPlan(1)
    plan = pb.NerPlan(256)
    with pytest.raises(pb.ParameterError):
        plan.execute(np.zeros((2, 128)), np.zeros(3))
    with pytest.raises(pb.ParameterError):
        plan.execute(np.zeros((2, 256)), np.array([1e9]))
    with pytest.raises(pb.ParameterError):
        plan.execute(np.zeros((2, 256)), np.array([np.nan]))
    u = rng.standard_normal((3, 4, 256)) + 1j * rng.standard_normal((3, 4, 256))
    kap = rng.uniform(-256, 256, size=(3, 4, 50))
    got = pb.nufft_ner(u, kap)
    assert got.shape == (3, 4, 50)
    want = O.ner_direct(u, kap)
    assert rel_l2(got, want) <= 1e-5


def test_gpu_nedplan_matches_reference_golden():
    from conftest import GOLDEN

    g = np.load(os.path.join(GOLDEN, "ned_axes.npz"))
    out1 = pb.NedPlan((32,)).execute(g["pos1"], g["v1"])
    out2 = pb.NedPlan((16, 24)).execute(g["pos2"], g["v2"], order="wrapped")
    e1, e1d = rel_l2(out1, g["out1"]), rel_l2(out1, g["direct1"])
    e2 = rel_l2(out2, g["out2_wrapped"])
    print(f"NedPlan 1-axis {e1:.2e} (direct {e1d:.2e}), 2-axis wrapped {e2:.2e}")
    assert out1.shape == g["out1"].shape and out2.shape == g["out2_wrapped"].shape
    assert e1 <= 1e-5 and e1d <= 1e-5 and e2 <= 1e-5


def test_gpu_nedplan_centered_2d_vs_direct_and_validation():
    rng = np.random.default_rng(5)
    pos = np.stack([rng.uniform(-16, 16, 300), rng.uniform(-8, 8, 300)], axis=1)
    vals = rng.standard_normal((300, 3)) + 1j * rng.standard_normal((300, 3))
    got = pb.nufft_ned(pos, vals, (32, 16))
    want = O.ned_direct(pos, vals, (32, 16))
    assert got.shape == (32, 16, 3)
    assert rel_l2(got, want) <= 1e-5
    with pytest.raises(pb.ParameterError):
        pb.NedPlan((32, 16)).execute(pos * 3, vals)
    with pytest.raises(pb.ParameterError):
        pb.NedPlan((32, 15))
    with pytest.raises(pb.ParameterError):
        pb.NedPlan((32, 16)).execute(pos, vals, order="sideways")


FORWARD_GOLDENS = ["forward_3d_16x16x64", "forward_3d_rect8x16x32", "forward_2d_64x128"]


@pytest.mark.parametrize("name", FORWARD_GOLDENS)
def test_gpu_forward_fourier_matches_reference_golden(name):
    g = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    f = pb.ScalarField(g["field"], tuple(g["spacing"]))
    rec = pb.forward_fourier(f, float(g["sound_speed"]), pb.WindowSpec(c=float(g["spec_c"]), K=int(g["spec_K"])))
    assert rec.samples.shape == g["samples"].shape and rec.samples.dtype == np.float64
    np.testing.assert_array_equal(rec.positions, g["positions"])
    np.testing.assert_array_equal(rec.weights, g["weights"])
    assert rec.dt == float(g["dt"]) and rec.n_lateral == tuple(int(n) for n in g["n_lateral"])
    err = rel_l2(rec.samples, g["samples"])
    print(f"{name}: rel-L2 {err:.3e}")
    assert err <= TOL


def test_gpu_forward_fourier_larger_vs_oracle_and_validation():
    from oracle import forward_oracle as F

    rng = np.random.default_rng(5)
    vals = np.zeros((64, 64, 256))
    vals[20:30, 35:44, 60:75] = 1.0
    vals += 0.05 * rng.standard_normal(vals.shape)
    sp = (0.2e-3, 0.2e-3, 30e-6)
    rec = pb.forward_fourier(pb.ScalarField(vals, sp), 1500.0)
    want, _, _, _ = F.forward_fourier(vals, sp, 1500.0)
    err = rel_l2(rec.samples, want)
    print(f"forward 64x64x256: rel-L2 {err:.3e}")
    assert err <= TOL
    # linearity and zero field
    rec2 = pb.forward_fourier(pb.ScalarField(2.0 * vals, sp), 1500.0)
    assert rel_l2(rec2.samples, 2.0 * rec.samples) <= 1e-6
    assert not np.any(pb.forward_fourier(pb.ScalarField(np.zeros((8, 8, 16)), sp), 1500.0).samples)
    with pytest.raises(pb.ParameterError, match="sound speed"):
        pb.forward_fourier(pb.ScalarField(vals, sp), 0.0)
    with pytest.raises(pb.ParameterError, match="even"):
        pb.forward_fourier(pb.ScalarField(np.zeros((8, 9, 16)), sp), 1500.0)
    with pytest.raises(pb.ParameterError, match="2D and 3D"):
        pb.forward_fourier(pb.ScalarField(np.zeros((4, 4, 4, 4)), (1, 1, 1, 1)), 1500.0)


def test_gpu_frames_file_stream_matches_per_frame_reconstruction(tmp_path):
    # config-5 style frames (one sensor layout) streamed from a PATARR01 file
    s = synth.make_3d(31, 16, 32, 20e-9, "jittered", 2)
    rng = np.random.default_rng(31)
    frames = np.stack([s.samples * rng.uniform(0.5, 1.5) + 0.01 * rng.standard_normal(s.samples.shape)
                       for _ in range(3)])
    src, dst = tmp_path / "frames.patarr", tmp_path / "volumes.patarr"
    pb.write_array(src, frames, spacing=(1.0, 1.0, s.dt), axes=("frame", "sensor", "t"))
    plan = pb.NedNerPlan(s.positions, s.weights, 32, s.dt, s.sound_speed, s.dx, s.n_lateral)
    h = pb.reconstruct_frames_file(plan, src, dst)
    vols, hr = pb.read_array(dst)
    assert hr.dims == h.dims == (3,) + plan.out_shape
    assert hr.meta["frames"] == [0, 1, 2]
    for k in range(3):
        rec = pb.SensorRecord(s.positions, s.weights, frames[k], s.dt, s.sound_speed, s.dx, s.n_lateral)
        want = pb.reconstruct_nedner(rec).values
        np.testing.assert_array_equal(vols[k], want)   # same plan arithmetic, bit-identical
        oracle, _ = O.reconstruct_nedner(s.positions, s.weights, frames[k], s.dt, s.sound_speed, s.dx, s.n_lateral)
        assert rel_l2(vols[k], oracle) <= TOL
    with pytest.raises(pb.ParameterError):
        pb.reconstruct_frames_file(pb.NedNerPlan(s.positions, s.weights, 64, s.dt, s.sound_speed, s.dx,
                                                 s.n_lateral), src, dst)


def _plan_env(s, **env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return pb.NedNerPlan(s.positions, s.weights, s.samples.shape[1], s.dt, s.sound_speed, s.dx, s.n_lateral)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_gpu_host_staging_bit_identical_to_device_conversion(name):
    """Host-core f64->f32 narrowing + f32 PCIe (default) == device-side conversion (f64 over PCIe)."""
    s = synth.CONFIGS[name]()
    a, _, bad = _plan_env(s, PATFFT_HOST_CONVERT=1).execute_checked(s.samples)
    b, _ = _plan_env(s, PATFFT_HOST_CONVERT=0).execute(s.samples)
    assert bad == 0
    assert np.array_equal(a, b)
    # misaligned (8-byte) pageable caller buffers on both sides, several row blocks
    buf_in = np.empty(s.samples.size + 1)
    sin = buf_in[1:].reshape(s.samples.shape)
    sin[...] = s.samples
    p = _plan_env(s, PATFFT_HOST_BLOCKS=3)
    buf_out = np.empty(a.size + 1)
    out = buf_out[1:].reshape(a.shape)
    p.execute(sin, out)
    assert np.array_equal(out, a)


def test_gpu_nonfinite_samples_raise_like_scalarfield():
    s = synth.CONFIGS["cfg2"]()
    bad = s.samples.copy()
    bad[7, 11] = np.nan
    r = pb.SensorRecord(s.positions, s.weights, bad, s.dt, s.sound_speed, s.dx, s.n_lateral)
    with pytest.raises(pb.DataValidationError, match="finite"):
        pb.reconstruct_nedner(r)
    f = pb.reconstruct_nedner(s.as_record())  # the plan still works afterwards
    assert np.all(np.isfinite(f.values))


def test_gpu_recycled_outputs_never_alias_live_results():
    s = synth.CONFIGS["cfg2"]()
    r = s.as_record()
    f1 = pb.reconstruct_nedner(r)
    keep = f1.values.copy()
    view = f1.values[3]
    del f1  # a view still references the array: it must not be reused
    r2 = pb.SensorRecord(s.positions, s.weights, 2.0 * s.samples, s.dt, s.sound_speed, s.dx, s.n_lateral)
    f2 = pb.reconstruct_nedner(r2)
    f3 = pb.reconstruct_nedner(r2)
    assert np.array_equal(view, keep[3])
    assert f2.values is not f3.values
    assert np.array_equal(f2.values, f3.values)
    assert np.allclose(f2.values, 2.0 * keep, rtol=1e-5, atol=1e-6 * np.abs(keep).max())
    del f2, f3, view
    f4 = pb.reconstruct_nedner(r)  # everything dropped: a pooled buffer comes back, refilled
    assert np.array_equal(f4.values, keep)


def _pinned(shape):
    import ctypes

    from paper_1501_02946_b200 import _lib
    lib = _lib.load()
    p = ctypes.c_void_p()
    n = int(np.prod(shape))
    _lib.check(lib.patfft_host_alloc(8 * n, ctypes.byref(p)))
    a = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), shape=(n,)).reshape(shape)
    return a, p


@pytest.mark.parametrize("frac", ["0.35", "1.0"])  # PATFFT_HOST_DIRECT sets both directions
def test_gpu_pinned_direct_split_bit_identical(frac):
    """Pinned caller buffers: part of the rows/voxels move as float64 by DMA (device conversion)."""
    from paper_1501_02946_b200 import _lib
    lib = _lib.load()
    s = synth.CONFIGS["cfg3"]()
    want, _ = _plan_env(s, PATFFT_HOST_DIRECT=0).execute(s.samples)
    p = _plan_env(s, PATFFT_HOST_DIRECT=frac)
    hin, pin = _pinned(s.samples.shape)
    hout, pout = _pinned(want.shape)
    try:
        hin[...] = s.samples
        _, _, bad = p.execute_checked(hin, hout)
        assert bad == 0
        assert np.array_equal(hout, want)
        hin[5, 9] = np.inf  # non-finite output must be counted in the direct and the staged part
        _, _, bad = p.execute_checked(hin, hout)
        assert bad > 0 and bad == int(np.count_nonzero(~np.isfinite(hout)))
    finally:
        lib.patfft_host_free(pin)
        lib.patfft_host_free(pout)


@pytest.mark.parametrize("scale", [1e-30, 1e-12, 1e12, 1e30])
def test_gpu_gridding_scale_invariance(scale):
    """The fp16 two-term gridding rescales samples by a power of two from their
    maximum: any overall amplitude gives the same relative answer."""
    s = synth.CONFIGS["cfg2"]()
    p = _plan_env(s, PATFFT_SPREAD_F16_MIN_ITEMS=0)  # the fp16 kernel even at this small size
    base, _ = p.execute(s.samples)
    got, _ = p.execute(s.samples * scale)
    err = rel_l2(got / scale, base)
    print(f"scale {scale:g}: rel-L2 vs unscaled {err:.3e}")
    assert err <= 3e-6  # fp32 rounding of the rescaled input (5e-7 measured); a broken scale shows as O(1)


@pytest.mark.parametrize("f16", [0, 1])
def test_gpu_gridding_forms_match_oracle(f16):
    """Both tensor-core gridding forms (3xTF32, fp16 two-term) forced on cfg3 vs the oracle."""
    s = synth.CONFIGS["cfg3"]()
    got, _ = _plan_env(s, PATFFT_SPREAD_F16=f16, PATFFT_SPREAD_F16_MIN_ITEMS=0).execute(s.samples)
    want, _ = O.reconstruct_nedner(s.positions, s.weights, s.samples, s.dt, s.sound_speed, s.dx, s.n_lateral)
    err = rel_l2(got, want)
    print(f"cfg3 gridding form f16={f16}: rel-L2 {err:.3e}")
    assert err <= TOL


def test_gpu_gridding_mixed_amplitudes_vs_oracle():
    """One loud sensor row next to quiet ones: still within the parity bar."""
    s = synth.CONFIGS["cfg2"]()
    smp = s.samples.copy()
    smp[17] *= 1e4
    smp[1000] *= 1e-4
    got, _ = _plan_env(s, PATFFT_SPREAD_F16_MIN_ITEMS=0).execute(smp)
    want, _ = O.reconstruct_nedner(s.positions, s.weights, smp, s.dt, s.sound_speed, s.dx, s.n_lateral)
    err = rel_l2(got, want)
    print(f"mixed amplitudes: rel-L2 {err:.3e}")
    assert err <= TOL


@pytest.mark.parametrize("nt", [96, 320, 384])
def test_gpu_fp16_gridding_short_time_blocks_vs_oracle(nt):
    """fp16 tensor-core gridding with N = 32 / 64 / 128 time samples per work item."""
    s = synth.make_3d(11, 32, nt, 20e-9, "jittered", 2)
    got, _ = _plan_env(s, PATFFT_SPREAD_F16_MIN_ITEMS=0).execute(s.samples)
    want, _ = O.reconstruct_nedner(s.positions, s.weights, s.samples, s.dt, s.sound_speed, s.dx, s.n_lateral)
    err = rel_l2(got, want)
    print(f"fp16 gridding T={nt}: rel-L2 {err:.3e}")
    assert err <= TOL
