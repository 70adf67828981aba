"""GPU parity at the headline configuration and on every compiled kernel variant.

* cfg4 (256^2 clustered sensors x Nt = 1024, north_star's named config)
  against a summary of the REFERENCE's own output
  (``tests/golden/large_cfg4.npz``, made by ``tests/golden/make_golden_large.py``
  from ``/root/reference/pkg/src/patfft/recon.py:358-379``): 16 full depth
  planes, a full lateral slice, every depth plane's L2 norm and the
  energy projection over depth.
* cfg5 (64 frames of 128^2 x 512 sharing one layout) through the batched
  device entry point against the reference's per-frame summaries
  (``tests/golden/large_cfg5.npz``).
* Small cases against the oracle (pinned to the reference in
  tests/test_oracle.py) chosen so that each compile-time instantiation on the
  headline path runs at least once: the fused NER kernel for T = 128 ... 2048
  (``ner_dct_kernel<8, 7, 7..11>`` with the float32-grade
  8-tap window, ``<12, 7, ..>`` with PATFFT_FP32_WINDOW=0), the lateral FFT kernels for oversampled
  lengths 64 ... 2048 (``colfft``/``rowfft`` ``<4, 6..9>``, ``<3, 10>``,
  ``<2, 11>``) and the inverse kernels at 256 / 512 / 1024.
"""

import hashlib
import os

import numpy as np
import pytest

import paper_1501_02946_b200 as pb
from conftest import GOLDEN, rel_l2
from oracle import nedner_oracle as O
from paper_1501_02946_b200 import synth

pytestmark = pytest.mark.gpu
TOL = 1e-4  # BASELINE.json north_star: rel-L2 <= 1e-4 on the reconstructed volume


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _env_plan(s, **env):
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


@pytest.mark.parametrize("fp32_window", [1, 0], ids=["taps8", "taps12"])
def test_gpu_cfg4_matches_reference_golden(fp32_window):
    """The headline config through the drop-in call (fp32-grade 8-tap windows,
    the default) and with the reference's own 12 taps (PATFFT_FP32_WINDOW=0)."""
    g = np.load(os.path.join(GOLDEN, "large_cfg4.npz"))
    s = synth.CONFIGS["cfg4"]()
    assert _sha(s.samples) == str(g["samples_sha256"]), "synthetic cfg4 record differs from the golden's"
    if fp32_window:
        f = pb.reconstruct_nedner(s.as_record())
    else:
        plan = _env_plan(s, PATFFT_FP32_WINDOW=0)
        wi = plan.window_info()
        assert wi["lateral_taps"] == 12 and wi["ner_taps"] == 12, wi
        img, _ = plan.execute(s.samples)
        f = pb.ScalarField(img, tuple(g["spacing"]))
    v = f.values
    assert v.shape == (256, 256, 1024)
    np.testing.assert_allclose(f.spacing, g["spacing"], rtol=1e-15)
    z = g["planes_z"]
    errs = {
        "planes": rel_l2(v[:, :, z], g["planes"]),
        "row_slice": rel_l2(v[int(g["row"])], g["row_slice"]),
        "plane_norms": rel_l2(np.linalg.norm(v.reshape(-1, v.shape[2]), axis=0), g["plane_norms"]),
        "depth_energy": rel_l2((v * v).sum(axis=2), g["depth_energy"]),
        "total_norm": abs(np.linalg.norm(v) / float(g["total_norm"]) - 1.0),
    }
    print(f"cfg4 vs reference ({'8' if fp32_window else '12'} taps): "
          + ", ".join(f"{k} rel-L2 {e:.3e}" for k, e in errs.items()) + f" (reference took {float(g['reference_seconds']):.0f} s on CPU)")
    assert max(errs.values()) <= TOL


def test_gpu_cfg5_64_frames_match_reference_golden():
    torch = pytest.importorskip("torch")
    g = np.load(os.path.join(GOLDEN, "large_cfg5.npz"))
    frames = list(synth.make_frames())
    assert len(frames) == 64
    for k, fr in enumerate(frames):
        assert _sha(fr.samples) == str(g["samples_sha256"][k]), f"frame {k} input differs from the golden's"
    s0 = frames[0]
    plan = pb.NedNerPlan(s0.positions, s0.weights, 512, s0.dt, s0.sound_speed, s0.dx, s0.n_lateral)
    dev = torch.device("cuda", 0)
    x = torch.from_numpy(np.stack([f.samples for f in frames]).astype(np.float32)).to(dev)
    y = torch.empty((64,) + plan.out_shape, dtype=torch.float32, device=dev)
    plan.execute_frames_device(64, x.data_ptr(), y.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
    torch.cuda.synchronize(dev)
    v = y.cpu().numpy().astype(np.float64)
    norms = np.linalg.norm(v.reshape(64, -1, v.shape[-1]), axis=1)
    worst = max(rel_l2(norms[k], g["plane_norms"][k]) for k in range(64))
    tot = np.abs(np.linalg.norm(v.reshape(64, -1), axis=1) / g["total_norms"] - 1).max()
    pe = [rel_l2(v[k][:, :, g["planes_z"]], g["planes"][i]) for i, k in enumerate(g["full_frames"])]
    print(f"cfg5 64 frames vs reference: worst per-frame plane-norm rel-L2 {worst:.3e}, total-norm {tot:.3e}, "
          f"planes of frames {list(g['full_frames'])}: " + ", ".join(f"{e:.3e}" for e in pe))
    assert worst <= TOL and tot <= TOL and max(pe) <= TOL


def _rect_record(seed, nl, nt, dt=20e-9, layout="uniform"):
    rng = np.random.default_rng(seed)
    m = int(np.prod(nl))
    half = np.asarray(nl, float) * synth.PITCH / 2
    if layout == "uniform":
        pos = rng.uniform(-half, half, size=(m, len(nl)))
    else:
        axes = [((np.arange(n) + 0.5) - n / 2.0) * synth.PITCH for n in nl]
        mesh = np.meshgrid(*axes, indexing="ij")
        pos = np.stack([mm.ravel() for mm in mesh], axis=-1)
        pos = pos + rng.uniform(-0.4 * synth.PITCH, 0.4 * synth.PITCH, size=pos.shape)
    depth = nt * synth.SOUND_SPEED * dt
    balls = []
    for _ in range(3):
        rad = rng.uniform(0.3e-3, 0.8e-3)
        lat = rng.uniform(-0.6, 0.6, size=2) * half
        balls.append((lat[0], lat[-1] if len(nl) == 2 else 0.0, rng.uniform(rad + 0.3e-3, 0.8 * depth), rad,
                      rng.uniform(0.5, 1.0)))
    samples = synth.ball_traces(pos, nt, dt, synth.SOUND_SPEED, balls)
    if not np.any(samples):  # keep the case meaningful: never zero -> zero
        samples += 1e-3 * rng.standard_normal(samples.shape)
    w = np.full(m, float(np.prod(np.asarray(nl) * synth.PITCH)) / m)
    return synth.SyntheticRecord(pos, w, samples, dt, synth.SOUND_SPEED, synth.PITCH, tuple(nl))


# (id, lateral sensors, Nt, dt, upsample, what it reaches)
VARIANTS = [
    ("T128_16x16", (16, 16), 128, 20e-9, 1, "ner_dct<8,7,7>"),
    ("T256_16x16", (16, 16), 256, 20e-9, 1, "ner_dct<8,7,8>"),
    ("T1024_32x32", (32, 32), 1024, 10e-9, 1, "ner_dct<8,7,10>, colfft/rowfft<4,6>"),
    ("T2048_32x32", (32, 32), 2048, 5e-9, 1, "ner_dct<8,7,11>"),
    ("lat256x16_T128", (256, 16), 128, 20e-9, 1, "rowfft<4,9>, inv_col<4,8>"),
    ("lat16x256_T128", (16, 256), 128, 20e-9, 1, "colfft<4,9>, inv_c2r<4,8>"),
    ("lat128x64_up2_T128", (128, 64), 128, 20e-9, 2, "inv_col<4,8>, inv_c2r<4,7>, upsampled NER"),
    ("lat512x8_T64", (512, 8), 64, 20e-9, 1, "rowfft<3,10>, inv_col<4,9>"),
    ("lat8x1024_T64", (8, 1024), 64, 20e-9, 1, "colfft<2,11>, inv_c2r<3,10>"),
    ("lat256x256_T128", (256, 256), 128, 20e-9, 1, "cfg4's lateral kernels colfft/rowfft<4,9>, inv<4,8>"),
]


@pytest.mark.parametrize("case", VARIANTS, ids=[v[0] for v in VARIANTS])
def test_gpu_kernel_variant_matches_oracle(case):
    name, nl, nt, dt, up, what = case
    s = _rect_record(sum(map(ord, name)), nl, nt, dt)
    f = pb.reconstruct_nedner(s.as_record(), upsample=up)
    want, _ = O.reconstruct_nedner(s.positions, s.weights, s.samples, s.dt, s.sound_speed, s.dx, s.n_lateral,
                                   upsample=up)
    assert f.values.shape == want.shape
    err = rel_l2(f.values, want)
    print(f"variant {name} ({what}): rel-L2 {err:.3e}")
    assert err <= TOL


@pytest.mark.parametrize("f16", [0, 1])
def test_gpu_cfg4_geometry_short_depth_both_gridding_forms(f16):
    """cfg4's 256^2 clustered layout (the headline gridding tiles and their
    sensor density) at Nt = 128, both tensor-core gridding forms, vs the oracle."""
    s = synth.make_3d(4, 256, 128, 80e-9, "clustered", 20, sigma=8e-3)
    old = {k: os.environ.get(k) for k in ("PATFFT_SPREAD_F16", "PATFFT_SPREAD_F16_MIN_ITEMS")}
    os.environ["PATFFT_SPREAD_F16"] = str(f16)
    os.environ["PATFFT_SPREAD_F16_MIN_ITEMS"] = "0"
    try:
        plan = pb.NedNerPlan(s.positions, s.weights, 128, s.dt, s.sound_speed, s.dx, s.n_lateral)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    got, _ = plan.execute(s.samples)
    want, _ = O.reconstruct_nedner(s.positions, s.weights, s.samples, s.dt, s.sound_speed, s.dx, s.n_lateral)
    err = rel_l2(got, want)
    print(f"cfg4 layout at Nt=128, gridding f16={f16}: rel-L2 {err:.3e}")
    assert err <= TOL


@pytest.mark.parametrize("nl,nt,slots", [((64, 64), 128, 3), ((128, 128), 128, 2), ((256, 256), 256, 3)])
def test_gpu_single_launch_lateral_matches_two_kernel_form(nl, nt, slots):
    """PATFFT_LAT_FUSED_SLOTS > 0: column and row FFTs in one launch with Y as an
    L2-resident ring (lateral.cu, latfused_kernel).  Same arithmetic per tile, so the
    volume is bit-identical to the default two-kernel form; also checked vs the oracle."""
    s = _rect_record(11 + nl[0], nl, nt, 20e-9, layout="jittered")
    base = pb.NedNerPlan(s.positions, s.weights, nt, s.dt, s.sound_speed, s.dx, s.n_lateral)
    ref, _ = base.execute(s.samples)
    ref = ref.copy()
    os.environ["PATFFT_LAT_FUSED_SLOTS"] = str(slots)
    try:
        plan = pb.NedNerPlan(s.positions, s.weights, nt, s.dt, s.sound_speed, s.dx, s.n_lateral)
        got, _ = plan.execute(s.samples)
        got2, _ = plan.execute(s.samples)  # flags are re-zeroed per launch
    finally:
        os.environ.pop("PATFFT_LAT_FUSED_SLOTS", None)
    assert np.array_equal(got, ref) and np.array_equal(got2, ref)
    want, _ = O.reconstruct_nedner(s.positions, s.weights, s.samples, s.dt, s.sound_speed, s.dx, s.n_lateral)
    err = rel_l2(got, want)
    print(f"single-launch lateral {nl} Nt={nt} slots={slots}: bit-identical to the two-kernel form, rel-L2 {err:.3e}")
    assert err <= TOL


@pytest.mark.parametrize("nl,nt,slots,lead", [((32, 32), 64, 2, 1), ((64, 64), 128, 6, 3), ((128, 128), 256, 4, 2)])
def test_gpu_single_launch_inverse_matches_two_kernel_form(nl, nt, slots, lead):
    """PATFFT_INV_FUSED_SLOTS > 0: the lateral inverse in one launch, the column-inverse output in an
    L2-resident ring that the C2R tiles of the same launch read (lateral.cu, invfused_kernel).  Same
    arithmetic per tile: bit-identical to the default two-kernel form."""
    s = _rect_record(23 + nl[0], nl, nt, 20e-9, layout="jittered")
    base = pb.NedNerPlan(s.positions, s.weights, nt, s.dt, s.sound_speed, s.dx, s.n_lateral)
    ref = base.execute(s.samples)[0].copy()
    os.environ["PATFFT_INV_FUSED_SLOTS"] = str(slots)
    os.environ["PATFFT_INV_FUSED_LEAD"] = str(lead)
    try:
        plan = pb.NedNerPlan(s.positions, s.weights, nt, s.dt, s.sound_speed, s.dx, s.n_lateral)
        got = plan.execute(s.samples)[0].copy()
        got2 = plan.execute(s.samples)[0]
    finally:
        os.environ.pop("PATFFT_INV_FUSED_SLOTS", None)
        os.environ.pop("PATFFT_INV_FUSED_LEAD", None)
    assert np.array_equal(got, ref) and np.array_equal(got2, ref)
    print(f"single-launch inverse {nl} Nt={nt} slots={slots} lead={lead}: bit-identical to the two-kernel form")


@pytest.mark.parametrize("nl,nt", [((8, 8), 8192), ((16,), 16384), ((8, 8), 6000)])
def test_gpu_records_longer_than_the_shared_memory_ner(nl, nt):
    """N_t > 4096 (oversampled depth length > 16384): beyond the shared-memory NER kernels, so the
    plan runs the cuFFT-based reference-length form (csrc/reflen.cu); the reference has no bound."""
    rng = np.random.default_rng(nt)
    m = int(np.prod(nl))
    half = np.asarray(nl, float) * synth.PITCH / 2
    pos = rng.uniform(-half, half, size=(m, len(nl)))
    t = np.arange(nt)
    samples = np.exp(-((t[None, :] - rng.uniform(200, nt * 0.8, size=(m, 1))) ** 2) / 50.0)
    samples += 1e-3 * rng.standard_normal((m, nt))
    w = np.full(m, float(np.prod(np.asarray(nl) * synth.PITCH)) / m)
    want, _ = O.reconstruct_nedner(pos, w, samples, 5e-9, synth.SOUND_SPEED, synth.PITCH, nl)
    got = pb.reconstruct_nedner(pb.SensorRecord(pos, w, samples, 5e-9, synth.SOUND_SPEED, synth.PITCH, nl))
    err = rel_l2(got.values, want)
    print(f"long record {nl} Nt={nt}: rel-L2 {err:.3e}")
    assert got.values.shape == want.shape and err <= TOL


def test_gpu_gridding_scale_hint_history_does_not_change_results():
    """fp16 gridding: the sample scale is speculated from the previous call's maximum and verified
    on the device (spread_tc.cu, check_scale_kernel); a wrong guess re-runs the gridding.  Whatever
    the history of a plan -- first call, data 1e6 louder, 1e-9 quieter, zeros, back again -- each
    volume is bit-identical to the one a fresh plan returns (whose first call always re-runs)."""
    s = synth.make_3d(4, 256, 128, 80e-9, "clustered", 20, sigma=8e-3)  # cfg4's layout: fp16 form
    def mk():
        os.environ["PATFFT_SPREAD_F16_MIN_ITEMS"] = "0"  # the fp16 form even for this short record
        try:
            return pb.NedNerPlan(s.positions, s.weights, 128, s.dt, s.sound_speed, s.dx, s.n_lateral)
        finally:
            os.environ.pop("PATFFT_SPREAD_F16_MIN_ITEMS", None)

    plan = mk()
    assert plan.window_info()["lateral_taps"] == 8
    scales = [1.0, 1.0, 1e6, 3e6, 1e-9, 0.0, 1.0, 1.9, 2.1]
    outs = [plan.execute(s.samples * a)[0].copy() for a in scales]
    for a, got in zip(scales, outs):
        fresh = mk().execute(s.samples * a)[0]
        assert np.array_equal(got, fresh), f"scale {a}: result depends on the plan's history"
    want, _ = O.reconstruct_nedner(s.positions, s.weights, s.samples, s.dt, s.sound_speed, s.dx, s.n_lateral)
    err = rel_l2(outs[0], want)
    print(f"scale-hint history: 9 calls bit-identical to fresh plans, rel-L2 vs oracle {err:.3e}")
    assert err <= TOL and not np.any(outs[5])


def test_gpu_window_selection():
    """Auto (alpha, beta) windows with K > 4 run with the float32-grade 8 taps;
    explicit windows and K <= 4 keep what was asked (nufft.py:133-149)."""
    s = synth.make_3d(3, 16, 64, 20e-9, "jittered", 1)

    def taps(spec):
        p = pb.NedNerPlan(s.positions, s.weights, 64, s.dt, s.sound_speed, s.dx, s.n_lateral, spec=spec)
        w = p.window_info()
        return w["lateral_taps"], w["ner_taps"]

    assert taps(None) == (8, 8)
    assert taps(pb.WindowSpec(K=5)) == (8, 8)
    assert taps(pb.WindowSpec(K=3)) == (6, 6)
    assert taps(pb.WindowSpec(K=6, alpha=9.41535318280861)) == (12, 12)


def _pinned_f64(shape):
    import ctypes

    from paper_1501_02946_b200 import _lib
    lib = _lib.load()
    p = ctypes.c_void_p()
    n = int(np.prod(shape))
    _lib.check(lib.patfft_host_alloc(8 * n, ctypes.byref(p)))
    a = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), shape=(n,)).reshape(shape)
    return a, p


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_gpu_batch_pipeline_bit_identical_to_single_calls(name):
    """patfft_nedner_execute_batch (record k+1 up / k-1 down while k computes)
    gives every record exactly the single-call result, with pageable and pinned
    caller buffers (the pinned ones move a share as float64 by DMA), and counts
    non-finite voxels per record."""
    from paper_1501_02946_b200 import _lib

    lib = _lib.load()
    s = synth.CONFIGS[name]()
    plan = pb.NedNerPlan(s.positions, s.weights, s.samples.shape[1], s.dt, s.sound_speed, s.dx, s.n_lateral)
    rng = np.random.default_rng(9)
    recs = [s.samples * rng.uniform(0.5, 2.0) for _ in range(5)]
    recs[3] = recs[3].copy()
    recs[3][11, 7] = np.nan
    want = [plan.execute_checked(r) for r in recs]
    vols, bad = plan.execute_batch(recs)
    for k in range(5):
        assert bad[k] == want[k][2]
        assert np.array_equal(vols[k], want[k][0], equal_nan=True)
    assert bad[3] > 0 and all(bad[k] == 0 for k in (0, 1, 2, 4))
    pins = [_pinned_f64(s.samples.shape) for _ in range(3)] + [_pinned_f64(plan.out_shape) for _ in range(3)]
    try:
        for k in range(3):
            pins[k][0][...] = recs[k]
        outs = [pins[3 + k][0] for k in range(3)]
        vols, bad = plan.execute_batch([pins[k][0] for k in range(3)], outs)
        for k in range(3):
            assert bad[k] == 0
            assert np.array_equal(outs[k], want[k][0])
    finally:
        for _, p in pins:
            lib.patfft_host_free(p)
