"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``patfft`` from /root/reference/pkg/src (read-only), builds small
seeded inputs, calls the reference's own public API
(``patfft.recon.reconstruct_nedner``, ``NerPlan``, ``NedPlan``,
``kappa``/``amplitude_factor``) and stores inputs + outputs as compressed
.npz fixtures next to this script.  The fixtures travel with the repo; the
GPU box never needs /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("PATFFT_REFERENCE", "/root/reference/pkg/src")
sys.dont_write_bytecode = True
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from patfft import forward as rforward  # noqa: E402  (reference)
from patfft import nufft as rnufft  # noqa: E402  (reference)
from patfft import recon as rrecon  # noqa: E402  (reference)

from paper_1501_02946_b200 import synth  # noqa: E402  (seeded inputs only)


def _record(pos, w, samples, dt, c, dx, nl):
    return rrecon.SensorRecord(positions=pos, weights=w, samples=samples, dt=dt,
                               sound_speed=c, dx=dx, n_lateral=nl)


ONLY = set(sys.argv[1:])  # optional fixture names: regenerate just those


def _save(name, **arrays):
    if ONLY and name not in ONLY:
        return
    if "samples" in arrays:  # a fixture whose data never reaches a sensor tests only zero -> zero
        assert np.abs(arrays["samples"]).max() > 0, f"{name}: all-zero samples"
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def recon_case(name, rec: synth.SyntheticRecord, out_dims=None, upsample=1, spec=None):
    r = _record(rec.positions, rec.weights, rec.samples, rec.dt, rec.sound_speed, rec.dx, rec.n_lateral)
    wspec = None if spec is None else rnufft.WindowSpec(**spec)
    f = rrecon.reconstruct_nedner(r, out_dims=out_dims, upsample=upsample, spec=wspec)
    spec = spec or {}
    _save(name,
          positions=rec.positions, weights=rec.weights, samples=rec.samples,
          dt=rec.dt, sound_speed=rec.sound_speed, dx=rec.dx, n_lateral=np.asarray(rec.n_lateral),
          out_dims=np.asarray(out_dims if out_dims is not None else rec.n_lateral),
          upsample=upsample,
          spec_c=spec.get("c", 2.0), spec_K=spec.get("K", 6),
          spec_alpha=np.nan if spec.get("alpha") is None else spec["alpha"],
          spec_beta=np.nan if spec.get("beta") is None else spec["beta"],
          values=f.values, spacing=np.asarray(f.spacing), imag_residual=f.meta["imag_residual"])


def main():
    # 1. config-1 geometry (2D) at full size: 128 sensors x Nt=512
    recon_case("recon_2d_cfg1", synth.make_2d(seed=11))
    # 2. small 3D jittered grid
    recon_case("recon_3d_jitter32", synth.make_3d(12, 32, 64, 20e-9, "jittered", 3))
    # 3. uniform-random 3D with out_dims != n_lateral and upsample 2
    recon_case("recon_3d_uniform16_up2", synth.make_3d(13, 16, 32, 20e-9, "uniform", 2),
               out_dims=(12, 16), upsample=2)
    # 4. clustered (positions clipped onto the aperture edge -> wrap-around bins)
    recon_case("recon_3d_cluster24", synth.make_3d(14, 24, 48, 20e-9, "clustered", 3, sigma=1.5e-3))
    # 5. non-default window spec
    recon_case("recon_3d_specK4", synth.make_3d(15, 16, 32, 20e-9, "uniform", 2), spec={"c": 2.0, "K": 4})
    # 6. 2D upsample 2, non-power-of-two depth (Nt = 96)
    recon_case("recon_2d_up2_nt96", synth.make_2d(seed=16, n=32, nt=96), upsample=2)
    # 7. rectangular lateral grid (16 x 24 sensors)
    rng = np.random.default_rng(17)
    nl = (16, 24)
    pos = np.stack([rng.uniform(-8, 8, 384), rng.uniform(-12, 12, 384)], axis=1) * synth.PITCH
    balls = [(0.3e-3, -0.5e-3, 2.0e-3, 0.7e-3, 1.0)]
    samples = synth.ball_traces(pos, 64, 20e-9, synth.SOUND_SPEED, balls)
    w = np.full(384, (16 * synth.PITCH) * (24 * synth.PITCH) / 384)
    recon_case("recon_3d_rect16x24",
               synth.SyntheticRecord(pos, w, samples, 20e-9, synth.SOUND_SPEED, synth.PITCH, nl))

    # 8. wide window (K = 8 -> 16 taps, the 32-slot spread ring) and narrow K = 2
    recon_case("recon_3d_specK8", synth.make_3d(18, 16, 32, 20e-9, "jittered", 2), spec={"c": 2.0, "K": 8})
    recon_case("recon_2d_specK2", synth.make_2d(seed=19, n=32, nt=128), spec={"c": 2.0, "K": 2})
    # 9. explicit window shape and a larger oversampling factor (c = 2.5)
    recon_case("recon_3d_spec_c25", synth.make_3d(20, 16, 32, 20e-9, "uniform", 2),
               spec={"c": 2.5, "K": 6, "alpha": 12.0, "beta": 2.3})
    # 9b. admissible but inaccurate explicit windows: the reference's answer carries their
    # truncation error (1e-3 .. 1e-2 away from the exact transform), which only a plan on the
    # reference's own oversampled lengths reproduces (csrc/reflen.cu)
    recon_case("recon_3d_badwin_c25", synth.make_3d(20, 16, 32, 20e-9, "uniform", 2),
               spec={"c": 2.5, "K": 6, "alpha": 12.0, "beta": 0.5})
    recon_case("recon_2d_badwin_up2", synth.make_2d(seed=23, n=32, nt=96), upsample=2,
               spec={"c": 2.2, "K": 3, "alpha": 9.0, "beta": 0.8})
    recon_case("recon_3d_badwin_up2", synth.make_3d(24, 12, 24, 40e-9, "jittered", 2), upsample=2,
               spec={"c": 2.5, "K": 4, "alpha": 11.0, "beta": 0.7})
    # 10. upsample 3 (non-power-of-two depth and lateral inverse sizes)
    # (dt = 100 ns: the 16 samples reach the ball; at 20 ns every trace was zero)
    recon_case("recon_3d_up3", synth.make_3d(21, 8, 16, 100e-9, "jittered", 1), upsample=3)
    # 11. every sensor exactly on the aperture corner / edges (wrap-around taps on both axes)
    rng = np.random.default_rng(22)
    n = 16
    half = n * synth.PITCH / 2
    edge = np.concatenate([rng.uniform(-half, half, size=(200, 2)),
                           np.array([[-half, -half], [half, half], [-half, half], [half, -half],
                                     [0.0, half], [half, 0.0], [-half, 0.0], [0.0, -half]])])
    balls = [(0.2e-3, 0.1e-3, 2.0e-3, 0.6e-3, 1.0)]
    # (dt = 60 ns: the 32 samples reach the ball; at 20 ns every trace was zero)
    samples = synth.ball_traces(edge, 32, 60e-9, synth.SOUND_SPEED, balls)
    w = np.full(edge.shape[0], (n * synth.PITCH) ** 2 / edge.shape[0])
    recon_case("recon_3d_edges16", synth.SyntheticRecord(edge, w, samples, 60e-9, synth.SOUND_SPEED, synth.PITCH,
                                                         (n, n)))

    # 12. complete grids: reconstruct_equispaced and reconstruct_interp_fft
    def grid_case(name, n_lateral, nt, seed, upsample=1, shuffle=True):
        rng = np.random.default_rng(seed)
        axes = [(np.arange(n) - n // 2) * synth.PITCH for n in n_lateral]
        mesh = np.meshgrid(*axes, indexing="ij")
        pos = np.stack([m.ravel() for m in mesh], axis=-1)
        if shuffle:
            pos = pos[rng.permutation(pos.shape[0])]
        if len(n_lateral) == 2:
            balls = [(0.3e-3, -0.2e-3, 1.6e-3, 0.5e-3, 1.0), (-0.4e-3, 0.3e-3, 1.0e-3, 0.3e-3, 0.7)]
            samples = synth.ball_traces(pos, nt, 20e-9, synth.SOUND_SPEED, balls)
        else:
            t = np.arange(nt) * 20e-9
            dist = np.hypot(pos[:, 0] - 0.4e-3, 1.5e-3)
            samples = np.exp(-((t[None, :] - dist[:, None] / synth.SOUND_SPEED) ** 2) / (2 * (40e-9) ** 2))
        w = np.full(pos.shape[0], float(np.prod([n * synth.PITCH for n in n_lateral])) / pos.shape[0])
        r = _record(pos, w, samples, 20e-9, synth.SOUND_SPEED, synth.PITCH, n_lateral)
        eq = rrecon.reconstruct_equispaced(r, upsample=upsample)
        ip = rrecon.reconstruct_interp_fft(r, upsample=upsample)
        _save(name, positions=pos, weights=w, samples=samples, dt=20e-9, sound_speed=synth.SOUND_SPEED,
              dx=synth.PITCH, n_lateral=np.asarray(n_lateral), upsample=upsample,
              values_equispaced=eq.values, values_interp=ip.values, spacing=np.asarray(eq.spacing))

    grid_case("grid_3d_16x16x64", (16, 16), 64, 23)
    grid_case("grid_3d_8x16x32_up2", (8, 16), 32, 24, upsample=2)
    grid_case("grid_2d_64x128", (64,), 128, 25)

    # component goldens: NER (per-row targets) and NED (1 and 2 axes)
    rng = np.random.default_rng(21)
    n = 64
    u = rng.standard_normal((5, n)) + 1j * rng.standard_normal((5, n))
    kap = rng.uniform(-n, n, size=(5, 40))
    ner = rnufft.NerPlan(n).execute(u, kap)
    ner_direct = rnufft.nudft_ner_direct(u, kap)
    kap_shared = rng.uniform(-n, n, size=33)
    ner_shared = rnufft.NerPlan(n).execute(u, kap_shared)
    _save("ner_rows", u=u, kappas=kap, out=ner, direct=ner_direct, kappas_shared=kap_shared, out_shared=ner_shared)

    pos1 = rng.uniform(-16, 16, size=93)
    v1 = rng.standard_normal(93) + 1j * rng.standard_normal(93)
    ned1 = rnufft.NedPlan((32,)).execute(pos1, v1)
    pos2 = np.stack([rng.uniform(-8, 8, 200), rng.uniform(-12, 12, 200)], axis=1)
    v2 = rng.standard_normal((200, 3)) + 1j * rng.standard_normal((200, 3))
    ned2 = rnufft.NedPlan((16, 24)).execute(pos2, v2, order="wrapped")
    _save("ned_axes", pos1=pos1, v1=v1, out1=ned1, direct1=rnufft.nudft_ned_direct(pos1, v1, (32,)),
          pos2=pos2, v2=v2, out2_wrapped=ned2)

    # forward model (forward.py:105-166) on phantoms rasterised by the reference
    def forward_case(name, dims, spacing, balls, spec=None, sound_speed=synth.SOUND_SPEED):
        ph = rforward.PhantomSpec(dims=dims, spacing=spacing, balls=[rforward.Ball(*b) for b in balls])
        f = ph.rasterize()
        wspec = None if spec is None else rnufft.WindowSpec(**spec)
        rec = rforward.forward_fourier(f, sound_speed, wspec)
        spec = spec or {}
        _save(name, field=f.values, spacing=np.asarray(f.spacing), sound_speed=sound_speed,
              spec_c=spec.get("c", 2.0), spec_K=spec.get("K", 6),
              samples=rec.samples, positions=rec.positions, weights=rec.weights, dt=rec.dt, dx=rec.dx,
              n_lateral=np.asarray(rec.n_lateral))

    p = synth.PITCH
    forward_case("forward_3d_16x16x64", (16, 16, 64), (p, p, 30e-6),
                 [((0.3e-3, -0.2e-3, 0.9e-3), 0.35e-3, 1.0), ((-0.5e-3, 0.4e-3, 1.3e-3), 0.25e-3, 0.6)])
    forward_case("forward_3d_rect8x16x32", (8, 16, 32), (1.5 * p, p, 30e-6),
                 [((0.1e-3, 0.2e-3, 0.5e-3), 0.3e-3, 0.8)], spec={"c": 2.0, "K": 4})
    forward_case("forward_2d_64x128", (64, 128), (p, 20e-6),
                 [((0.4e-3, 1.0e-3), 0.3e-3, 1.0), ((-1.5e-3, 1.8e-3), 0.5e-3, 0.5)])

    # window pair and warp known answers
    spec = rnufft.WindowSpec().resolved(2.0)
    xs = np.linspace(-3.5, 3.5, 57)
    th = np.linspace(-10, 10, 41)
    _save("window_pair", alpha=spec.alpha, beta=spec.beta, x=xs, ft=rnufft.window_ft_eval(spec, xs),
          theta=th, psi=rnufft.window_eval(spec, th),
          n_over_226=rnufft.NedPlan((226, 226)).n_over[0],
          kappa_345=rrecon.kappa(np.array([3.0, 0.0]), 4.0), amp_345=rrecon.amplitude_factor(3.0, 4.0))


if __name__ == "__main__":
    main()
