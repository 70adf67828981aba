"""Seeded random reconstruction problems of odd shapes for the parity sweep
(tests/test_gpu_fuzz.py, tools/fuzz_parity.py): 2D / 3D, non-power-of-two sizes,
out_dims != n_lateral, upsample 1-3, sensors on the aperture edge, windows with any
c / K and auto or explicit admissible (alpha, beta)."""
import math

import numpy as np

from paper_1501_02946_b200 import synth

SIZES = [8, 12, 16, 20, 24, 32, 40, 48, 64]


def draw(seed):
    rng = np.random.default_rng(seed)
    nlat = int(rng.integers(1, 3))
    nl = tuple(int(rng.choice(SIZES)) for _ in range(nlat))
    nt = int(rng.choice([16, 24, 32, 40, 48, 64, 96, 128, 192]))
    up = int(rng.choice([1, 1, 1, 2, 3]))
    dt = float(rng.choice([20e-9, 40e-9, 60e-9]))
    m = int(np.prod(nl))
    half = np.asarray(nl, float) * synth.PITCH / 2
    pos = rng.uniform(-half, half, size=(m, nlat))
    if rng.random() < 0.3:  # some sensors exactly on the aperture edges
        k = rng.integers(0, m, size=max(1, m // 20))
        pos[k, 0] = rng.choice([-half[0], half[0]], size=k.size)
    depth = nt * synth.SOUND_SPEED * dt
    if nlat == 2:
        balls = [(rng.uniform(-0.5, 0.5) * half[0], rng.uniform(-0.5, 0.5) * half[1], rng.uniform(0.2, 0.7) * depth,
                  rng.uniform(0.2e-3, 0.6e-3), rng.uniform(0.5, 1.0)) for _ in range(3)]
        samples = synth.ball_traces(pos, nt, dt, synth.SOUND_SPEED, balls)
    else:
        t = np.arange(nt) * dt
        dist = np.hypot(pos[:, 0] - 0.3e-3, 0.4 * depth)
        samples = np.exp(-((t[None, :] - dist[:, None] / synth.SOUND_SPEED) ** 2) / (2 * (2 * dt) ** 2))
    samples = samples + 1e-3 * rng.standard_normal(samples.shape)
    w = np.full(m, float(np.prod(np.asarray(nl) * synth.PITCH)) / m)
    out_dims = None
    if rng.random() < 0.3:
        out_dims = tuple(int(rng.choice([s for s in SIZES if s <= 2 * x])) for x in nl)
    c = float(rng.choice([1.5, 2.0, 2.0, 2.5, 3.0]))
    K = int(rng.integers(2, 9))
    alpha = beta = None
    if rng.random() < 0.4:
        lo, hi = max(c, math.pi) * 1.02, math.pi * (2 * c - 1) * 0.98
        if hi > lo:
            alpha = float(rng.uniform(lo, hi))
            beta = float(rng.uniform(0.3, 1.2) * K / c)
    if rng.random() < 0.5:  # non-uniform quadrature weights h_m (sum = aperture measure, recon.py:157-164)
        w = rng.uniform(0.2, 1.8, size=m)
        w *= float(np.prod(np.asarray(nl) * synth.PITCH)) / w.sum()
    return dict(positions=pos, weights=w, samples=samples, dt=dt, n_lateral=nl, out_dims=out_dims, upsample=up,
                c=c, K=K, alpha=alpha, beta=beta,
                desc=f"seed {seed}: nl={nl} nt={nt} up={up} out_dims={out_dims} c={c} K={K} alpha={alpha} beta={beta}")


def window_dynamic_range(case):
    """psi(0) / psi(pi) of the explicit window: the deapodisation and the NER pre-window amplify the
    float32 rounding of the gridding / FFTs by this factor towards the Nyquist frequencies (4.6 for
    the reference's default window)."""
    if case["alpha"] is None or case["beta"] is None:
        return 1.0
    from scipy.special import i0

    a, b = case["alpha"], case["beta"]
    return float(i0(b * a) / i0(b * math.sqrt(max(a * a - math.pi ** 2, 0.0))))


def draw_fast(seed):
    """Power-of-two problems that stay on the fast kernels (tensor-core gridding in both forms,
    shared-memory lateral FFTs, DCT-form NER, fused depth inverse): layouts, sample amplitudes over
    60 decades, out_dims, upsample, auto windows with K >= 4."""
    rng = np.random.default_rng(seed)
    nlat = 2 if rng.random() < 0.8 else 1
    nl = tuple(int(rng.choice([16, 32, 64])) for _ in range(nlat))
    nt = int(rng.choice([64, 128, 256, 512]))
    up = int(rng.choice([1, 1, 2]))
    dt = float(rng.choice([20e-9, 40e-9]))
    m = int(np.prod(nl)) * int(rng.choice([1, 1, 2]))  # up to twice as many sensors as grid points
    half = np.asarray(nl, float) * synth.PITCH / 2
    kind = rng.choice(["uniform", "clustered", "line"])
    if kind == "uniform":
        pos = rng.uniform(-half, half, size=(m, nlat))
    elif kind == "clustered":
        pos = np.clip(rng.normal(0.0, 0.25, size=(m, nlat)) * half, -half, half)
    else:  # all sensors on a few grid lines (very uneven gridding tiles)
        pos = rng.uniform(-half, half, size=(m, nlat))
        pos[:, 0] = rng.choice(np.linspace(-0.9, 0.9, 5), size=m) * half[0]
    depth = nt * synth.SOUND_SPEED * dt
    if nlat == 2:
        balls = [(rng.uniform(-0.5, 0.5) * half[0], rng.uniform(-0.5, 0.5) * half[1], rng.uniform(0.2, 0.7) * depth,
                  rng.uniform(0.2e-3, 0.6e-3), rng.uniform(0.5, 1.0)) for _ in range(3)]
        samples = synth.ball_traces(pos, nt, dt, synth.SOUND_SPEED, balls)
    else:
        t = np.arange(nt) * dt
        dist = np.hypot(pos[:, 0] - 0.3e-3, 0.4 * depth)
        samples = np.exp(-((t[None, :] - dist[:, None] / synth.SOUND_SPEED) ** 2) / (2 * (2 * dt) ** 2))
    samples = (samples + 1e-3 * rng.standard_normal(samples.shape)) * 10.0 ** float(rng.uniform(-30, 30))
    if rng.random() < 0.3:  # a few sensors far louder / quieter than the rest
        k = rng.integers(0, m, size=3)
        samples[k] *= 10.0 ** rng.uniform(-4, 4, size=(3, 1))
    w = np.full(m, float(np.prod(np.asarray(nl) * synth.PITCH)) / m)
    out_dims = None
    if rng.random() < 0.3:
        out_dims = tuple(int(rng.choice([16, 32, 64])) for _ in nl)
    K = int(rng.choice([4, 6, 6, 8]))
    if rng.random() < 0.5:
        w = rng.uniform(0.2, 1.8, size=m)
        w *= float(np.prod(np.asarray(nl) * synth.PITCH)) / w.sum()
    return dict(positions=pos, weights=w, samples=samples, dt=dt, n_lateral=nl, out_dims=out_dims, upsample=up,
                c=2.0, K=K, alpha=None, beta=None,
                desc=f"fast seed {seed}: nl={nl} M={m} {kind} nt={nt} up={up} out_dims={out_dims} K={K}")
