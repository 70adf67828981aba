"""Seeded synthetic sensor records shaped like BASELINE.json's configs.

There is no public dataset for this path (the paper's instrument data are
not available), so every benchmark and parity case runs on these seeded
stand-ins.  Geometry and signal models follow SURVEY.md section 8(d):

* positions: cell-centred jittered grid, uniform random, or clustered
  Gaussian (clipped to the aperture, which the reference's inclusive bound
  allows -- recon.py:131-136);
* weights: uniform h_m = X^(d-1)/M (the reference requires sum h = X^(d-1),
  recon.py:157-164);
* 3D signals: analytic N-wave of uniform balls, p = A (r - ct)/(2r) for
  |r - ct| <= R (the closed form the reference's forward.py:203-224 uses);
* 2D signals: Gaussian pulses (sigma = 2 dt) delayed by distance / c.

Everything is float64 on the host, like the reference's SensorRecord.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SOUND_SPEED = 1500.0
PITCH = 0.2e-3


@dataclass
class SyntheticRecord:
    positions: np.ndarray   # (M, d-1) metres
    weights: np.ndarray     # (M,)
    samples: np.ndarray     # (M, T) float64
    dt: float
    sound_speed: float
    dx: float
    n_lateral: tuple
    name: str = ""

    def as_record(self):
        from .recon import SensorRecord
        return SensorRecord(self.positions, self.weights, self.samples, self.dt,
                            self.sound_speed, self.dx, self.n_lateral)


def _jittered(rng, n_lateral, dx):
    axes = [((np.arange(n) + 0.5) - n / 2.0) * dx for n in n_lateral]
    mesh = np.meshgrid(*axes, indexing="ij")
    pos = np.stack([m.ravel() for m in mesh], axis=-1)
    return pos + rng.uniform(-0.4 * dx, 0.4 * dx, size=pos.shape)


def _uniform(rng, n_lateral, dx, m):
    half = np.asarray(n_lateral, float) * dx / 2.0
    return rng.uniform(-half, half, size=(m, len(n_lateral)))


def _clustered(rng, n_lateral, dx, m, sigma):
    half = np.asarray(n_lateral, float) * dx / 2.0
    return np.clip(rng.normal(0.0, sigma, size=(m, len(n_lateral))), -half, half)


def _uniform_weights(n_lateral, dx, m):
    meas = float(np.prod([n * dx for n in n_lateral]))
    return np.full(m, meas / m)


def ball_traces(positions, nt, dt, c, balls, out=None):
    """Sum of N-wave traces p = A (r - ct)/(2r), |r - ct| <= R, per sensor."""
    m = positions.shape[0]
    out = np.zeros((m, nt)) if out is None else out
    sens = np.concatenate([positions, np.zeros((m, 1))], axis=1)
    for (cx, cy, cz, rad, amp) in balls:
        centre = np.array([cx, cy, cz]) if sens.shape[1] == 3 else np.array([cx, cz])
        dist = np.linalg.norm(sens - centre, axis=1)
        lo = np.clip(np.floor((dist - rad) / (c * dt)).astype(np.int64), 0, nt)
        width = int(np.ceil(2 * rad / (c * dt))) + 3
        idx = lo[:, None] + np.arange(width)[None, :]
        valid = idx < nt
        idx_c = np.minimum(idx, nt - 1)
        u = c * dt * idx_c
        val = amp * (dist[:, None] - u) / (2.0 * dist[:, None])
        val[(np.abs(dist[:, None] - u) > rad) | ~valid] = 0.0
        rows = np.broadcast_to(np.arange(m)[:, None], idx.shape)
        np.add.at(out, (rows[valid], idx_c[valid]), val[valid])
    return out


def _balls(rng, count, half_lat, depth_max, lateral_dims=2):
    balls = []
    for _ in range(count):
        rad = rng.uniform(0.5e-3, 1.5e-3)
        amp = rng.uniform(0.5, 1.0)
        lat = rng.uniform(-0.7 * half_lat, 0.7 * half_lat, size=2)
        depth = rng.uniform(rad + 0.5e-3, max(rad + 0.6e-3, 0.8 * depth_max - rad))
        balls.append((lat[0], lat[1] if lateral_dims == 2 else 0.0, depth, rad, amp))
    return balls


def make_2d(seed=1, n=128, nt=512, dt=20e-9, sources=3):
    """Config 1: 128 jittered sensors on a 25.6 mm line, Gaussian pulses."""
    rng = np.random.default_rng(seed)
    pos = _jittered(rng, (n,), PITCH)
    t = np.arange(nt) * dt
    sig = 2 * dt
    depth_max = nt * SOUND_SPEED * dt
    samples = np.zeros((n, nt))
    for _ in range(sources):
        sx = rng.uniform(-0.35, 0.35) * n * PITCH
        sz = rng.uniform(2e-3, 0.8 * depth_max)
        amp = rng.uniform(0.5, 1.0)
        dist = np.hypot(pos[:, 0] - sx, sz)
        samples += amp * np.exp(-((t[None, :] - dist[:, None] / SOUND_SPEED) ** 2) / (2 * sig * sig))
    return SyntheticRecord(pos, _uniform_weights((n,), PITCH, n), samples, dt, SOUND_SPEED, PITCH, (n,), "cfg1-2d")


def make_3d(seed, n, nt, dt, layout, nballs, sigma=None):
    rng = np.random.default_rng(seed)
    nl = (n, n)
    m = n * n
    if layout == "jittered":
        pos = _jittered(rng, nl, PITCH)
    elif layout == "uniform":
        pos = _uniform(rng, nl, PITCH, m)
    elif layout == "clustered":
        pos = _clustered(rng, nl, PITCH, m, sigma)
    else:
        raise ValueError(layout)
    half = n * PITCH / 2
    balls = _balls(rng, nballs, half, nt * SOUND_SPEED * dt)
    samples = ball_traces(pos, nt, dt, SOUND_SPEED, balls)
    return SyntheticRecord(pos, _uniform_weights(nl, PITCH, m), samples, dt, SOUND_SPEED, PITCH, nl,
                           f"{layout}-{n}x{n}x{nt}")


CONFIGS = {
    # name: (builder, description) -- BASELINE.json configs, SURVEY.md 8(d)
    "cfg1": lambda seed=1: make_2d(seed),
    "cfg2": lambda seed=2: make_3d(seed, 64, 256, 20e-9, "jittered", 3),
    "cfg3": lambda seed=3: make_3d(seed, 128, 512, 20e-9, "uniform", 10),
    "cfg4": lambda seed=4: make_3d(seed, 256, 1024, 10e-9, "clustered", 20, sigma=8e-3),
}

DESCRIPTIONS = {
    "cfg1": "2D 128 jittered sensors x Nt=512, dt=20ns, 3 Gaussian-pulse sources -> (128, 512)",
    "cfg2": "3D 64x64 jittered sensors x Nt=256, dt=20ns, 3 balls -> (64, 64, 256)",
    "cfg3": "3D 128x128 uniform-random sensors x Nt=512, dt=20ns, 10 balls -> (128, 128, 512)",
    "cfg4": "3D 256x256 clustered (sigma 8mm) sensors x Nt=1024, dt=10ns, 20 balls -> (256, 256, 1024)",
    "cfg5": "3D batched: 64 frames of 128x128 jittered sensors x Nt=512 sharing one layout",
}


def make_frames(seed=5, frames=64, n=128, nt=512, dt=20e-9):
    """Config 5: one jittered layout, per-frame ball sets. Yields SyntheticRecord."""
    rng = np.random.default_rng(seed)
    nl = (n, n)
    pos = _jittered(rng, nl, PITCH)
    w = _uniform_weights(nl, PITCH, n * n)
    for f in range(frames):
        frng = np.random.default_rng([seed, f])
        balls = _balls(frng, 3, n * PITCH / 2, nt * SOUND_SPEED * dt)
        yield SyntheticRecord(pos, w, ball_traces(pos, nt, dt, SOUND_SPEED, balls), dt, SOUND_SPEED, PITCH,
                              nl, f"frame{f}")
