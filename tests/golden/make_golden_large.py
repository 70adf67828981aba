"""Golden summaries of the REFERENCE at BASELINE.json's large configs.

Run in the build container (where /root/reference exists), ~2 min + ~25 GB
RSS for cfg4 and a few minutes for the cfg5 frames:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_large.py [cfg4] [cfg5]

The full volumes are too large to commit (cfg4 is 0.5 GB of float64), so the
fixtures hold compact, sensitive summaries of the reference's own output of
``patfft.recon.reconstruct_nedner`` (``/root/reference/pkg/src/patfft/recon.py:358-379``):

* cfg4 (256^2 clustered sensors x Nt = 1024, seed 4):
  - 16 full depth planes (float32; z = 8, 72, ..., 968 -- every 64th plane
    from 8), one full lateral slice (row 128, all depths, float32),
  - the L2 norm of every depth plane (float64), the full-volume L2 norm,
  - the energy projection over depth, sum_z v^2 (256 x 256 float64; the plain
    sum over depth is ~0 -- the l = 0 plane is zero, recon.py:289 -- so it
    would only compare rounding noise),
  - sha256 of the float64 input samples, so the GPU test can prove it
    regenerated the same record from ``synth.CONFIGS['cfg4']``.
* cfg5 (64 frames of 128^2 jittered sensors x Nt = 512 sharing one layout):
  - per frame: L2 norm of every depth plane, full-volume L2 norm, sha256 of
    the input samples;
  - frames 0, 31 and 63: 8 full depth planes each (float32).

The GPU tests (tests/test_gpu_parity.py) regenerate the inputs with
``paper_1501_02946_b200.synth`` and compare their device output with these
numbers at the north_star bar (rel-L2 <= 1e-4).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("PATFFT_REFERENCE", "/root/reference/pkg/src")
sys.dont_write_bytecode = True
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from patfft import recon as rrecon  # noqa: E402  (reference)

from paper_1501_02946_b200 import synth  # noqa: E402  (seeded inputs only)

CFG4_PLANES = np.arange(8, 1024, 64)          # 16 depth planes
CFG4_ROW = 128
CFG5_FRAMES_FULL = (0, 31, 63)
CFG5_PLANES = np.arange(16, 512, 64)          # 8 depth planes


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _ref(s):
    r = rrecon.SensorRecord(positions=s.positions, weights=s.weights, samples=s.samples, dt=s.dt,
                            sound_speed=s.sound_speed, dx=s.dx, n_lateral=s.n_lateral)
    return rrecon.reconstruct_nedner(r)


def make_cfg4():
    s = synth.CONFIGS["cfg4"]()
    t0 = time.perf_counter()
    f = _ref(s)
    dt = time.perf_counter() - t0
    v = f.values
    assert v.shape == (256, 256, 1024)
    out = os.path.join(HERE, "large_cfg4.npz")
    np.savez_compressed(out, samples_sha256=sha(s.samples), planes_z=CFG4_PLANES,
                        planes=v[:, :, CFG4_PLANES].astype(np.float32), row=CFG4_ROW,
                        row_slice=v[CFG4_ROW].astype(np.float32),
                        plane_norms=np.linalg.norm(v.reshape(-1, v.shape[2]), axis=0),
                        total_norm=np.linalg.norm(v), depth_energy=(v * v).sum(axis=2),
                        spacing=np.asarray(f.spacing), imag_residual=f.meta["imag_residual"],
                        reference_seconds=dt)
    print(f"cfg4 reference {dt:.1f} s -> {out} ({os.path.getsize(out) / 1e6:.1f} MB)")


def _frame(args):
    idx, s = args
    v = _ref(s).values
    rec = {"idx": idx, "sha": sha(s.samples), "plane_norms": np.linalg.norm(v.reshape(-1, v.shape[2]), axis=0),
           "total": float(np.linalg.norm(v))}
    if idx in CFG5_FRAMES_FULL:
        rec["planes"] = v[:, :, CFG5_PLANES].astype(np.float32)
    return rec


def make_cfg5(workers=4):
    from multiprocessing import Pool

    frames = list(enumerate(synth.make_frames()))
    t0 = time.perf_counter()
    with Pool(workers) as pool:
        recs = sorted(pool.map(_frame, frames, chunksize=1), key=lambda r: r["idx"])
    dt = time.perf_counter() - t0
    out = os.path.join(HERE, "large_cfg5.npz")
    np.savez_compressed(out, samples_sha256=np.array([r["sha"] for r in recs]),
                        plane_norms=np.stack([r["plane_norms"] for r in recs]),
                        total_norms=np.array([r["total"] for r in recs]),
                        full_frames=np.array(CFG5_FRAMES_FULL), planes_z=CFG5_PLANES,
                        planes=np.stack([r["planes"] for r in recs if "planes" in r]),
                        reference_seconds=dt, workers=workers)
    print(f"cfg5 reference {dt:.1f} s ({workers} workers) -> {out} ({os.path.getsize(out) / 1e6:.1f} MB)")


if __name__ == "__main__":
    which = set(sys.argv[1:]) or {"cfg4", "cfg5"}
    if "cfg4" in which:
        make_cfg4()
    if "cfg5" in which:
        make_cfg5()
