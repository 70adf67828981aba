"""Randomised sweep of the standalone APIs (row f): NerPlan, NedPlan, forward_fourier vs the oracle (GPU box)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_02946_b200 as pb
from oracle import nedner_oracle as O, forward_oracle as FO
from paper_1501_02946_b200 import synth

def rl2(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
worst = {"ner": 0, "ned": 0, "fwd": 0}; refused = []; fails = []
for i in range(n):
    rng = np.random.default_rng(4000 + i)
    c = float(rng.choice([1.5, 2.0, 2.0, 2.5, 3.0])); K = int(rng.integers(2, 9))
    spec = pb.WindowSpec(c=c, K=K)
    # --- NerPlan
    nn = int(rng.choice([16, 24, 32, 48, 64, 96, 128, 256])); rows = int(rng.integers(1, 6)); m = int(rng.integers(1, 40))
    u = rng.standard_normal((rows, nn)) + 1j * rng.standard_normal((rows, nn))
    ner = O.NerOracle(nn, c, K)
    shared = rng.random() < 0.5
    kap = rng.uniform(-ner.kappa_max, ner.kappa_max, size=(m,) if shared else (rows, m))
    kap.flat[0] = float(np.round(kap.flat[0] * 2) / 2)  # an exact half-integer target (integer c*kappa at c=2)
    try:
        got = pb.NerPlan(nn, spec).execute(u, kap)
        want = ner.shared(u, kap) if shared else ner.rows(u, kap)
        e = rl2(got, want); worst["ner"] = max(worst["ner"], e)
        if e > 1e-4: fails.append(f"ner seed {4000+i} n={nn} c={c} K={K} shared={shared}: {e:.2e}")
    except pb.DeviceError as ex:
        refused.append(f"ner n={nn} c={c} K={K}: {str(ex)[:70]}")
    # --- NedPlan
    nl = tuple(int(rng.choice([8, 12, 16, 24, 32])) for _ in range(int(rng.integers(1, 3))))
    M = int(rng.integers(5, 200)); nv = int(rng.choice([1, 3, 8]))
    pos = rng.uniform(-0.5, 0.5, size=(M, len(nl))) * np.asarray(nl)
    vals = rng.standard_normal((M, nv)) + 1j * rng.standard_normal((M, nv))
    try:
        got = pb.NedPlan(nl, spec).execute(pos, vals)
        want = O.NedOracle(nl, c, K).execute(pos, vals, wrapped=False)
        e = rl2(got, want); worst["ned"] = max(worst["ned"], e)
        if e > 1e-4: fails.append(f"ned seed {4000+i} nl={nl} c={c} K={K}: {e:.2e}")
    except pb.DeviceError as ex:
        refused.append(f"ned nl={nl} c={c} K={K}: {str(ex)[:70]}")
    # --- forward_fourier
    fl = tuple(int(rng.choice([8, 16, 32])) for _ in range(int(rng.integers(1, 3)))); nt = int(rng.choice([16, 32, 64, 128]))
    field = rng.standard_normal(fl + (nt,)) * np.exp(-np.arange(nt) / (0.4 * nt))
    dx = synth.PITCH; dy = dx * float(rng.choice([0.15, 0.3, 0.6]))
    try:
        f = pb.ScalarField(field, (dx,) * len(fl) + (dy,))
        got = pb.forward_fourier(f, synth.SOUND_SPEED, spec)
        want = FO.forward_fourier(field, (dx,) * len(fl) + (dy,), synth.SOUND_SPEED, c, K)
        ws = want[0] if isinstance(want, tuple) else want
        e = rl2(got.samples, np.asarray(ws).reshape(got.samples.shape)); worst["fwd"] = max(worst["fwd"], e)
        if e > 1e-4: fails.append(f"fwd seed {4000+i} fl={fl} nt={nt} c={c} K={K}: {e:.2e}")
    except pb.DeviceError as ex:
        refused.append(f"fwd fl={fl} nt={nt} c={c} K={K}: {str(ex)[:70]}")
print("worst", {k: f"{v:.2e}" for k, v in worst.items()}, "fails", len(fails), "refused", len(refused))
for f in fails[:20]: print("FAIL", f)
for r in refused[:12]: print("REFUSED", r)
