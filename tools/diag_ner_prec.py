"""Precision probe: GPU vs the float64 oracle on white-noise records, and the cfg4 linearity residual."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_02946_b200 as pb  # noqa: E402
from oracle import nedner_oracle as O  # noqa: E402
from paper_1501_02946_b200 import synth  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


for n, nt in [(16, 1024), (32, 512), (16, 2048)]:
    s = synth.make_3d(5, n, nt, 10e-9, "jittered", 1)
    r = s.as_record()
    r.samples = np.random.default_rng(3).standard_normal(r.samples.shape)
    g = pb.reconstruct_nedner(r).values
    o = O.reconstruct_nedner(r.positions, r.weights, r.samples, r.dt, r.sound_speed, r.dx, r.n_lateral)[0]
    print(f"noise {n}x{n}x{nt}: rel-L2 vs oracle {rel(g, o):.3e}", flush=True)
    s2 = synth.make_3d(6, n, nt, 10e-9, "jittered", 1)
    g2 = pb.reconstruct_nedner(s2.as_record()).values
    r2 = s2.as_record()
    o2 = O.reconstruct_nedner(r2.positions, r2.weights, r2.samples, r2.dt, r2.sound_speed, r2.dx, r2.n_lateral)[0]
    print(f"balls {n}x{n}x{nt}: rel-L2 vs oracle {rel(g2, o2):.3e}", flush=True)

s = synth.CONFIGS["cfg4"]()
r1 = s.as_record()
noise = np.random.default_rng(1).standard_normal(r1.samples.shape)
r2 = s.as_record()
r2.samples = noise
r3 = s.as_record()
r3.samples = 0.5 * r1.samples - 2.0 * noise
f1 = pb.reconstruct_nedner(r1).values
f1b = pb.reconstruct_nedner(r1).values
f2 = pb.reconstruct_nedner(r2).values
f3 = pb.reconstruct_nedner(r3).values
print("cfg4 deterministic", np.array_equal(f1, f1b), "finite", bool(np.all(np.isfinite(f1))))
print("cfg4 linearity residual %.3e" % rel(f3, 0.5 * f1 - 2.0 * f2))
