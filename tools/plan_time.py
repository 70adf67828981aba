"""Plan creation time (first call for a new sensor layout) per BASELINE config (GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_02946_b200 import NedNerPlan, synth
for name in ("cfg1", "cfg2", "cfg3", "cfg4"):
    rec = synth.CONFIGS[name]()
    if isinstance(rec, (list, tuple)): rec = rec[0]
    for k in range(2):
        t0 = time.perf_counter()
        p = NedNerPlan(rec.positions, rec.weights, rec.samples.shape[1], rec.dt, rec.sound_speed, rec.dx, rec.n_lateral)
        dt = time.perf_counter() - t0
        p.close()
    print(name, f"plan creation {dt*1e3:.1f} ms")
