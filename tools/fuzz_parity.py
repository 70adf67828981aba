"""Randomised parity sweep: the drop-in vs the CPU oracle on small seeded records of odd shapes
(2D / 3D, non-power-of-two sizes, out_dims != n_lateral, upsample 1-3, windows with any c / K and
auto or explicit admissible alpha / beta).  usage (GPU box): python tools/fuzz_parity.py [n] [seed0]"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_02946_b200 as pb  # noqa: E402
from oracle import nedner_oracle as O  # noqa: E402  (checker)
from paper_1501_02946_b200 import synth  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from fuzz_cases import draw, window_dynamic_range  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
worst, fails, unsupported = 0.0, [], []
for i in range(n):
    cs = draw(seed0 + i)
    pos, w, samples, dt, nl, out_dims, up = (cs[k] for k in "positions weights samples dt n_lateral out_dims upsample".split())
    c, K, alpha, beta, desc = cs["c"], cs["K"], cs["alpha"], cs["beta"], cs["desc"]
    dr = window_dynamic_range(cs)
    if dr > 100:
        desc += f" [window dynamic range {dr:.0f}]"
    try:
        spec = pb.WindowSpec(c=c, K=K, alpha=alpha, beta=beta)
        rec = pb.SensorRecord(pos, w, samples, dt, synth.SOUND_SPEED, synth.PITCH, nl)
    except Exception as e:  # inadmissible draw
        print("skip", desc, type(e).__name__)
        continue
    try:
        want, _ = O.reconstruct_nedner(pos, w, samples, dt, synth.SOUND_SPEED, synth.PITCH, nl, out_dims=out_dims,
                                       upsample=up, spec=(c, K, alpha, beta))
    except Exception as e:
        print("oracle refuses", desc, type(e).__name__, str(e)[:80])
        try:
            pb.reconstruct_nedner(rec, out_dims=out_dims, upsample=up, spec=spec)
            fails.append(desc + " -- GPU accepted what the oracle refuses")
        except Exception as e2:
            print("   GPU too:", type(e2).__name__)
        continue
    try:
        got = pb.reconstruct_nedner(rec, out_dims=out_dims, upsample=up, spec=spec).values
    except pb.DeviceError as e:
        unsupported.append(desc + " :: " + str(e)[:100])
        continue
    err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
    worst = max(worst, err)
    flag = "" if err <= 1e-4 else "  <-- FAIL"
    print(f"{err:.2e} {desc}{flag}")
    if err > 1e-4 or got.shape != want.shape:
        fails.append(desc + f" rel-L2 {err:.2e}")
print(f"worst rel-L2 {worst:.2e}; {len(fails)} failures; {len(unsupported)} refused as unsupported")
for f in fails:
    print("FAIL", f)
for u in unsupported:
    print("UNSUPPORTED", u)
