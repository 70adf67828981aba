"""Run one golden through the drop-in (debugging aid: compute-sanitizer python tools/ref_dbg.py NAME)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_02946_b200 as pb
name = sys.argv[1]
g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", name + ".npz"))
a, b = float(g["spec_alpha"]), float(g["spec_beta"])
spec = pb.WindowSpec(c=float(g["spec_c"]), K=int(g["spec_K"]), alpha=None if np.isnan(a) else a, beta=None if np.isnan(b) else b)
rec = pb.SensorRecord(g["positions"], g["weights"], g["samples"], float(g["dt"]), float(g["sound_speed"]), float(g["dx"]),
                      tuple(int(n) for n in g["n_lateral"]))
f = pb.reconstruct_nedner(rec, out_dims=tuple(int(n) for n in g["out_dims"]), upsample=int(g["upsample"]), spec=spec)
print(name, "rel-L2", np.linalg.norm(f.values - g["values"]) / np.linalg.norm(g["values"]))
