"""Where does the GPU volume differ from the oracle for one fuzz draw?  python tools/fuzz_diag.py SEED"""
import os, sys, math
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv_seed = int(sys.argv[1])
import paper_1501_02946_b200 as pb
from oracle import nedner_oracle as O
from paper_1501_02946_b200 import synth
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from fuzz_cases import draw
cs = draw(sys.argv_seed)
pos, w, samples, dt, nl, out_dims, up = (cs[k] for k in "positions weights samples dt n_lateral out_dims upsample".split())
c, K, alpha, beta = cs["c"], cs["K"], cs["alpha"], cs["beta"]
if os.environ.get("FUZZ_NO_EDGES"):
    pos = pos * (1.0 - 1e-9)
print("draw:", nl, samples.shape, up, out_dims, c, K, alpha, beta)
spec = pb.WindowSpec(c=c, K=K, alpha=alpha, beta=beta)
rec = pb.SensorRecord(pos, w, samples, dt, synth.SOUND_SPEED, synth.PITCH, nl)
got = pb.reconstruct_nedner(rec, out_dims=out_dims, upsample=up, spec=spec).values
want, _ = O.reconstruct_nedner(pos, w, samples, dt, synth.SOUND_SPEED, synth.PITCH, nl, out_dims=out_dims, upsample=up, spec=(c, K, alpha, beta))
exact, _ = O.reconstruct_nedner(pos, w, samples, dt, synth.SOUND_SPEED, synth.PITCH, nl, out_dims=out_dims, upsample=up)
d = got - want
print("rel-L2 gpu-vs-ref %.3e  ref-vs-exact %.3e  gpu-vs-exact %.3e" % (np.linalg.norm(d) / np.linalg.norm(want), np.linalg.norm(want - exact) / np.linalg.norm(exact), np.linalg.norm(got - exact) / np.linalg.norm(exact)))
D = np.fft.fftn(d)
W = np.fft.fftn(want)
idx = np.argsort(np.abs(D).ravel())[::-1][:12]
for k in idx:
    u = np.unravel_index(k, D.shape)
    print("bin", u, "|D| %.3e  |W| %.3e" % (abs(D[u]), abs(W[u])))
# energy of the difference per depth frequency and per lateral frequency
for ax in range(d.ndim):
    e = np.sum(np.abs(D) ** 2, axis=tuple(a for a in range(d.ndim) if a != ax))
    top = np.argsort(e)[::-1][:6]
    print("axis", ax, "top diff-energy bins", [(int(t), float(e[t] / e.sum())) for t in top])
