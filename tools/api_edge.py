"""Drop-in robustness: argument forms a caller of the reference may pass (GPU box)."""
import os, sys, threading
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_02946_b200 as pb
from oracle import nedner_oracle as O
from paper_1501_02946_b200 import synth

def rl2(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
s = synth.make_3d(77, 16, 64, 20e-9, "uniform", 2)
want, _ = O.reconstruct_nedner(s.positions, s.weights, s.samples, s.dt, s.sound_speed, s.dx, s.n_lateral)
def check(name, rec, **kw):
    try:
        f = pb.reconstruct_nedner(rec, **kw)
        print(f"{name}: rel-L2 {rl2(f.values, want):.2e} dtype {f.values.dtype} flags C={f.values.flags.c_contiguous}")
    except Exception as e:
        print(f"{name}: {type(e).__name__}: {str(e)[:120]}")
R = pb.SensorRecord
check("baseline", R(s.positions, s.weights, s.samples, s.dt, s.sound_speed, s.dx, s.n_lateral))
check("float32 samples", R(s.positions, s.weights, s.samples.astype(np.float32), s.dt, s.sound_speed, s.dx, s.n_lateral))
check("fortran-order samples", R(s.positions, s.weights, np.asfortranarray(s.samples), s.dt, s.sound_speed, s.dx, s.n_lateral))
big = np.zeros((s.samples.shape[0], 2 * s.samples.shape[1])); big[:, ::2] = s.samples
check("strided view samples", R(s.positions, s.weights, big[:, ::2], s.dt, s.sound_speed, s.dx, s.n_lateral))
check("list inputs", R(s.positions.tolist(), s.weights.tolist(), s.samples.tolist(), s.dt, s.sound_speed, s.dx, list(s.n_lateral)))
check("numpy ints", R(s.positions, s.weights, s.samples, np.float64(s.dt), np.float32(1500.0), np.float64(s.dx), np.array(s.n_lateral)), upsample=np.int64(1), out_dims=np.array([16, 16]))
check("readonly samples", R(s.positions, s.weights, (lambda a: (a.setflags(write=False), a)[1])(s.samples.copy()), s.dt, s.sound_speed, s.dx, s.n_lateral))
# reference-side errors
for name, kw in [("upsample 0", dict(upsample=0)), ("upsample 1.5", dict(upsample=1.5)), ("odd out_dims", dict(out_dims=(15, 16))),
                 ("out_dims wrong rank", dict(out_dims=(16,))), ("bad spec", dict(spec=pb.WindowSpec(c=2.0, K=6, alpha=1.0)) if False else dict())]:
    check(name, R(s.positions, s.weights, s.samples, s.dt, s.sound_speed, s.dx, s.n_lateral), **kw)
for name, fn in [("c<=1", lambda: pb.WindowSpec(c=1.0)), ("K=0", lambda: pb.WindowSpec(K=0)), ("alpha<pi", lambda: pb.WindowSpec(alpha=3.0)), ("beta<0", lambda: pb.WindowSpec(beta=-1.0))]:
    try: fn(); print(name, "accepted")
    except Exception as e: print(name, type(e).__name__)
nan = s.samples.copy(); nan[3, 5] = np.nan
check("NaN sample", R(s.positions, s.weights, nan, s.dt, s.sound_speed, s.dx, s.n_lateral))
# many plans (LRU eviction) and threads
for n in (8, 12, 16, 20, 24, 32, 8, 12):
    t = synth.make_3d(5, n, 32, 40e-9, "uniform", 1)
    f = pb.reconstruct_nedner(t.as_record())
print("plan churn ok", f.values.shape)
errs = []
def worker(k):
    try:
        for _ in range(5):
            f = pb.reconstruct_nedner(R(s.positions, s.weights, s.samples * (k + 1), s.dt, s.sound_speed, s.dx, s.n_lateral))
            e = rl2(f.values, want * (k + 1))
            if e > 1e-4: errs.append((k, e))
    except Exception as ex:
        errs.append((k, repr(ex)))
ths = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
[t.start() for t in ths]; [t.join() for t in ths]
print("threads:", "ok" if not errs else errs[:3])
