"""Where the public drop-in call spends its time at cfg4 (host side of the e2e path)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_02946_b200 import reconstruct_nedner, synth  # noqa: E402
from paper_1501_02946_b200.recon import _plan_for, _out_dims, WindowSpec  # noqa: E402


def t(fn, n=5):
    fn()
    xs = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        xs.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(xs))


for p in ("/sys/kernel/mm/transparent_hugepage/enabled", "/sys/kernel/mm/transparent_hugepage/defrag"):
    try:
        print(p, open(p).read().strip())
    except OSError as e:
        print(p, e)
rec = synth.CONFIGS[os.environ.get("CFG", "cfg4")]()
r = rec.as_record()
n_out = 256 * 256 * 1024
print("np.empty+fill 537MB  %.2f ms" % t(lambda: np.empty(n_out).fill(1.0)))
print("np.empty only        %.2f ms" % t(lambda: np.empty(n_out)))
print("as_record            %.2f ms" % t(lambda: rec.as_record()))
dims = _out_dims(tuple(r.n_lateral), None)
print("plan lookup          %.2f ms" % t(lambda: _plan_for(r, dims, 1, WindowSpec(), 0)))
plan = _plan_for(r, dims, 1, WindowSpec(), 0)
out = np.empty(plan.out_shape)
s = np.ascontiguousarray(r.samples)
print("execute, reused out  %.2f ms" % t(lambda: plan.execute(s, out)))
print("execute, fresh out   %.2f ms" % t(lambda: plan.execute(s)))
print("reconstruct_nedner   %.2f ms" % t(lambda: reconstruct_nedner(r)))
