"""Time patfft_nedner_execute_batch on cfg4 for several direct-DMA shares (host-buffer e2e path).

usage (GPU box): PATFFT_HOST_TRACE=1 python tools/batch_probe.py [n] [fin,fout ...]
"""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_02946_b200 import NedNerPlan, _lib, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
shares = sys.argv[2:] or ["0.4,0.4"]
rec = synth.CONFIGS["cfg4"]()
lib = _lib.load()


def pinned(nbytes):
    p = ctypes.c_void_p()
    _lib.check(lib.patfft_host_alloc(nbytes, ctypes.byref(p)))
    return p


for sh in shares:
    fin, fout = sh.split(",")
    os.environ["PATFFT_BATCH_DIRECT_IN"] = fin
    os.environ["PATFFT_BATCH_DIRECT_OUT"] = fout
    plan = NedNerPlan(rec.positions, rec.weights, rec.samples.shape[1], rec.dt, rec.sound_speed, rec.dx, rec.n_lateral)
    nin, nout = rec.samples.size, int(np.prod(plan.out_shape))
    hin = pinned(8 * nin)
    np.ctypeslib.as_array(ctypes.cast(hin, ctypes.POINTER(ctypes.c_double)), shape=(nin,))[:] = rec.samples.ravel()
    houts = [pinned(8 * nout) for _ in range(2)]

    def batch(k):
        pin = (ctypes.c_void_p * k)(*[hin.value] * k)
        pout = (ctypes.c_void_p * k)(*[houts[i % 2].value for i in range(k)])
        bad = (ctypes.c_int64 * k)()
        _lib.check(lib.patfft_nedner_execute_batch(plan.handle, k, pin, pout, bad))

    batch(3)
    t0 = time.perf_counter()
    batch(n)
    dt = (time.perf_counter() - t0) / n
    print(f"direct in {fin} out {fout}: {1e3 * dt:.2f} ms/record", flush=True)
    for p in [hin] + houts:
        lib.patfft_host_free(p)
    plan.close()
