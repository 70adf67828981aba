"""Run a few device-resident reconstructions (for ncu / compute-sanitizer)."""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_02946_b200 import NedNerPlan, _lib, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--warm", type=int, default=0,
                help="reconstructions before cudaProfilerStart (use with ncu --profile-from-start off): the "
                     "first call of a plan re-runs the gridding because it has no sample-scale hint yet")
args = ap.parse_args()
rec = synth.CONFIGS[args.config]()
plan = NedNerPlan(rec.positions, rec.weights, rec.samples.shape[1], rec.dt, rec.sound_speed, rec.dx, rec.n_lateral)
lib = _lib.load()
s32 = np.ascontiguousarray(rec.samples, dtype=np.float32)
d_in, d_out = ctypes.c_void_p(), ctypes.c_void_p()
_lib.check(lib.patfft_device_alloc(0, s32.nbytes, ctypes.byref(d_in)))
_lib.check(lib.patfft_device_alloc(0, 4 * int(np.prod(plan.out_shape)), ctypes.byref(d_out)))
st = ctypes.c_void_p(plan.stream())
_lib.check(lib.patfft_memcpy_h2d(d_in, _lib.ptr(s32), s32.nbytes, st))
for _ in range(args.warm):
    plan.execute_device(d_in.value, d_out.value, st.value)
_lib.check(lib.patfft_stream_sync(st))
if args.warm:
    ctypes.CDLL("libcudart.so").cudaProfilerStart()
for _ in range(args.iters):
    plan.execute_device(d_in.value, d_out.value, st.value)
_lib.check(lib.patfft_stream_sync(st))
if args.warm:
    ctypes.CDLL("libcudart.so").cudaProfilerStop()
out = np.empty(plan.out_shape, dtype=np.float32)
_lib.check(lib.patfft_memcpy_d2h(_lib.ptr(out), d_out, out.nbytes, st))
_lib.check(lib.patfft_stream_sync(st))
print("ok", args.config, float(np.abs(out).max()))
