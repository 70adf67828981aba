"""Would frames overlap pay?  64 cfg5 frames through one plan on one stream vs two plans (32 frames
each) on two streams.  (GPU box)"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_02946_b200 import NedNerPlan, synth
recs = synth.CONFIGS["cfg5"]() if "cfg5" in synth.CONFIGS else None
rec = synth.make_3d(5, 128, 512, 20e-9, "jittered", 10)
dev = torch.device("cuda", 0)
F = 64
x = torch.randn(F, rec.samples.shape[0], 512, device=dev)
mk = lambda: NedNerPlan(rec.positions, rec.weights, 512, rec.dt, rec.sound_speed, rec.dx, rec.n_lateral)
pa, pb_ = mk(), mk()
y = torch.empty((F,) + pa.out_shape, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
def one():
    pa.execute_frames_device(F, x.data_ptr(), y.data_ptr(), s1.cuda_stream)
def two():
    h = F // 2
    pa.execute_frames_device(h, x.data_ptr(), y.data_ptr(), s1.cuda_stream)
    pb_.execute_frames_device(h, x[h:].data_ptr(), y[h:].data_ptr(), s2.cuda_stream)
for fn, name in ((one, "one stream"), (two, "two streams")):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5): fn()
    torch.cuda.synchronize()
    print(name, (time.perf_counter() - t0) / 5 * 1e3, "ms per 64 frames")
