#!/usr/bin/env python
"""Benchmark of the GPU forward model (forward_fourier, forward.py:105-166).

    python tools/bench_forward.py [--n 256] [--nt 1024] [--steps 20] [--warmup 3] [--no-cpu-baseline]

One step = full-grid traces of one (n, n, nt) initial-pressure field:
the lateral column / row FFT kernels of the reconstruction (cuFFT R2C on non-power-of-two grids), the fused NER-at-+-ky + depth-IFFT kernel
(csrc/ner_api.cu forward_kernel), the lateral inverse kernels (cuFFT C2R otherwise).  ``value`` is device-resident
(float32 field already in HBM, L2 flushed between steps, CUDA events on the
plan stream); ``e2e`` is the host entry point (float64 field in, float64
traces out, H2D/D2H inside).  The CPU baseline is the oracle restatement of
the reference (oracle/forward_oracle.py) on a bounded sample: the lateral
FFTs and depth IFFTs on 1/16 of the depth planes / rows and the NER on 1/16 of
the rows, extrapolated linearly.  Prints one JSON line.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1501_02946_b200 import ForwardPlan, _lib  # noqa: E402


def cpu_seconds(vals, spacing, sound_speed, frac):
    """Oracle forward model on a 1/frac slice of the work, extrapolated."""
    import scipy.fft as sfft

    from oracle import forward_oracle as F
    from oracle import nedner_oracle as O

    n0, n1, nt = vals.shape
    t0 = time.perf_counter()
    k = max(1, int(nt * frac))
    sfft.fftn(np.fft.ifftshift(vals[:, :, :k], axes=(0, 1)).astype(np.complex128), axes=(0, 1),
              workers=O._threads())                                     # lateral FFT on k depth planes
    t_lat = (time.perf_counter() - t0) * nt / k
    rows = max(1, int(n0 * n1 * frac))
    fb = (np.random.default_rng(0).standard_normal((rows, nt)) + 0j)
    j2 = np.linspace(0, 100, rows)
    nt2 = 2 * nt
    w = sfft.fftfreq(nt2) * nt2 / 2.0
    prop = j2[:, None] < w ** 2
    ky = np.where(prop, np.sign(w) * np.sqrt(np.maximum(w ** 2 - j2[:, None], 0.0)), 0.0)
    t1 = time.perf_counter()
    plan = O.NerOracle(nt)
    g = plan.rows(fb, ky) + plan.rows(fb, -ky)                          # NER at +-ky (forward.py:151-153)
    sfft.ifft(g, axis=-1, workers=O._threads())                         # depth IFFT (forward.py:155)
    t_ner = (time.perf_counter() - t1) * (n0 * n1) / rows
    del F
    return 2 * t_lat + t_ner, time.perf_counter() - t0                  # forward + inverse lateral FFTs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--nt", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    n, nt = args.n, args.nt
    c = 1500.0
    spacing = (0.2e-3, 0.2e-3, c * 10e-9)
    vals = np.random.default_rng(7).standard_normal((n, n, nt))
    plan = ForwardPlan(vals.shape, spacing)
    lib = _lib.load()

    def dalloc(nbytes):
        p = ctypes.c_void_p()
        _lib.check(lib.patfft_device_alloc(0, nbytes, ctypes.byref(p)))
        return p

    nvox = vals.size
    d_field, d_out, d_flush = dalloc(4 * nvox), dalloc(4 * nvox), dalloc(512 << 20)
    f32 = vals.astype(np.float32)
    stream = ctypes.c_void_p(0)
    LEGACY = 1  # cudaStreamLegacy: the plan's kernels and the events share the legacy default stream
    _lib.check(lib.patfft_memcpy_h2d(d_field, _lib.ptr(f32), f32.nbytes, stream))
    _lib.check(lib.patfft_stream_sync(stream))
    ev = []
    for _ in range(2 * args.steps):
        e = ctypes.c_void_p()
        _lib.check(lib.patfft_event_create(ctypes.byref(e)))
        ev.append(e)
    for _ in range(args.warmup):
        plan.execute_device(d_field.value, d_out.value, LEGACY)
    _lib.check(lib.patfft_stream_sync(stream))
    times = []
    for i in range(args.steps):
        _lib.check(lib.patfft_l2_flush(d_flush, 512 << 20, stream))
        _lib.check(lib.patfft_event_record(ev[2 * i], stream))
        plan.execute_device(d_field.value, d_out.value, LEGACY)
        _lib.check(lib.patfft_event_record(ev[2 * i + 1], stream))
    _lib.check(lib.patfft_stream_sync(stream))
    for i in range(args.steps):
        ms = ctypes.c_float()
        _lib.check(lib.patfft_event_elapsed_ms(ev[2 * i], ev[2 * i + 1], ctypes.byref(ms)))
        times.append(ms.value)
    ms_step = float(np.mean(times))
    # e2e: float64 host field -> float64 host traces (pageable numpy buffers, as the Python API)
    plan.execute(vals)
    et = []
    for _ in range(max(3, args.steps // 4)):
        t0 = time.perf_counter()
        plan.execute(vals)
        et.append(time.perf_counter() - t0)
    e2e_s = float(np.mean(et))
    # algorithmic bytes: field f32 in + traces f32 out + the half spectrum written and read twice
    spec = 8.0 * n * (n // 2 + 1) * nt
    alg = 4.0 * nvox * 2 + 4 * spec
    cpu = None
    if not args.no_cpu_baseline:
        os.environ.setdefault("PAT_THREADS", str(os.cpu_count() or 1))
        full, meas = cpu_seconds(vals, spacing, c, 1.0 / 16)
        cpu = {"value": nvox / full, "unit": "samples/s", "cores": int(os.environ["PAT_THREADS"]), "kind": "port",
               "sample": "oracle forward model: lateral FFTs on 1/16 of the depth planes, NER + depth IFFT on "
                         "1/16 of the rows, extrapolated", "measured_s": meas}
    line = {"metric": "forward-model sensor samples/sec (forward_fourier, full grid)", "value": nvox / (ms_step / 1e3),
            "unit": "samples/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "dtype": "f32/c64", "data": "synthetic (seeded N(0,1) field)",
            "config": {"workload": f"forward_fourier {n}x{n}x{nt}", "l2": "flushed (512 MiB write) between steps"},
            "roofline": {"bound": "hbm", "achieved": alg / (ms_step / 1e3) / 1e9, "unit": "GB/s",
                         "peak": 6546.9, "frac": alg / (ms_step / 1e3) / 1e9 / 6546.9, "algorithmic_bytes": alg,
                         "note": "whole step (cuFFT R2C + fused NER/IFFT kernel + cuFFT C2R) against the HBM peak"},
            "e2e": {"value": nvox / e2e_s, "unit": "samples/s", "ms_per_step": 1e3 * e2e_s,
                    "h2d_bytes_per_step": 8 * nvox, "d2h_bytes_per_step": 8 * nvox,
                    "path": "ForwardPlan.execute (C ABI patfft_forward_execute), pageable float64 numpy buffers"},
            "cpu_baseline": cpu}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
