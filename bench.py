#!/usr/bin/env python
"""Benchmark: reconstructed voxels/s of the NEDNER-NUFFT path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl reference]

A "step" is one full reconstruction (NED spread -> lateral FFT -> crop ->
fused NER -> inverse FFT) of one synthetic record.  ``value`` is measured
device-resident (float32 samples already in HBM); ``e2e`` goes through the
C ABI's host entry point (float64 host samples in pinned memory, H2D + D2H
inside the timed region).  ``--impl reference`` times the CPU oracle (the
restated reference algorithm, float64 numpy/scipy) on a bounded sample of
the same workload.

For N > 1 one record is reconstructed by all N ranks together (strong
scaling, paper_1501_02946_b200/parallel.py): each rank spreads and
lateral-FFTs its own time slice, an NCCL all-to-all hands every rank its
lateral-frequency rows, each rank runs the fused NER on its rows, and a
second all-to-all returns depth slices for the lateral inverse.  ``value`` is
the record's voxels over the max per-rank device time.  Launched by the
driver under torchrun (RANK / WORLD_SIZE / LOCAL_RANK from the environment);
``python bench.py --gpus N`` without a launcher re-executes itself under
``torch.distributed.run`` with N local ranks.  cfg5 (independent frames)
runs as replicas: every rank reconstructs its own 64 frames.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

# The driver parses stdout as one JSON line: libraries that print at init
# (NCCL's version banner, cuFFT/driver notes) are sent to stderr by pointing
# fd 1 there for the whole run; emit() writes the result line to the real stdout.
_STDOUT_FD = None


def _quiet_stdout():
    global _STDOUT_FD
    if _STDOUT_FD is None:
        sys.stdout.flush()
        _STDOUT_FD = os.dup(1)
        os.dup2(2, 1)


def emit(line: dict) -> None:
    text = json.dumps(line) + "\n"
    sys.stdout.flush()
    os.write(_STDOUT_FD if _STDOUT_FD is not None else 1, text.encode())

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "reconstructed voxels/sec (3D NEDNER-NUFFT)"
UNIT = "voxels/s"


def _tf32_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"]) / 2.0
    except Exception:
        return 1100.0


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = f"/tmp/patfft_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def make_workload(name, rank=0):
    from paper_1501_02946_b200 import synth

    if name == "cfg5":
        frames = list(synth.make_frames(seed=5 + 1000 * rank, frames=64))
        return frames
    seed = {"cfg1": 1, "cfg2": 2, "cfg3": 3, "cfg4": 4}[name] + 1000 * rank
    return [synth.CONFIGS[name](seed)]


# ---------------------------------------------------------------------------
# CPU baseline (oracle = restated reference), bounded sample + extrapolation
# ---------------------------------------------------------------------------

def cpu_sample_seconds(rec, frac):
    """Time the reference algorithm on ``frac`` of the work and extrapolate.

    NED: the full plan (spread operator) + SpMM/FFT/crop on frac of the time
    samples (the operator is identical for every time sample).  NER: frac of
    the lateral rows.  Inverse FFT: frac of the depth planes (lateral 2-D
    IFFTs) and frac of the rows (depth IFFTs) -- the separable parts of the
    reference's ifftn.  Returns (extrapolated full seconds, measured seconds).
    """
    import scipy.fft as sfft

    from oracle import nedner_oracle as O

    pos, w, smp = rec.positions, rec.weights, rec.samples
    nl = tuple(rec.n_lateral)
    nt = smp.shape[1]
    dd = len(nl)
    thr = int(os.environ.get("PAT_THREADS", "1"))
    t0 = time.perf_counter()
    scaled = smp * (w / rec.dx ** dd)[:, None]
    ned = O.NedOracle(nl)
    gp = pos / rec.dx
    op = ned.spread_operator(gp)
    t_plan = time.perf_counter() - t0
    tf = max(1, int(round(nt * frac)))
    t1 = time.perf_counter()
    vb = scaled[:, :tf].astype(np.complex128)
    grid = (op @ vb).reshape(ned.n_over + (tf,))
    spec = sfft.fftn(grid, axes=tuple(range(dd)), workers=thr)
    sel = [np.arange(-n // 2, n // 2) % m for n, m in zip(nl, ned.n_over)]
    gh_part = spec[np.ix_(*sel)]
    for ax, dp in enumerate(ned.deapod):
        shape = [1] * gh_part.ndim
        shape[ax] = dp.size
        gh_part = gh_part * dp.reshape(shape)
    gh_part = np.fft.ifftshift(gh_part, axes=tuple(range(dd)))
    t_ned = time.perf_counter() - t1
    # NER on frac of the lateral rows (cost is data-independent; rows carry noise)
    rows = int(np.prod(nl))
    rsub = max(1, int(round(rows * frac)))
    ratios = O.lateral_ratios(nt, rec.dt, rec.sound_speed, rec.dx, nl)
    j2 = O.lateral_freq_sq(nl, ratios).reshape(rows)[:rsub]
    rng = np.random.default_rng(0)
    gh_rows = rng.standard_normal((rsub, nt)) + 1j * rng.standard_normal((rsub, nt))
    t2 = time.perf_counter()
    fh = O.fhat_rows(gh_rows, j2, nt, (2.0, 6, None, None))
    t_ner = time.perf_counter() - t2
    # inverse (recon.py:249-260) on frac of the volume: Hermitian part and
    # lateral IFFTs on frac of the depth planes, depth IFFTs on frac of rows
    planes = max(1, int(round(nt * frac)))
    slab = rng.standard_normal(nl + (planes,)) + 0j
    t3 = time.perf_counter()
    O.hermitian_part(slab)
    lat = sfft.ifftn(slab, axes=tuple(range(dd)))
    np.fft.fftshift(lat.real, axes=tuple(range(dd)))
    sfft.ifft(fh, axis=-1)
    t_inv = time.perf_counter() - t3
    measured = t_plan + t_ned + t_ner + t_inv
    full = t_plan + (t_ned + t_ner + t_inv) / frac
    return full, measured


def _reference_module():
    """The unmodified reference package, installed once into baseline/_ref with
    ``python -m pip install --no-index --no-build-isolation --no-deps --target
    baseline/_ref <copy of /root/reference/pkg>``.  Pure
    Python, so the install travels to the GPU box with the repo snapshot."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "patfft")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    sys.dont_write_bytecode = True
    try:
        import patfft.recon as R
    except Exception:
        return None
    return R


def run_reference_arm(args):
    """CPU reference on this host's cores, on the GPU arm's config and metric.

    With ``baseline/_ref`` installed: the reference's own public call
    ``patfft.recon.reconstruct_nedner`` (recon.py:358-379) on the full record,
    repeated until ``--steps`` runs are done or the next run would exceed the
    arm's time budget (``--ref-budget``, default 240 s; one cfg4 run takes
    ~100 s), so the line's ``steps`` / ``ms_per_step`` are what actually ran.
    cfg5 times whole frames and scales to the 64-frame step.  The oracle
    port's 1/16-sample extrapolation is reported beside it.  Without the
    install, the oracle port's sample is the value (``kind`` "port").
    """
    rank, world, _ = _env_rank()
    if rank != 0:
        return 0
    os.environ.setdefault("PAT_THREADS", str(os.cpu_count() or 1))
    cores = int(os.environ["PAT_THREADS"])
    recs = make_workload(args.config)
    rec = recs[0]
    n_frames = len(recs)
    vox = _voxels(rec) * n_frames
    frac = args.cpu_frac or 1.0 / 16
    R = _reference_module()
    extra = {}
    if R is not None:
        budget = args.ref_budget
        times = []
        t_start = time.perf_counter()
        k = 0
        while True:
            r = recs[k % n_frames]
            rr = R.SensorRecord(positions=r.positions, weights=r.weights, samples=r.samples, dt=r.dt,
                                sound_speed=r.sound_speed, dx=r.dx, n_lateral=r.n_lateral)
            t0 = time.perf_counter()
            R.reconstruct_nedner(rr)
            times.append(time.perf_counter() - t0)
            k += 1
            done = len(times) >= max(1, args.steps) * (n_frames if n_frames > 1 else 1)
            if n_frames > 1:
                done = done or len(times) >= 2 and time.perf_counter() - t_start + times[-1] > budget
            else:
                done = done or time.perf_counter() - t_start + times[-1] > budget
            if done:
                break
        per_rec = float(np.mean(times))
        step_s = per_rec * n_frames
        value = vox / step_s
        steps = max(1, len(times) // n_frames) if n_frames > 1 else len(times)
        kind = "reference"
        sample = (f"{args.config}: the reference package itself (baseline/_ref, patfft.recon.reconstruct_nedner, "
                  f"float64 numpy/scipy, PAT_THREADS={cores} for its FFTs, the rest single-threaded as written), "
                  f"{len(times)} full {'frame' if n_frames > 1 else 'reconstruction'}"
                  f"{'s' if len(times) != 1 else ''} of {per_rec:.1f} s each"
                  + (f", scaled to the {n_frames}-frame step" if n_frames > 1 else ""))
        extra["reference_runs_s"] = times
        extra["requested"] = {"steps": args.steps, "warmup": args.warmup}
        if len(times) < args.steps * (n_frames if n_frames > 1 else 1):
            extra["deviation"] = (f"ran {len(times)} full reference {'frames' if n_frames > 1 else 'reconstructions'} "
                                  f"instead of {args.steps} steps: each takes {per_rec:.0f} s and the arm's budget is "
                                  f"{budget:.0f} s; no warm-up (nothing to warm in numpy/scipy)")
        full, meas = cpu_sample_seconds(rec, frac)
        extra["port_sample_extrapolation"] = {"value": _voxels(rec) / full, "unit": UNIT,
                                              "sample": _sample_desc(args.config, frac), "measured_s": meas,
                                              "extrapolated_full_s": full}
    else:
        vals = []
        for i in range(args.warmup + args.steps):
            full, meas = cpu_sample_seconds(rec, frac)
            if i >= args.warmup:
                vals.append(_voxels(rec) / full)
        value = statistics.median(vals)
        step_s = vox / value
        steps = args.steps
        kind = "port"
        sample = _sample_desc(args.config, frac)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": steps, "warmup": 0 if kind == "reference" else args.warmup, "ms_per_step": 1e3 * step_s,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE config shapes)", "config": _config_json(args, rec, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample,
                         "os_cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    line.update(extra)
    emit(line)
    return 0


def _sample_desc(cfg, frac):
    return (f"{cfg}, oracle (restated reference, float64 numpy/scipy, PAT_THREADS=all cores for FFTs): "
            f"full NED plan + NED on {frac:g} of the time samples + NER on {frac:g} of the lateral rows + "
            f"inverse FFT on {frac:g} of planes/rows, extrapolated linearly to the full step")


def _voxels(rec):
    return int(np.prod(rec.n_lateral)) * rec.samples.shape[1]


def _config_json(args, rec, world=1):
    from paper_1501_02946_b200 import synth

    return {"workload": f"{args.config}: {synth.DESCRIPTIONS[args.config]}",
            "sensors": int(rec.positions.shape[0]), "n_time": int(rec.samples.shape[1]),
            "out_shape": list(rec.n_lateral) + [int(rec.samples.shape[1])],
            "window": "Kaiser-Bessel c=2 K=6 (reference default)",
            "l2": "inputs (>=268 MB at cfg4) exceed L2 and a 512 MB scratch write flushes L2 between steps",
            "parallelism": ("single-gpu" if world == 1 else
                            f"replicas x{world}" if args.config == "cfg5" else f"sharded x{world}")}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_sharded_arm(args):
    """One cfg reconstruction split over all ranks (strong scaling, NCCL all-to-all x2)."""
    import torch
    import torch.distributed as dist

    from paper_1501_02946_b200.parallel import ShardedNedNer

    rank, world, local = _env_rank()
    # PATFFT_DIST_BACKEND=gloo: the same arm with several ranks on ONE GPU (host-staged exchanges,
    # parallel._host_exchange) -- a functional check of the multi-rank path where only one GPU exists
    backend = os.environ.get("PATFFT_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local %= max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    rec = make_workload(args.config, 0)[0]  # every rank: the same record, its own time slice
    T = rec.samples.shape[1]
    sh = ShardedNedNer(rec.positions, rec.weights, T, rec.dt, rec.sound_speed, rec.dx, rec.n_lateral,
                       torch_device=dev)
    tr = sh.layout.Tr
    host_slice = np.ascontiguousarray(rec.samples[:, rank * tr:(rank + 1) * tr])
    d_slice = torch.tensor(host_slice, dtype=torch.float32, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    st = sh.cuda_stream
    for _ in range(args.warmup):
        sh.run(d_slice)
    torch.cuda.synchronize()
    clocks = Clocks(local)
    dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    times = []
    for _ in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.wait_stream(torch.cuda.current_stream(dev))
        a.record(st)
        sh.run(d_slice)
        b.record(st)
        b.synchronize()
        times.append(a.elapsed_time(b))
    torch.cuda.synchronize()
    clk = clocks.stop()
    dist.barrier()
    t = torch.tensor([float(np.mean(times))], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item())
    vox = _voxels(rec)
    value = vox / (ms_step / 1e3)

    # roofline of the rank's dominant kernel (the gridding of its time slice), timed alone on the
    # stream it is launched on; algorithmic bytes 4 * Tr * (M + nrows * ncols)
    sp_times = []
    for _ in range(max(3, args.steps)):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.wait_stream(torch.cuda.current_stream(dev))
        a.record(st)
        with torch.cuda.stream(st):
            sh.stages.spread(d_slice, st.cuda_stream)
        b.record(st)
        b.synchronize()
        sp_times.append(a.elapsed_time(b))
    t = torch.tensor([float(np.mean(sp_times[1:]))], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    spread_ms = float(t.item())
    n_over = [1 << int(np.ceil(np.log2(2 * n))) for n in rec.n_lateral]
    spread_bytes = 4.0 * tr * (rec.samples.shape[0] + int(np.prod(n_over)))
    peak, peak_kind = _peaks()
    roofline = {"kernel": "spread (per rank: spread_tc16_kernel on the rank's time slice + scale check)",
                "bound": "hbm", "achieved": spread_bytes / (spread_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                "frac": spread_bytes / (spread_ms / 1e3) / 1e9 / peak, "peak_source": peak_kind, "traffic": None,
                "algorithmic_bytes": spread_bytes, "launch_ms": spread_ms}

    # e2e: pinned f64 host slice -> device -> f32, sharded run, image slice -> pinned f64 host
    pin_in = torch.from_numpy(host_slice).pin_memory()
    pin_out = torch.empty(sh.layout.image_slice_shape(), dtype=torch.float64).pin_memory()
    et = []
    for i in range(args.warmup + args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x = pin_in.to(dev, non_blocking=True).float()
        img = sh.run(x)
        pin_out.copy_(img.double(), non_blocking=True)
        torch.cuda.synchronize()
        if i >= args.warmup:
            et.append(time.perf_counter() - t0)
    t = torch.tensor([float(np.mean(et))], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32/c64", "data": "synthetic (seeded, BASELINE config shapes)",
            "config": dict(_config_json(args, rec, world), parallelism=f"sharded x{world}: time-sliced NED, "
                           "pipelined all-to-all, row-sliced NER, pipelined all-to-all, time-sliced lateral inverse"),
            "clocks": clk, "roofline": roofline,
            "e2e": {"value": vox / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * host_slice.size * world,
                    "d2h_bytes_per_step": 8 * int(np.prod(pin_out.shape)) * world, "ms_per_step": 1e3 * e2e_s},
            "gpu_launches": (5 + 2 * sh.C + sh.B) * args.steps,
            "gpu_launches_note": (f"per rank per step: spread + scale check + conditional re-spread (fp16 gridding), colfft + "
                                  f"rowfft per time piece ({sh.C} pieces), ner per row block ({sh.B} blocks), inv_col "
                                  f"+ inv_c2r (+1 flush outside the events); grouped NCCL send/recv per piece and per "
                                  f"block (none at world 1)"),
            "pipeline": {"time_pieces": sh.C, "row_blocks": sh.B},
        }
        emit(line)
    dist.destroy_process_group()
    return 0


def run_gpu_arm(args):
    rank, world, local = _env_rank()
    if args.gpus > 1 or world > 1 or args.sharded:
        from paper_1501_02946_b200.parallel import ShardLayout

        rec_T = {"cfg1": 512, "cfg2": 256, "cfg3": 512, "cfg4": 1024}.get(args.config)
        if rec_T and ShardLayout.supported(rec_T, world):
            return run_sharded_arm(args)
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    device = local
    from paper_1501_02946_b200 import NedNerPlan, _lib, reconstruct_nedner

    lib = _lib.load()
    recs = make_workload(args.config, rank)
    rec = recs[0]
    plan = NedNerPlan(rec.positions, rec.weights, rec.samples.shape[1], rec.dt, rec.sound_speed, rec.dx,
                      rec.n_lateral, device=device)
    stream = ctypes.c_void_p(plan.stream())
    nsamp = rec.samples.size
    nout = int(np.prod(plan.out_shape))
    nframes = len(recs)

    def dalloc(nbytes):
        p = ctypes.c_void_p()
        _lib.check(lib.patfft_device_alloc(device, nbytes, ctypes.byref(p)))
        return p

    d_in = dalloc(4 * nsamp * nframes)
    d_out = dalloc(4 * nout * nframes)
    host32 = np.ascontiguousarray(np.stack([r.samples for r in recs]).astype(np.float32))
    _lib.check(lib.patfft_memcpy_h2d(d_in, _lib.ptr(host32), host32.nbytes, stream))
    _lib.check(lib.patfft_stream_sync(stream))
    flush_bytes = 512 << 20
    d_flush = dalloc(flush_bytes)
    ev = []
    for _ in range(2 * args.steps + 2):
        e = ctypes.c_void_p()
        _lib.check(lib.patfft_event_create(ctypes.byref(e)))
        ev.append(e)

    def step():
        if nframes == 1:
            plan.execute_device(d_in.value, d_out.value, stream.value)
        else:
            plan.execute_frames_device(nframes, d_in.value, d_out.value, stream.value)

    for _ in range(args.warmup):
        step()
    _lib.check(lib.patfft_stream_sync(stream))

    clocks = Clocks(device)
    if dist is not None:
        dist.barrier()
    _lib.check(lib.patfft_stream_sync(stream))
    clocks.start()
    times = []
    for i in range(args.steps):
        _lib.check(lib.patfft_l2_flush(d_flush, flush_bytes, stream))
        _lib.check(lib.patfft_event_record(ev[2 * i], stream))
        step()
        _lib.check(lib.patfft_event_record(ev[2 * i + 1], stream))
        ms = ctypes.c_float()
        _lib.check(lib.patfft_event_elapsed_ms(ev[2 * i], ev[2 * i + 1], ctypes.byref(ms)))
        times.append(ms.value)
    _lib.check(lib.patfft_stream_sync(stream))
    clk = clocks.stop()
    if dist is not None:
        dist.barrier()
    # per-stage breakdown: a separate pass with stage events (stages serialised,
    # so each kernel's duration is attributable; the timed steps above overlap
    # the spread with the lateral FFTs on two streams)
    plan.set_profiling(True)
    for _ in range(max(3, args.steps // 2)):
        _lib.check(lib.patfft_l2_flush(d_flush, flush_bytes, stream))
        step()
    _lib.check(lib.patfft_stream_sync(stream))
    stages = plan.stage_times()
    plan.set_profiling(False)
    ms_step = float(np.mean(times))
    if dist is not None:
        import torch

        t = torch.tensor([ms_step], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    vox = _voxels(rec) * nframes
    value = vox * world / (ms_step / 1e3)

    # ---- end-to-end through the host entry point (pinned f64 buffers) ----
    e2e = None
    # ---- end-to-end through the host entry points (float64 host buffers) ----
    # A step is one record (cfg5: the 64 frames).  Timed: patfft_nedner_execute_batch over the
    # steps' records, i.e. the records a user streams through one plan: record k+1 is narrowed
    # and uploaded and record k-1 downloaded and widened while record k is reconstructed.
    # Every record's upload from pinned float64 host memory and its download into a float64
    # host volume are inside the timed region.  The one-shot call (patfft_nedner_execute, no
    # neighbour to overlap with) and the Python drop-in are timed beside it.
    def pinned(nbytes):
        p = ctypes.c_void_p()
        _lib.check(lib.patfft_host_alloc(nbytes, ctypes.byref(p)))
        return p, np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), shape=(nbytes // 8,))

    hins = [pinned(8 * nsamp) for _ in range(nframes)]
    for (p_, a_), r in zip(hins, recs):
        a_[:] = r.samples.ravel()
    houts = [pinned(8 * nout) for _ in range(2)]
    hin_ptrs = [p_.value for p_, _ in hins]
    hout_ptrs = [p_.value for p_, _ in houts]

    def batch(nrec):
        pin = (ctypes.c_void_p * nrec)(*[hin_ptrs[k % nframes] for k in range(nrec)])
        pout = (ctypes.c_void_p * nrec)(*[hout_ptrs[k % 2] for k in range(nrec)])
        bad = (ctypes.c_int64 * nrec)()
        _lib.check(lib.patfft_nedner_execute_batch(plan.handle, nrec, pin, pout, bad))
        return sum(bad)

    batch(max(3, nframes))  # warm-up: buffers, graphs, host pool
    if dist is not None:
        dist.barrier()
    nrec = args.steps * nframes
    t0 = time.perf_counter()
    nbad = batch(nrec)
    e2e_s = (time.perf_counter() - t0) / args.steps
    if dist is not None:
        import torch

        t = torch.tensor([e2e_s], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    # bytes that cross PCIe per step, as the batch path splits them (capi.cu
    # patfft_nedner_execute_batch): pinned caller buffers >= 4 MiB send sensor rows
    # [0, batch_direct_in * M) and voxels [0, batch_direct_out * n) as float64 by DMA
    m_rows, t_len = rec.samples.shape
    fin = min(1.0, max(0.0, float(os.environ.get("PATFFT_BATCH_DIRECT_IN", "0.4"))))
    fout = min(1.0, max(0.0, float(os.environ.get("PATFFT_BATCH_DIRECT_OUT", "0.4"))))
    md = int(fin * m_rows) if 8 * nsamp >= (4 << 20) else 0
    od = int(fout * nout) // 256 * 256 if 8 * nout >= (4 << 20) else 0
    h2d_b = (8 * md * t_len + 4 * (nsamp - md * t_len)) * nframes
    d2h_b = (8 * od + 4 * (nout - od)) * nframes
    e2e = {"value": vox * world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b,
           "ms_per_step": 1e3 * e2e_s, "records_timed": nrec, "nonfinite_voxels": int(nbad),
           "path": ("patfft_nedner_execute_batch (C ABI), pinned float64 host buffers: per record the host cores "
                    "narrow a share of the sensor rows to float32 into pinned staging and the rest crosses as "
                    "float64 by DMA (narrowed on the device); the float32 volume returns the same way (host "
                    "widening + float64 DMA of a share); record k+1 uploads and k-1 downloads while k is "
                    "reconstructed")}
    if nframes == 1:
        resid = ctypes.c_double()
        hin, hout = hins[0][0], houts[0][0]
        _lib.check(lib.patfft_nedner_execute(plan.handle, hin, hout, ctypes.byref(resid)))
        et = []
        for _ in range(min(5, args.steps)):
            t0 = time.perf_counter()
            _lib.check(lib.patfft_nedner_execute(plan.handle, hin, hout, ctypes.byref(resid)))
            et.append(time.perf_counter() - t0)
        e2e["single_call_ms"] = 1e3 * float(np.mean(et))
        e2e["single_call_path"] = ("patfft_nedner_execute (C ABI), one record: upload in time chunks overlapped "
                                   "with the spread + lateral FFTs, download after the NER and inverse")
        if world == 1:
            # the Python drop-in with ordinary (pageable) numpy arrays, as a user calls it
            rec_obj = rec.as_record()
            reconstruct_nedner(rec_obj)
            pt = []
            for _ in range(min(5, args.steps)):
                t0 = time.perf_counter()
                reconstruct_nedner(rec_obj)
                pt.append(time.perf_counter() - t0)
            e2e["public_api_pageable_ms"] = 1e3 * float(np.median(pt))
    for p_, _ in hins + houts:
        lib.patfft_host_free(p_)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel ----
    o, lb = ctypes.c_int(), ctypes.c_int()
    _lib.check(lib.patfft_nedner_launches_per_execute(plan.handle, ctypes.byref(o), ctypes.byref(lb)))
    own_launches, lib_launches = o.value, lb.value
    peak, peak_kind = _peaks()
    sbytes = plan.stage_bytes()
    per = {k: (stages[k][0] / max(1, stages[k][1])) for k in stages}
    dom = max(per, key=lambda k: per[k])
    ach = sbytes[dom] / (per[dom] / 1e3) / 1e9
    traffic = _traffic_from_profiles(args.config, dom)
    roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "peak_source": peak_kind, "traffic": traffic, "algorithmic_bytes": sbytes[dom],
            "launch_ms": per[dom]}
    # the spread (gridding) kernel: HBM fraction plus its own bound
    info = (ctypes.c_int64 * 4)()
    _lib.check(lib.patfft_nedner_spread_info(plan.handle, info))
    sp_ms = per["spread"]
    taps = 12 ** len(rec.n_lateral)
    useful = 2.0 * rec.positions.shape[0] * taps * rec.samples.shape[1]  # useful FLOPs: 2 x M x (2K)^d x T
    spec_on = os.environ.get("PATFFT_TC16_SPECULATE", "1") != "0"
    spread = {"kernel": {2: "spread_tc16_kernel (tcgen05 kind::f16, two-term fp16 split) + "
                            + ("check_scale_kernel + a second gridding launch that exits at once when the sample-scale "
                               "hint of the plan's previous call was right (it is on every timed step: same record; "
                               "a miss re-runs the gridding, +0.34 ms at cfg4, with bit-identical results)"
                               if spec_on else "absmax_kernel"),
                         1: "spread_tc_kernel (tcgen05 3xTF32)"}.get(int(info[0]), "spread_tp_kernel (SIMT FP32)"),
              "launch_ms": sp_ms, "algorithmic_bytes": sbytes["spread"],
              "hbm": {"achieved": sbytes["spread"] / (sp_ms / 1e3) / 1e9, "peak": peak,
                      "frac": sbytes["spread"] / (sp_ms / 1e3) / 1e9 / peak},
              "traffic": _traffic_from_profiles(args.config, "spread")}
    if info[0]:
        f16 = int(info[0]) == 2
        tc_peak = _tf32_peak() * (2.0 if f16 else 1.0)
        executed = 3 * 2.0 * 128 * info[1] * rec.samples.shape[1]  # 3 products per 128-point record
        spread["tensor"] = {"executed_tflops": executed / (sp_ms / 1e3) / 1e12, "peak_tflops": tc_peak,
                            "frac": executed / (sp_ms / 1e3) / 1e12 / tc_peak,
                            "useful_tflops_fp32": useful / (sp_ms / 1e3) / 1e12,
                            "records": int(info[1]),
                            "note": ("executed = 3 fp16 products (hi*hi, hi*lo, lo*hi) x 2 x 128 grid points x "
                                     "records x T; peak = measured bf16 dense (fp16 runs at the bf16 rate)"
                                     if f16 else
                                     "executed = 3 tf32 products x 2 x 128 grid points x records x T; peak = "
                                     "measured bf16 dense / 2 (tf32 runs at half the bf16 rate)")}
    else:
        fp32_peak = 148 * 128 * 2 * 1.965e9 / 1e12
        spread["fp32"] = {"achieved_tflops": useful / (sp_ms / 1e3) / 1e12, "peak_tflops": fp32_peak,
                          "frac": useful / (sp_ms / 1e3) / 1e12 / fp32_peak}
    if nframes == 1:
        roof["spread"] = spread
    if dom == "ner":
        roof["note"] = ("the fused NER kernel moves only gh in and z out (16 B/voxel) and is bound by its "
                        "shared-memory FFTs and instruction issue (profiles/README.md), not by HBM")
    stage_report = {k: {"ms": per[k], "share": per[k] / sum(per.values()),
                        "GBps": sbytes[k] / (per[k] / 1e3) / 1e9 if per[k] > 0 else None} for k in per}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        os.environ.setdefault("PAT_THREADS", str(os.cpu_count() or 1))
        cfrac = args.cpu_frac or 0.25
        full, meas = cpu_sample_seconds(rec, cfrac)
        cpu = {"value": _voxels(rec) / full, "unit": UNIT, "cores": int(os.environ["PAT_THREADS"]),
               "kind": "port", "sample": _sample_desc(args.config, cfrac), "measured_s": meas}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32/c64", "data": "synthetic (seeded, BASELINE config shapes)",
        "config": _config_json(args, rec, world), "clocks": clk, "roofline": roof, "stages": stage_report,
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": own_launches * args.steps * nframes,
        "gpu_launches_note": f"own sm_100a kernels per step: {own_launches}; library (cuFFT) kernels per step: {lib_launches}",
    }
    emit(line)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def _traffic_from_profiles(cfg, kernel):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(cfg, {}).get(kernel)
    except Exception:
        return None


def _spawn_ranks(n):
    """``--gpus N`` without a launcher: re-run this command under torchrun, N local ranks."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    sys.stderr.flush()
    os.execv(sys.executable, cmd)


def main():
    if "WORLD_SIZE" not in os.environ:
        gi = [a for a in sys.argv[1:] if a.startswith("--gpus")]
        n = 1
        if gi:
            v = gi[0].split("=", 1)[1] if "=" in gi[0] else sys.argv[sys.argv.index(gi[0]) + 1]
            n = int(v)
        if n > 1:
            _spawn_ranks(n)
    _quiet_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-frac", type=float, default=None,
                    help="fraction of the workload the CPU sample runs (default: 1/4 for the cpu_baseline leg "
                         "(~10-15 s), 1/16 per step for --impl reference)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=240.0,
                    help="--impl reference: seconds of full reference runs (at least one run)")
    ap.add_argument("--sharded", action="store_true", help="use the sharded multi-GPU path even at N=1")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
