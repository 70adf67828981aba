"""Multi-GPU NEDNER: one reconstruction split over torch.distributed ranks.

One process per GPU.  The reference has no distributed code; this follows
the decomposition BASELINE.json's north star asks for:

1. NED + lateral FFT sharded by *time sample* -- the spreading operator is
   the same for every time sample, so each rank grids its own time slice
   with a replicated plan (no communication);
2. all-to-all #1 (NCCL over NVLink/NVSwitch): time slices -> lateral
   frequency row ownership;
3. NER + depth inverse FFT on the rank's rows (row-local);
4. all-to-all #2: row ownership -> time (depth) slices;
5. lateral inverse FFT of the rank's depth slice -> image slice.

The per-rank stages run on the GPU through the C ABI
(``patfft_nedner_shard_*``); the exchanges are ``all_to_all_single`` on the
current CUDA stream, so kernels and collectives are ordered without host
synchronisation.  Buffers are float32 tensors (complex values as pairs).

The stage backend is pluggable only so the orchestration (partitioning,
layouts, exchanges) can be exercised on CPU with gloo in the tests; the
product backend is ``GpuStages`` and there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .recon import _out_dims
from .window import WindowSpec


class ShardLayout:
    """Sizes shared by every rank of a sharded reconstruction."""

    def __init__(self, n_lat, out_dims, n_time, world):
        self.n_lat = n_lat
        self.N0 = out_dims[0] if n_lat == 2 else 1
        self.N1 = out_dims[-1]
        self.N1h = self.N1 // 2 + 1
        self.T = n_time
        self.world = world
        self.Tr = n_time // world
        self.rows_total = self.N0 * self.N1h
        self.row_starts = [q * self.rows_total // world for q in range(world + 1)]

    def rows(self, q):
        return self.row_starts[q + 1] - self.row_starts[q]

    def image_slice_shape(self):
        return ((self.N0, self.N1) if self.n_lat == 2 else (self.N1,)) + (self.Tr,)

    @staticmethod
    def supported(n_time, world, upsample=1):
        tr = n_time // world if world else 0
        return upsample == 1 and world >= 1 and n_time % world == 0 and tr >= 2 and (tr & (tr - 1)) == 0


class GpuStages:
    """Per-rank stages on the B200 (sharded C plan)."""

    def __init__(self, positions, weights, n_time, dt, sound_speed, dx, n_lateral, out_dims, spec, rank, world,
                 device):
        lib = _lib.load()
        positions = np.atleast_2d(np.asarray(positions, dtype=np.float64))
        n_lateral = tuple(int(n) for n in np.atleast_1d(n_lateral))
        if positions.shape[1] != len(n_lateral):
            positions = positions.T
        weights = np.asarray(weights, dtype=np.float64).ravel()
        nlat = len(out_dims)
        scale = np.ascontiguousarray(weights / dx ** nlat)
        gpos = np.ascontiguousarray((positions / dx) * (np.asarray(out_dims, float) / np.asarray(n_lateral, float)))
        dy = sound_speed * dt
        desc = _lib.NednerDesc()
        desc.n_lat = nlat
        desc.out_dims[0] = out_dims[0]
        desc.out_dims[1] = out_dims[-1] if nlat == 2 else 0
        desc.n_time = int(n_time)
        desc.upsample = 1
        desc.n_sensors = positions.shape[0]
        ratios = [n_time * dy / (n * dx) for n in n_lateral]
        desc.lat_ratio[0] = ratios[0]
        desc.lat_ratio[1] = ratios[-1]
        desc.spec_c = float(spec.c)
        desc.spec_K = int(spec.K)
        desc.spec_alpha = math.nan if spec.alpha is None else float(spec.alpha)
        desc.spec_beta = math.nan if spec.beta is None else float(spec.beta)
        h = ctypes.c_void_p()
        _lib.check(lib.patfft_nedner_plan_create_sharded(
            ctypes.byref(desc), gpos.ctypes.data_as(_lib._D), scale.ctypes.data_as(_lib._D), int(device), int(rank),
            int(world), ctypes.byref(h)))
        self._lib = lib
        self._h = h

    @staticmethod
    def _stream(stream):
        return ctypes.c_void_p(stream or 0)

    def forward(self, samples_slice, gh_send, stream=0):
        _lib.check(self._lib.patfft_nedner_shard_forward(self._h, ctypes.c_void_p(samples_slice.data_ptr()),
                                                         ctypes.c_void_p(gh_send.data_ptr()), self._stream(stream)))

    def ner(self, gh_recv, z_send, stream=0):
        _lib.check(self._lib.patfft_nedner_shard_ner(self._h, ctypes.c_void_p(gh_recv.data_ptr()),
                                                     ctypes.c_void_p(z_send.data_ptr()), self._stream(stream)))

    def inverse(self, z_recv, image_slice, stream=0):
        _lib.check(self._lib.patfft_nedner_shard_inverse(self._h, ctypes.c_void_p(z_recv.data_ptr()),
                                                         ctypes.c_void_p(image_slice.data_ptr()), self._stream(stream)))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.patfft_nedner_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedNedNer:
    """Reconstruct one record across all ranks of a torch.distributed group.

    Every rank builds the plan from the same sensor layout; ``run`` takes the
    rank's time slice ``samples[:, rank*Tr:(rank+1)*Tr]`` (a device tensor,
    float32) and returns the rank's depth slice of the image
    ``image[..., rank*Tr:(rank+1)*Tr]``.
    """

    def __init__(self, positions, weights, n_time, dt, sound_speed, dx, n_lateral, out_dims=None,
                 spec: WindowSpec | None = None, group=None, device=None, stages=None, torch_device=None):
        import torch
        import torch.distributed as dist

        self.torch = torch
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        n_lateral = tuple(int(n) for n in np.atleast_1d(n_lateral))
        dims = _out_dims(n_lateral, out_dims)
        spec = spec if spec is not None else WindowSpec()
        if not ShardLayout.supported(n_time, self.world):
            raise ValueError("sharded NEDNER needs N_t / world to be a power of two")
        self.layout = L = ShardLayout(len(dims), dims, int(n_time), self.world)
        if torch_device is None:
            torch_device = torch.device("cuda", torch.cuda.current_device()) if device is None else \
                torch.device("cuda", device)
        self.tdev = torch_device
        if stages is None:
            stages = GpuStages(positions, weights, n_time, dt, sound_speed, dx, n_lateral, dims, spec, self.rank,
                               self.world, torch_device.index)
        self.stages = stages
        f32 = dict(dtype=torch.float32, device=torch_device)
        rm = L.rows(self.rank)
        self.gh_send = torch.empty(L.rows_total * L.Tr * 2, **f32)
        self.gh_recv = torch.empty(self.world * rm * L.Tr * 2, **f32)
        self.z_send = torch.empty(self.world * rm * L.Tr * 2, **f32)
        self.z_recv = torch.empty(L.rows_total * L.Tr * 2, **f32)
        self.image = torch.empty(L.image_slice_shape(), **f32)
        self.send1 = [L.rows(q) * L.Tr * 2 for q in range(self.world)]
        self.recv1 = [rm * L.Tr * 2] * self.world
        self.send2 = self.recv1
        self.recv2 = self.send1
        # A dedicated (non-default) stream: the C stages treat a NULL stream as
        # "the plan's own stream", which would not be ordered with torch's
        # legacy default stream.
        self.cuda_stream = torch.cuda.Stream(device=torch_device) if torch_device.type == "cuda" else None

    def run(self, samples_slice):
        """Enqueue one sharded reconstruction; returns this rank's image slice.

        Work is ordered after everything already queued on the caller's current
        stream and the caller's stream waits for the result.
        """
        if self.cuda_stream is None:
            return self._run(samples_slice, 0)
        torch = self.torch
        cur = torch.cuda.current_stream(self.tdev)
        self.cuda_stream.wait_stream(cur)
        with torch.cuda.stream(self.cuda_stream):
            out = self._run(samples_slice, self.cuda_stream.cuda_stream)
        cur.wait_stream(self.cuda_stream)
        return out

    def _run(self, samples_slice, s):
        self.stages.forward(samples_slice, self.gh_send, s)
        self.dist.all_to_all_single(self.gh_recv, self.gh_send, output_split_sizes=self.recv1,
                                    input_split_sizes=self.send1, group=self.group)
        self.stages.ner(self.gh_recv, self.z_send, s)
        self.dist.all_to_all_single(self.z_recv, self.z_send, output_split_sizes=self.recv2,
                                    input_split_sizes=self.send2, group=self.group)
        self.stages.inverse(self.z_recv, self.image, s)
        return self.image
