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

    def spread(self, samples_slice, stream=0):
        _lib.check(self._lib.patfft_nedner_shard_spread(self._h, ctypes.c_void_p(samples_slice.data_ptr()),
                                                        self._stream(stream)))

    def lateral(self, t_begin, t_end, gh_chunk, stream=0):
        _lib.check(self._lib.patfft_nedner_shard_lateral(self._h, int(t_begin), int(t_end),
                                                         ctypes.c_void_p(gh_chunk.data_ptr()), self._stream(stream)))

    def ner_rows(self, gh_recv, in_tchunk, row_begin, row_end, z_block, stream=0):
        _lib.check(self._lib.patfft_nedner_shard_ner_rows(self._h, ctypes.c_void_p(gh_recv.data_ptr()), int(in_tchunk),
                                                          int(row_begin), int(row_end),
                                                          ctypes.c_void_p(z_block.data_ptr()), self._stream(stream)))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.patfft_nedner_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _host_staged(dist, group, tensor):
    """CUDA tensors over a backend without device point-to-point (gloo): stage through the host.
    NCCL, the product path, sends and receives the device buffers directly."""
    return tensor.is_cuda and dist.get_backend(group) != "nccl"


def _host_exchange(dist, group, rank, pairs):
    """pairs[q] = (send view to rank q, recv view from rank q); synchronous, returns no work handles."""
    sends = {q: sv.cpu() for q, (sv, _) in enumerate(pairs) if q != rank}
    recvs = {q: rv.new_empty(rv.shape, device="cpu") for q, (_, rv) in enumerate(pairs) if q != rank}
    ops = []
    for q in sends:
        ops.append(dist.P2POp(dist.isend, sends[q], q, group=group))
        ops.append(dist.P2POp(dist.irecv, recvs[q], q, group=group))
    for w in (dist.batch_isend_irecv(ops) if ops else []):
        w.wait()
    for q, (_, rv) in enumerate(pairs):
        if q != rank:
            rv.copy_(recvs[q])
    return []


def _pow2_at_most(n, cap):
    c = 1
    while c * 2 <= min(n, cap):
        c *= 2
    return c


class ShardedNedNer:
    """Reconstruct one record across all ranks of a torch.distributed group.

    Every rank builds the plan from the same sensor layout; ``run`` takes the
    rank's time slice ``samples[:, rank*Tr:(rank+1)*Tr]`` (a device tensor,
    float32) and returns the rank's depth slice of the image
    ``image[..., rank*Tr:(rank+1)*Tr]``.  The returned tensor is this object's
    output buffer and is overwritten by the next ``run`` (pass ``out=`` to
    keep results apart).

    Schedule per rank (each exchange overlaps the compute that follows it):

    1. spread the whole slice (one gridding launch: the tensor-core kernel
       wants long time blocks);
    2. lateral FFTs in ``time_chunks`` pieces of Tr / C samples; the
       exchange of piece c (rows of every destination, one grouped NCCL
       send/recv) runs while piece c + 1 is transformed;
    3. NER in ``row_blocks`` blocks of the rank's rows; the exchange of block
       b (its depth slices back to their owners) runs while block b + 1 is
       interpolated;
    4. lateral inverse of the rank's depth slice.

    Receive buffers are laid out so that nothing is repacked: piece c from
    rank q lands as time chunk q*C + c of ``[chunk][rows_mine][Tr/C]``, which
    the NER kernel reads directly, and block b of rank q lands at its global
    rows of ``[rows_total][Tr]``, which the inverse reads directly.  At world
    size 1 there is no exchange and the buffers alias (the single-GPU
    pipeline with three launches).
    """

    def __init__(self, positions, weights, n_time, dt, sound_speed, dx, n_lateral, out_dims=None,
                 spec: WindowSpec | None = None, group=None, device=None, stages=None, torch_device=None,
                 time_chunks=None, row_blocks=None):
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
        P = self.world
        # pieces of Tr / C >= 32 samples (lateral kernels' time tile); none at world 1
        self.C = C = (1 if P == 1 else _pow2_at_most(max(1, L.Tr // 32), 4)) if time_chunks is None else int(time_chunks)
        if C < 1 or L.Tr % C or (C > 1 and (L.Tr // C) % 32) or (L.Tr // C) & (L.Tr // C - 1):
            raise ValueError("time_chunks must split N_t / world into power-of-two pieces of >= 32 samples")
        self.Trc = Trc = L.Tr // C
        self.B = B = (1 if P == 1 else 4) if row_blocks is None else int(row_blocks)
        f32 = dict(dtype=torch.float32, device=torch_device)
        rm = L.rows(self.rank)
        self.rm = rm
        # a block partition every rank computes the same way for every rank's rows
        self.bounds = [[b * L.rows(q) // B for b in range(B + 1)] for q in range(P)]
        if min(self.bounds[self.rank][b + 1] - self.bounds[self.rank][b] for b in range(B)) < 1:
            raise ValueError("more row blocks than rows on a rank")
        self.gh_send = torch.empty(C * L.rows_total * Trc * 2, **f32)       # [c][rows_total][Trc]
        self.gh_recv = self.gh_send if P == 1 else torch.empty(P * C * rm * Trc * 2, **f32)  # [q*C+c][rm][Trc]
        self.z_send = torch.empty(P * rm * L.Tr * 2, **f32)                 # per block b: [q][rows_b][Tr]
        self.z_recv = self.z_send if (P == 1 and B == 1) else torch.empty(L.rows_total * L.Tr * 2, **f32)
        self.image = torch.empty(L.image_slice_shape(), **f32)
        # A dedicated (non-default) stream: the C stages treat a NULL stream as
        # "the plan's own stream", which would not be ordered with torch's
        # legacy default stream.
        self.cuda_stream = torch.cuda.Stream(device=torch_device) if torch_device.type == "cuda" else None

    # ---- buffer views ----------------------------------------------------
    def _gh_send_chunk(self, c):
        n = self.layout.rows_total * self.Trc * 2
        return self.gh_send[c * n:(c + 1) * n]

    def _gh_send_rows(self, c, q):
        L, w = self.layout, self.Trc * 2
        return self._gh_send_chunk(c)[L.row_starts[q] * w:L.row_starts[q + 1] * w]

    def _gh_recv_piece(self, q, c):
        n = self.rm * self.Trc * 2
        k = q * self.C + c
        return self.gh_recv[k * n:(k + 1) * n]

    def _z_block(self, b):
        L = self.layout
        b0 = self.bounds[self.rank][b]
        return self.z_send[self.world * b0 * L.Tr * 2:self.world * self.bounds[self.rank][b + 1] * L.Tr * 2]

    def _z_block_dst(self, b, q):
        L = self.layout
        nb = self.bounds[self.rank][b + 1] - self.bounds[self.rank][b]
        return self._z_block(b)[q * nb * L.Tr * 2:(q + 1) * nb * L.Tr * 2]

    def _z_recv_rows(self, b, q):
        L = self.layout
        r0 = L.row_starts[q] + self.bounds[q][b]
        r1 = L.row_starts[q] + self.bounds[q][b + 1]
        return self.z_recv[r0 * L.Tr * 2:r1 * L.Tr * 2]

    def _exchange(self, pairs):
        """One grouped exchange: pairs[q] = (send view to rank q, recv view from rank q)."""
        dist = self.dist
        snd, rcv = pairs[self.rank]
        rcv.copy_(snd)  # own share: a device copy on the compute stream
        if _host_staged(dist, self.group, snd):
            return _host_exchange(dist, self.group, self.rank, pairs)
        ops = []
        for q, (sv, rv) in enumerate(pairs):
            if q == self.rank:
                continue
            ops.append(dist.P2POp(dist.isend, sv, q, group=self.group))
            ops.append(dist.P2POp(dist.irecv, rv, q, group=self.group))
        return dist.batch_isend_irecv(ops) if ops else []

    # ---- one reconstruction ----------------------------------------------
    def run(self, samples_slice, out=None):
        """Enqueue one sharded reconstruction; returns this rank's image slice.

        Work is ordered after everything already queued on the caller's current
        stream and the caller's stream waits for the result.
        """
        if self.cuda_stream is None:
            img = self._run(samples_slice, 0)
        else:
            torch = self.torch
            cur = torch.cuda.current_stream(self.tdev)
            self.cuda_stream.wait_stream(cur)
            with torch.cuda.stream(self.cuda_stream):
                img = self._run(samples_slice, self.cuda_stream.cuda_stream)
            cur.wait_stream(self.cuda_stream)
        if out is not None:
            out.copy_(img)
            return out
        return img

    def _run(self, samples_slice, s):
        L, P, C, B = self.layout, self.world, self.C, self.B
        st = self.stages
        st.spread(samples_slice, s)
        works = []
        for c in range(C):
            st.lateral(c * self.Trc, (c + 1) * self.Trc, self._gh_send_chunk(c), s)
            if P > 1:  # piece c to every row owner while piece c + 1 is transformed
                works += self._exchange([(self._gh_send_rows(c, q), self._gh_recv_piece(q, c)) for q in range(P)])
        for w in works:
            w.wait()
        works = []
        for b in range(B):
            b0, b1 = self.bounds[self.rank][b], self.bounds[self.rank][b + 1]
            st.ner_rows(self.gh_recv, self.Trc, b0, b1, self._z_block(b), s)
            if self.z_recv is not self.z_send:  # block b back to the depth owners while b + 1 runs
                works += self._exchange([(self._z_block_dst(b, q), self._z_recv_rows(b, q)) for q in range(P)])
        for w in works:
            w.wait()
        st.inverse(self.z_recv, self.image, s)
        return self.image


# ---------------------------------------------------------------------------
# General schedule: any even N_t, any upsample, any lateral size of the plan
# ---------------------------------------------------------------------------

class SliceLayout:
    """Partition of the general schedule: time (and depth) ranges with even
    boundaries -- the lateral kernels pack two time samples per transform --
    and the lateral rows of the half spectrum, split as evenly as possible.
    ``out_rows(q)``: the rows of the (upsampled) half spectrum ``z`` that rank
    q's NER writes (recon.py:225-246: a lateral Nyquist row lands twice)."""

    def __init__(self, n_lat, out_dims, n_time, world, upsample=1):
        if n_time % 2 or n_time // 2 < world:
            raise ValueError("general sharding needs an even N_t with at least 2 samples per rank")
        self.n_lat, self.world, self.up, self.T = n_lat, world, int(upsample), int(n_time)
        self.N0 = out_dims[0] if n_lat == 2 else 1
        self.N1 = out_dims[-1]
        self.N1h = self.N1 // 2 + 1
        self.N0u = self.N0 * self.up if n_lat == 2 else 1
        self.N1u = self.N1 * self.up
        self.N1uh = self.N1u // 2 + 1
        self.Tu = self.T * self.up
        self.rows_total = self.N0 * self.N1h
        self.rows_out_total = self.N0u * self.N1uh
        self.t_starts = [2 * ((q * (self.T // 2)) // world) for q in range(world + 1)]
        self.row_starts = [q * self.rows_total // world for q in range(world + 1)]

    def t_range(self, q):
        return self.t_starts[q], self.t_starts[q + 1]

    def tu_range(self, q):
        return self.up * self.t_starts[q], self.up * self.t_starts[q + 1]

    def t_slice_max(self):
        return max(self.t_starts[q + 1] - self.t_starts[q] for q in range(self.world))

    def out_rows(self, q):
        rows = []
        for r in range(self.row_starts[q], self.row_starts[q + 1]):
            j0w, j1 = divmod(r, self.N1h)
            if self.n_lat != 2:
                j0u = [0]
            elif self.up == 1:
                j0u = [j0w]
            else:
                a = j0w if j0w < self.N0 // 2 else j0w - self.N0
                j0u = [self.N0 // 2, self.N0u - self.N0 // 2] if a == -(self.N0 // 2) else [a if a >= 0 else self.N0u + a]
            rows += [j * self.N1uh + j1 for j in j0u]
        return rows

    def image_slice_shape(self, q):
        a, b = self.tu_range(q)
        return ((self.N0u, self.N1u) if self.n_lat == 2 else (self.N1u,)) + (b - a,)


class GpuSliceStages:
    """Per-rank stages of the general schedule on the B200 (sliced C plan)."""

    def __init__(self, positions, weights, n_time, dt, sound_speed, dx, n_lateral, out_dims, upsample, spec, t_slice,
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
        desc.upsample = int(upsample)
        desc.n_sensors = positions.shape[0]
        ratios = [n_time * dy / (n * dx) for n in n_lateral]
        desc.lat_ratio[0] = ratios[0]
        desc.lat_ratio[1] = ratios[-1]
        desc.spec_c = float(spec.c)
        desc.spec_K = int(spec.K)
        desc.spec_alpha = math.nan if spec.alpha is None else float(spec.alpha)
        desc.spec_beta = math.nan if spec.beta is None else float(spec.beta)
        h = ctypes.c_void_p()
        _lib.check(lib.patfft_nedner_plan_create_slice(
            ctypes.byref(desc), gpos.ctypes.data_as(_lib._D), scale.ctypes.data_as(_lib._D), int(device), int(t_slice),
            ctypes.byref(h)))
        self._lib = lib
        self._h = h

    def forward(self, samples_slice, gh_part, stream=0):
        _lib.check(self._lib.patfft_nedner_shard_forward(self._h, ctypes.c_void_p(samples_slice.data_ptr()),
                                                         ctypes.c_void_p(gh_part.data_ptr()), ctypes.c_void_p(stream or 0)))

    def ner(self, gh_rows, row_begin, row_end, z_full, stream=0):
        _lib.check(self._lib.patfft_nedner_slice_ner(self._h, ctypes.c_void_p(gh_rows.data_ptr()), int(row_begin),
                                                     int(row_end), ctypes.c_void_p(z_full.data_ptr()),
                                                     ctypes.c_void_p(stream or 0)))

    def inverse(self, z_slice, image_slice, stream=0):
        _lib.check(self._lib.patfft_nedner_shard_inverse(self._h, ctypes.c_void_p(z_slice.data_ptr()),
                                                         ctypes.c_void_p(image_slice.data_ptr()),
                                                         ctypes.c_void_p(stream or 0)))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.patfft_nedner_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GeneralShardedNedNer:
    """One reconstruction across the ranks of a torch.distributed group, for
    every case the reference handles on one process: any even N_t (uneven
    time slices with even boundaries), any ``upsample`` (recon.py:392-394),
    any lateral size.  ``ShardedNedNer`` is the pipelined fast path for
    power-of-two N_t / world and upsample 1; this class trades its in-place
    receive layouts for plain packing copies:

    1. NED + lateral FFT of the rank's time slice (no communication);
    2. rows of every slice to their owner (grouped send/recv), assembled
       into ``[rows_mine][N_t]``;
    3. NER + depth inverse of the owned rows into their rows of the
       (upsampled, zero-padded) half spectrum;
    4. depth slices of those rows to their owners, scattered into
       ``[N0u * N1uh][upsample * slice]`` (rows nobody owns stay zero);
    5. lateral inverse of the rank's depth slice.

    ``run`` takes ``samples[:, t0:t1]`` of the rank's ``layout.t_range(rank)``
    and returns ``image[..., up*t0:up*t1]`` (a buffer reused by the next call
    unless ``out=`` is given).
    """

    def __init__(self, positions, weights, n_time, dt, sound_speed, dx, n_lateral, out_dims=None, upsample=1,
                 spec: WindowSpec | None = None, group=None, device=None, stages=None, torch_device=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        n_lateral = tuple(int(n) for n in np.atleast_1d(n_lateral))
        dims = _out_dims(n_lateral, out_dims)
        if int(upsample) != upsample or upsample < 1:
            raise ValueError("upsample must be a positive integer")
        spec = spec if spec is not None else WindowSpec()
        self.layout = L = SliceLayout(len(dims), dims, int(n_time), self.world, int(upsample))
        if torch_device is None:
            torch_device = torch.device("cuda", torch.cuda.current_device()) if device is None else \
                torch.device("cuda", device)
        self.tdev = torch_device
        t0, t1 = L.t_range(self.rank)
        if stages is None:
            stages = GpuSliceStages(positions, weights, n_time, dt, sound_speed, dx, n_lateral, dims, int(upsample),
                                    spec, t1 - t0, torch_device.index)
        self.stages = stages
        f32 = dict(dtype=torch.float32, device=torch_device)
        P, rm = self.world, L.row_starts[self.rank + 1] - L.row_starts[self.rank]
        self.rm = rm
        self.gh_part = torch.empty(L.rows_total, t1 - t0, 2, **f32)
        self.gh_rows = torch.empty(rm, L.T, 2, **f32)
        self.z_full = torch.zeros(L.rows_out_total, L.Tu, 2, **f32)   # rows of other ranks stay zero
        u0, u1 = L.tu_range(self.rank)
        self.z_slice = torch.zeros(L.rows_out_total, u1 - u0, 2, **f32)  # zero-padding rows: re-zeroed per run
        self.image = torch.empty(L.image_slice_shape(self.rank), **f32)
        self.out_idx = [torch.tensor(L.out_rows(q), dtype=torch.long, device=torch_device) for q in range(P)]
        self.cuda_stream = torch.cuda.Stream(device=torch_device) if torch_device.type == "cuda" else None

    def _exchange(self, sends, recvs):
        dist = self.dist
        recvs[self.rank].copy_(sends[self.rank])
        if _host_staged(dist, self.group, sends[self.rank]):
            _host_exchange(dist, self.group, self.rank, list(zip(sends, recvs)))
            return
        ops = []
        for q in range(self.world):
            if q != self.rank:
                ops.append(dist.P2POp(dist.isend, sends[q], q, group=self.group))
                ops.append(dist.P2POp(dist.irecv, recvs[q], q, group=self.group))
        for w in (dist.batch_isend_irecv(ops) if ops else []):
            w.wait()

    def run(self, samples_slice, out=None):
        if self.cuda_stream is None:
            img = self._run(samples_slice, 0)
        else:
            torch = self.torch
            cur = torch.cuda.current_stream(self.tdev)
            self.cuda_stream.wait_stream(cur)
            with torch.cuda.stream(self.cuda_stream):
                img = self._run(samples_slice, self.cuda_stream.cuda_stream)
            cur.wait_stream(self.cuda_stream)
        if out is not None:
            out.copy_(img)
            return out
        return img

    def _run(self, samples_slice, s):
        torch, L, P, me = self.torch, self.layout, self.world, self.rank
        st = self.stages
        st.forward(samples_slice, self.gh_part, s)
        # rows of my time slice -> their owners; theirs -> columns [t0, t1) of my rows
        sends = [self.gh_part[L.row_starts[q]:L.row_starts[q + 1]] for q in range(P)]   # contiguous row blocks
        recvs = [torch.empty(self.rm, L.t_starts[q + 1] - L.t_starts[q], 2, dtype=torch.float32, device=self.tdev)
                 for q in range(P)]
        self._exchange(sends, recvs)
        for q in range(P):
            self.gh_rows[:, L.t_starts[q]:L.t_starts[q + 1]] = recvs[q]
        st.ner(self.gh_rows, L.row_starts[me], L.row_starts[me + 1], self.z_full, s)
        # depth slices of my output rows -> their owners, scattered into z_slice at their rows
        mine = self.z_full.index_select(0, self.out_idx[me])
        sends = [mine[:, L.up * L.t_starts[q]:L.up * L.t_starts[q + 1]].contiguous() for q in range(P)]
        u0, u1 = L.tu_range(me)
        recvs = [torch.empty(len(self.out_idx[q]), u1 - u0, 2, dtype=torch.float32, device=self.tdev) for q in range(P)]
        self._exchange(sends, recvs)
        if L.up > 1:  # the lateral inverse works in place: the zero-padding rows must be zero again
            self.z_slice.zero_()
        for q in range(P):
            self.z_slice.index_copy_(0, self.out_idx[q], recvs[q])
        st.inverse(self.z_slice, self.image, s)
        return self.image


def sharded_nedner(positions, weights, n_time, dt, sound_speed, dx, n_lateral, out_dims=None, upsample=1, spec=None,
                   **kw):
    """The fastest multi-GPU schedule that covers the request: ``ShardedNedNer``
    (pipelined, in-place layouts) for upsample 1, power-of-two N_t / world and
    lateral / depth grids, else ``GeneralShardedNedNer``."""
    import torch.distributed as dist

    n_lateral_t = tuple(int(n) for n in np.atleast_1d(n_lateral))
    dims = _out_dims(n_lateral_t, out_dims)
    world = dist.get_world_size(kw.get("group"))
    pow2 = all(n & (n - 1) == 0 for n in dims) and n_time & (n_time - 1) == 0
    if upsample == 1 and pow2 and ShardLayout.supported(n_time, world) and n_time // world >= 32:
        return ShardedNedNer(positions, weights, n_time, dt, sound_speed, dx, n_lateral, out_dims=out_dims, spec=spec,
                             **kw)
    return GeneralShardedNedNer(positions, weights, n_time, dt, sound_speed, dx, n_lateral, out_dims=out_dims,
                                upsample=upsample, spec=spec, **kw)
