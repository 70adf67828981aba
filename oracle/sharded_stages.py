"""CPU (float64) model of the per-rank stages of the sharded GPU pipeline.

TEST INFRASTRUCTURE ONLY: it lets tests/test_sharded_gloo.py run
``paper_1501_02946_b200.parallel.ShardedNedNer`` -- partitioning, buffer
layouts and the two all-to-all exchanges -- on CPU ranks over gloo.  Each
stage produces exactly what the matching ``patfft_nedner_shard_*`` CUDA stage
produces (same layout, same sign conventions), computed with the oracle's
restatement of the reference (nedner_oracle.py):

* forward : (spread + lateral) NED of the time slice (nufft.py:400-418), Hermitian part on
            the lateral Nyquist planes (recon.py:218-222), half spectrum in
            j1, multiplied by (-1)^(j0+j1) (the GPU grids on a centred
            oversampled plane and skips the output fftshift -- the two signs
            cancel);
* ner     : (ner_rows) warped NER + amplitude/band (recon.py:274-308), scaled by
            1/(N0 N1 T) and inverse-FFT'd along depth;
* inverse : lateral inverse FFT (C2R along j1).
"""

from __future__ import annotations

import numpy as np

from . import nedner_oracle as O


class NumpyStages:
    def __init__(self, positions, weights, n_time, dt, sound_speed, dx, n_lateral, out_dims, spec, rank, world):
        positions = np.atleast_2d(np.asarray(positions, dtype=np.float64))
        self.n_lateral = tuple(int(n) for n in np.atleast_1d(n_lateral))
        if positions.shape[1] != len(self.n_lateral):
            positions = positions.T
        self.dims = tuple(out_dims)
        self.nlat = len(self.dims)
        self.scale = np.asarray(weights, dtype=np.float64).ravel() / dx ** self.nlat
        self.gpos = (positions / dx) * (np.asarray(self.dims, float) / np.asarray(self.n_lateral, float))
        self.spec = (spec.c, spec.K, spec.alpha, spec.beta)
        self.T = int(n_time)
        self.rank, self.world = rank, world
        self.Tr = self.T // world
        self.N0 = self.dims[0] if self.nlat == 2 else 1
        self.N1 = self.dims[-1]
        self.N1h = self.N1 // 2 + 1
        self.rows_total = self.N0 * self.N1h
        self.row_starts = [q * self.rows_total // world for q in range(world + 1)]
        ratios = O.lateral_ratios(self.T, dt, sound_speed, dx, self.n_lateral)
        jt1 = O.wrapped_freqs(self.N1, ratios[-1]) ** 2
        jt0 = O.wrapped_freqs(self.N0, ratios[0]) ** 2 if self.nlat == 2 else np.zeros(1)
        self.j2 = (jt0[:, None] + jt1[None, : self.N1h]).ravel()
        j0 = O.wrapped_freqs(self.N0) if self.nlat == 2 else np.zeros(1)
        j1 = O.wrapped_freqs(self.N1)[: self.N1h]
        self.sign = ((-1.0) ** (np.rint(j0[:, None] + j1[None, :]).astype(np.int64) % 2)).ravel()

    @staticmethod
    def _c(t, n=None):
        a = t.detach().cpu().numpy().view(np.complex64)
        return a if n is None else a[:n]

    @staticmethod
    def _put(t, arr):
        t.copy_(t.new_tensor(np.ascontiguousarray(arr, dtype=np.complex64).view(np.float32).ravel()))

    # pipelined stages (ShardedNedNer): spread keeps the slice's spectrum, lateral
    # hands out time pieces of it, ner_rows works on a block of the rank's rows
    def spread(self, samples_slice, stream=0):
        self._half = self._forward_half(samples_slice)

    def lateral(self, t_begin, t_end, gh_chunk, stream=0):
        self._put(gh_chunk, self._half[:, t_begin:t_end])

    def ner_rows(self, gh_recv, in_tchunk, row_begin, row_end, z_block, stream=0):
        rm = self.row_starts[self.rank + 1] - self.row_starts[self.rank]
        chunks = self._c(gh_recv).reshape(self.T // in_tchunk, rm, in_tchunk)
        rows = np.concatenate(list(chunks), axis=1)[row_begin:row_end]  # (rows, T), time chunk k = t // in_tchunk
        r0 = self.row_starts[self.rank] + row_begin
        fh = O.fhat_rows(rows.astype(np.complex128), self.j2[r0:r0 + row_end - row_begin], self.T, self.spec)
        z = np.fft.ifft(fh, axis=-1) * self.T / (self.N0 * self.N1 * self.T)
        self._put(z_block, np.stack([z[:, q * self.Tr:(q + 1) * self.Tr] for q in range(self.world)]))

    def forward(self, samples_slice, gh_send, stream=0):
        self._put(gh_send, self._forward_half(samples_slice))

    def _forward_half(self, samples_slice):
        s = samples_slice.detach().cpu().numpy().astype(np.float64) * self.scale[:, None]
        gh = O.NedOracle(self.dims, *self.spec).execute(self.gpos, s.astype(np.complex128), wrapped=True)
        b = gh
        for ax in range(self.nlat):  # Hermitian part in the lateral axes (recon.py:218-222)
            b = np.roll(np.flip(b, axis=ax), 1, axis=ax)
        sym = 0.5 * (gh + np.conj(b))
        if self.nlat == 1:
            sym = sym[None]
        return sym[:, : self.N1h, :].reshape(self.rows_total, self.Tr) * self.sign[:, None]

    def ner(self, gh_recv, z_send, stream=0):
        rm = self.row_starts[self.rank + 1] - self.row_starts[self.rank]
        blocks = self._c(gh_recv).reshape(self.world, rm, self.Tr)
        rows = np.concatenate(list(blocks), axis=1)  # (rm, T)
        r0 = self.row_starts[self.rank]
        fh = O.fhat_rows(rows.astype(np.complex128), self.j2[r0:r0 + rm], self.T, self.spec)
        z = np.fft.ifft(fh, axis=-1) * self.T / (self.N0 * self.N1 * self.T)
        out = np.stack([z[:, q * self.Tr:(q + 1) * self.Tr] for q in range(self.world)])
        self._put(z_send, out)

    def inverse(self, z_recv, image_slice, stream=0):
        z = self._c(z_recv).astype(np.complex128).reshape(self.N0, self.N1h, self.Tr)
        if self.nlat == 2:
            z = np.fft.ifft(z, axis=0) * self.N0
        img = np.fft.irfft(z, n=self.N1, axis=1) * self.N1
        if self.nlat == 1:
            img = img[0]
        image_slice.copy_(image_slice.new_tensor(img.astype(np.float32)))
        z_recv.fill_(float("nan"))  # the CUDA stage transforms its input in place: nothing of it may be reused


class NumpySliceStages(NumpyStages):
    """CPU model of the general schedule's stages (GpuSliceStages /
    patfft_nedner_slice_ner): same layouts and sign convention, any even N_t,
    any upsample (recon.py:225-246 row placement and Nyquist splits)."""

    def __init__(self, positions, weights, n_time, dt, sound_speed, dx, n_lateral, out_dims, upsample, spec, layout):
        super().__init__(positions, weights, n_time, dt, sound_speed, dx, n_lateral, out_dims, spec, 0, 1)
        self.L = layout
        self.up = int(upsample)

    def forward(self, samples_slice, gh_part, stream=0):
        s = samples_slice.detach().cpu().numpy().astype(np.float64) * self.scale[:, None]
        gh = O.NedOracle(self.dims, *self.spec).execute(self.gpos, s.astype(np.complex128), wrapped=True)
        b = gh
        for ax in range(self.nlat):
            b = np.roll(np.flip(b, axis=ax), 1, axis=ax)
        sym = 0.5 * (gh + np.conj(b))
        if self.nlat == 1:
            sym = sym[None]
        half = sym[:, : self.N1h, :].reshape(self.rows_total, s.shape[1]) * self.sign[:, None]
        gh_part.copy_(gh_part.new_tensor(np.ascontiguousarray(half, dtype=np.complex64).view(np.float32).reshape(
            self.rows_total, s.shape[1], 2)))

    def ner(self, gh_rows, row_begin, row_end, z_full, stream=0):
        L, up = self.L, self.up
        rows = gh_rows.detach().cpu().numpy().reshape(row_end - row_begin, self.T * 2).view(np.complex64)
        fh = O.fhat_rows(rows.astype(np.complex128), self.j2[row_begin:row_end], self.T, self.spec)
        if up > 1:
            fh = O.zero_pad_axis(fh, 1, up)
        z = np.fft.ifft(fh, axis=-1) * (self.T * up) / (self.N0 * self.N1 * self.T)
        zf = z_full.detach().cpu().numpy().reshape(L.rows_out_total, L.Tu * 2).view(np.complex64).copy()
        for i, r in enumerate(range(row_begin, row_end)):
            j0w, j1 = divmod(r, self.N1h)
            f = 0.5 if (up > 1 and j1 == self.N1 // 2) else 1.0
            if self.nlat != 2:
                dst = [0]
            elif up == 1:
                dst = [j0w]
            else:
                a = j0w if j0w < self.N0 // 2 else j0w - self.N0
                if a == -(self.N0 // 2):
                    dst, f = [self.N0 // 2, L.N0u - self.N0 // 2], 0.5 * f
                else:
                    dst = [a if a >= 0 else L.N0u + a]
            for j in dst:
                zf[j * L.N1uh + j1] = f * z[i]
        z_full.copy_(z_full.new_tensor(zf.view(np.float32).reshape(L.rows_out_total, L.Tu, 2)))

    def inverse(self, z_slice, image_slice, stream=0):
        L = self.L
        tur = z_slice.shape[1]
        z = z_slice.detach().cpu().numpy().reshape(L.rows_out_total, tur * 2).view(np.complex64).astype(np.complex128)
        z = z.reshape(L.N0u, L.N1uh, tur)
        if self.nlat == 2:
            z = np.fft.ifft(z, axis=0) * L.N0u
        img = np.fft.irfft(z, n=L.N1u, axis=1) * L.N1u
        if self.nlat == 1:
            img = img[0]
        image_slice.copy_(image_slice.new_tensor(img.astype(np.float32)))
        z_slice.fill_(float("nan"))  # consumed in place by the CUDA stage
