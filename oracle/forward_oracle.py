"""CPU oracle of the forward model -- TEST INFRASTRUCTURE ONLY.

numpy/scipy float64 restatement of ``patfft.forward.forward_fourier``
(/root/reference/pkg/src/patfft/forward.py:105-172).  Only ``tests/`` may
import it (the product path is ``paper_1501_02946_b200.forward``).  Pinned
by ``tests/test_oracle.py`` against the ``forward_*.npz`` goldens that
``tests/golden/make_golden.py`` produced with the reference itself.
"""

from __future__ import annotations

import numpy as np
import scipy.fft as sfft

from .nedner_oracle import NerOracle, _threads, lateral_freq_sq


def forward_fourier(values, spacing, sound_speed, c=2.0, K=6, alpha=None, beta=None):
    """Returns (traces (rows, N_t), positions (rows, d-1), weights (rows,), dt)."""
    vals = np.asarray(values, dtype=np.float64)
    if sound_speed <= 0:                                                     # forward.py:112-113
        raise ValueError("sound speed must be positive")
    if vals.ndim not in (2, 3):                                              # forward.py:115-116
        raise ValueError("forward operator supports 2D and 3D fields")
    n_lateral = vals.shape[:-1]
    nt = vals.shape[-1]
    if nt % 2 or any(n % 2 for n in n_lateral):                              # forward.py:118-119
        raise ValueError("grid sizes must be even")
    lat_axes = tuple(range(vals.ndim - 1))
    fh = sfft.fftn(np.fft.ifftshift(vals, axes=lat_axes).astype(np.complex128), axes=lat_axes,
                   workers=_threads())                                       # forward.py:124
    nt2 = 2 * nt                                                             # forward.py:136-137
    wvals = sfft.fftfreq(nt2) * nt2 / 2.0
    depth_extent = nt * spacing[-1]                                          # forward.py:138-140
    ratios = tuple(depth_extent / (n * spacing[ax]) for ax, n in enumerate(n_lateral))
    j2 = lateral_freq_sq(n_lateral, ratios)                                  # forward.py:141
    w2 = wvals ** 2                                                          # forward.py:142-147
    prop = j2[..., None] < w2
    ky = np.where(prop, np.sign(wvals) * np.sqrt(np.maximum(w2 - j2[..., None], 0.0)), 0.0)
    scale = np.zeros(ky.shape)
    np.divide(wvals * np.ones_like(j2)[..., None], 2.0 * ky, out=scale, where=ky != 0)
    rows = int(np.prod(n_lateral))                                           # forward.py:149-153
    plan = NerOracle(nt, c, K, alpha, beta)
    fb = fh.reshape(rows, nt)
    kb = ky.reshape(rows, nt2)
    ghat = (plan.rows(fb, kb) + plan.rows(fb, -kb)).reshape(ky.shape)
    ghat *= scale * prop
    traces = sfft.ifft(ghat, axis=-1, workers=_threads())[..., :nt]         # forward.py:155-157
    traces = sfft.ifftn(traces, axes=lat_axes, workers=_threads())
    traces = np.fft.fftshift(traces, axes=lat_axes).real
    dx = spacing[0]                                                          # forward.py:159-161
    axes = [(np.arange(n) - n // 2) * dx for n in n_lateral]                # forward.py:169-172
    mesh = np.meshgrid(*axes, indexing="ij")
    positions = np.stack([m.ravel() for m in mesh], axis=-1)
    weights = np.full(rows, dx ** len(n_lateral))
    return traces.reshape(rows, nt), positions, weights, spacing[-1] / sound_speed
