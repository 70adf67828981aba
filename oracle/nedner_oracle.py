"""CPU oracle for the NEDNER-NUFFT reconstruction -- TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference algorithm
(``patfft.recon.reconstruct_nedner`` and the NUFFT plans it uses).  It is
the *checker*: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product path (``paper_1501_02946_b200``) never imports or calls it and
fails loudly when its CUDA library is missing.

Parity pin: ``tests/test_oracle.py`` checks every function here against the
golden vectors in ``tests/golden/`` that ``tests/golden/make_golden.py``
produced by running the *reference itself* (imported from
``/root/reference/pkg/src``) in the build container.

Each function names the reference lines (``/root/reference/pkg/src/patfft``)
whose behaviour it restates.  The computation is float64/complex128
throughout, exactly like the reference.
"""

from __future__ import annotations

import math
import os

import numpy as np
import scipy.fft as sfft
import scipy.sparse as sps
from scipy.special import i0

# nufft.py:59-61 -- fraction of the admissible support bound pi*(2c-1)
ALPHA_FRACTION = 0.999
# recon.py:48
WEIGHT_SUM_RTOL = 1e-6


def _threads() -> int:
    """FFT worker count (the reference reads PAT_THREADS, nufft.py:64-68)."""
    try:
        return max(1, int(os.environ.get("PAT_THREADS", "1")))
    except ValueError:
        return 1


# ---------------------------------------------------------------------------
# window pair and sizing (nufft.py:83-187)
# ---------------------------------------------------------------------------

def even_fast_len(target: float) -> int:
    """Smallest even scipy-fast length >= target (nufft.py:83-89)."""
    n = sfft.next_fast_len(max(int(math.ceil(target)), 2))
    while n % 2:
        n = sfft.next_fast_len(n + 1)
    return n


def resolve_window(c: float, K: int, alpha, beta, c_eff: float):
    """Concrete (alpha, beta) for an effective oversampling (nufft.py:133-149).

    Returns the tuple (c_eff, K, alpha, beta).  Raises ValueError when the
    support is inadmissible (the reference raises ParameterError there).
    """
    if c_eff < c:
        raise ValueError("effective oversampling below requested factor")
    a = ALPHA_FRACTION * math.pi * (2.0 * c_eff - 1.0) if alpha is None else float(alpha)
    hi = math.pi * (2.0 * c_eff - 1.0)
    if not (a > c_eff and a < hi) or a <= math.pi:
        raise ValueError(f"window support alpha={a} inadmissible for c={c_eff}")
    if beta is None:
        rad = (K / c_eff) ** 2 - (math.pi / a) ** 2
        b = math.sqrt(rad) if rad > 0 else math.pi * K * (2.0 - 1.0 / c_eff) / a
    else:
        b = float(beta)
    return (c_eff, int(K), a, b)


def kb_window(win, theta):
    """psi(theta) = I0(beta*sqrt(alpha^2-theta^2)), zero outside (nufft.py:159-165)."""
    _, _, a, b = win
    theta = np.asarray(theta, dtype=np.float64)
    arg = b * np.sqrt(np.maximum(a * a - theta * theta, 0.0))
    return np.where(np.abs(theta) <= a, i0(arg), 0.0)


def kb_window_ft(win, x):
    """psi_hat(x) = 2*alpha*sinh(s)/s, s = alpha*sqrt(beta^2-x^2) (nufft.py:168-187).

    Negative radicand continues sinh as sin; |s^2| < 1e-9 uses the series.
    """
    _, _, a, b = win
    x = np.asarray(x, dtype=np.float64)
    s2 = a * a * (b * b - x * x)
    out = np.empty_like(s2)
    tiny = np.abs(s2) < 1e-9
    up = (s2 >= 0) & ~tiny
    dn = (s2 < 0) & ~tiny
    r = np.sqrt(s2[up])
    out[up] = np.sinh(r) / r
    r = np.sqrt(-s2[dn])
    out[dn] = np.sin(r) / r
    q = s2[tiny]
    out[tiny] = 1.0 + q / 6.0 + q * q / 120.0
    return 2.0 * a * out


# ---------------------------------------------------------------------------
# direct sums (nufft.py:194-240) -- exact O(N*M) checks for the fast paths
# ---------------------------------------------------------------------------

def ner_direct(u, kappas):
    """sum_n u_n exp(-2 pi i kappa n / N) per row (nufft.py:194-216)."""
    u = np.asarray(u, dtype=np.complex128)
    kappas = np.asarray(kappas, dtype=np.float64)
    n = u.shape[-1]
    grid = np.arange(n)
    if kappas.ndim == 1:
        return u @ np.exp(-2j * np.pi * np.outer(grid, kappas) / n)
    ub = u.reshape(-1, n)
    kb = kappas.reshape(ub.shape[0], -1)
    out = np.stack([np.exp(-2j * np.pi * np.outer(k, grid) / n) @ row for row, k in zip(ub, kb)])
    return out.reshape(kappas.shape)


def ned_direct(positions, values, out_dims):
    """Exact NED sum onto a centred grid (nufft.py:219-240)."""
    positions = np.asarray(positions, dtype=np.float64)
    if positions.ndim == 1:
        positions = positions[:, None]
    values = np.asarray(values, dtype=np.complex128)
    out_dims = tuple(int(n) for n in np.atleast_1d(out_dims))
    axes = [np.arange(-n // 2, n // 2) for n in out_dims]
    mesh = np.meshgrid(*axes, indexing="ij")
    ph = sum(np.outer(mesh[a].ravel(), positions[:, a]) / n for a, n in enumerate(out_dims))
    return (np.exp(-2j * np.pi * ph) @ values).reshape(out_dims + values.shape[1:])


# ---------------------------------------------------------------------------
# fast NER (nufft.py:270-332)
# ---------------------------------------------------------------------------

class NerOracle:
    """Fast non-equispaced-range transform of length n (nufft.py:270-332)."""

    def __init__(self, n: int, c=2.0, K=6, alpha=None, beta=None):
        self.n = int(n)
        self.n_over = even_fast_len(c * n)                       # nufft.py:278
        self.c_eff = self.n_over / self.n                         # nufft.py:279
        self.win = resolve_window(c, K, alpha, beta, self.c_eff)  # nufft.py:280
        theta = 2.0 * np.pi * np.arange(self.n) / self.n - np.pi  # nufft.py:281
        self.prewin = 1.0 / kb_window(self.win, theta)            # nufft.py:282
        self.taps = np.arange(-K + 1, K + 1)                      # nufft.py:283
        self.norm = 1.0 / (2.0 * np.pi * self.c_eff)              # nufft.py:284
        self.kappa_max = self.n_over / 2.0                        # nufft.py:285

    def bins_weights(self, kappas):
        """Oversampled bins and complex weights per target (nufft.py:287-293)."""
        k0 = np.floor(self.c_eff * kappas).astype(np.int64)
        bins = k0[..., None] + self.taps
        off = kappas[..., None] - bins / self.c_eff
        w = self.norm * kb_window_ft(self.win, off) * np.exp(-1j * np.pi * off)
        return bins % self.n_over, w

    def rows(self, u, kappas, block_rows=None):
        """Per-row targets: u (R, n), kappas (R, m) -> (R, m) (nufft.py:295-332)."""
        u = np.asarray(u, dtype=np.complex128)
        kappas = np.asarray(kappas, dtype=np.float64)
        nrows, m = kappas.shape
        if block_rows is None:                                    # nufft.py:316-317
            block_rows = max(1, 4_000_000 // max(1, m * len(self.taps)))
        out = np.empty((nrows, m), dtype=np.complex128)
        for lo in range(0, nrows, block_rows):
            hi = min(lo + block_rows, nrows)
            spec = sfft.fft(u[lo:hi] * self.prewin, n=self.n_over, axis=-1, workers=_threads())
            bins, w = self.bins_weights(kappas[lo:hi])
            r = np.arange(hi - lo)[:, None, None]
            out[lo:hi] = np.sum(w * spec[r, bins], axis=-1)
        return out

    def shared(self, u, kappas):
        """One target vector for every row (nufft.py:319-327)."""
        u = np.asarray(u, dtype=np.complex128)
        kappas = np.asarray(kappas, dtype=np.float64)
        bins, w = self.bins_weights(kappas)
        spec = sfft.fft(u.reshape(-1, self.n) * self.prewin, n=self.n_over, axis=-1, workers=_threads())
        return np.einsum("mk,bmk->bm", w, spec[:, bins]).reshape(u.shape[:-1] + kappas.shape)


# ---------------------------------------------------------------------------
# fast NED (nufft.py:345-418)
# ---------------------------------------------------------------------------

class NedOracle:
    """Fast non-equispaced-data transform onto a centred grid (nufft.py:345-418)."""

    def __init__(self, out_dims, c=2.0, K=6, alpha=None, beta=None):
        self.out_dims = tuple(int(n) for n in np.atleast_1d(out_dims))
        self.K = int(K)
        self.n_over = tuple(even_fast_len(c * n) for n in self.out_dims)          # nufft.py:360
        self.c_eff = tuple(m / n for m, n in zip(self.n_over, self.out_dims))     # nufft.py:361
        resolve_window(c, K, alpha, beta, min(self.c_eff))                        # nufft.py:362
        self.wins = [resolve_window(c, K, alpha, beta, ce) for ce in self.c_eff]  # nufft.py:363
        self.taps = np.arange(-K + 1, K + 1)
        self.deapod = []                                                          # nufft.py:367-371
        for ax, n in enumerate(self.out_dims):
            j = np.arange(-n // 2, n // 2)
            psi = kb_window(self.wins[ax], 2.0 * np.pi * j / n)
            self.deapod.append(1.0 / (2.0 * np.pi * self.c_eff[ax] * psi))

    def axis_bins_weights(self, x, ax):
        """Per-axis oversampled bins and real weights (nufft.py:373-378)."""
        k0 = np.floor(self.c_eff[ax] * x).astype(np.int64)
        bins = k0[:, None] + self.taps
        off = x[:, None] - bins / self.c_eff[ax]
        return bins % self.n_over[ax], kb_window_ft(self.wins[ax], off)

    def spread_operator(self, positions):
        """Sparse (prod n_over, M) spreading matrix (nufft.py:380-398)."""
        m = positions.shape[0]
        if len(self.out_dims) == 1:
            b, w = self.axis_bins_weights(positions[:, 0], 0)
            rows, vals = b.ravel(), w.ravel()
            cols = np.repeat(np.arange(m), b.shape[1])
        else:
            b0, w0 = self.axis_bins_weights(positions[:, 0], 0)
            b1, w1 = self.axis_bins_weights(positions[:, 1], 1)
            rows = (b0[:, :, None] * self.n_over[1] + b1[:, None, :]).ravel()
            vals = (w0[:, :, None] * w1[:, None, :]).ravel()
            cols = np.repeat(np.arange(m), b0.shape[1] * b1.shape[1])
        size = int(np.prod(self.n_over))
        return sps.coo_matrix((vals, (rows, cols)), shape=(size, m)).tocsr()

    def execute(self, positions, values, wrapped=True):
        """Spread, oversampled FFT, centred crop, deapodise (nufft.py:400-418)."""
        positions = np.asarray(positions, dtype=np.float64)
        if positions.ndim == 1:
            positions = positions[:, None]
        values = np.asarray(values, dtype=np.complex128)
        single = values.ndim == 1
        vb = values[:, None] if single else values
        grid = (self.spread_operator(positions) @ vb).reshape(self.n_over + (vb.shape[1],))
        nax = len(self.n_over)
        spec = sfft.fftn(grid, axes=tuple(range(nax)), workers=_threads())
        sel = [np.arange(-n // 2, n // 2) % m for n, m in zip(self.out_dims, self.n_over)]
        out = spec[np.ix_(*sel)]
        for ax, dp in enumerate(self.deapod):
            shape = [1] * out.ndim
            shape[ax] = dp.size
            out = out * dp.reshape(shape)
        if wrapped:
            out = np.fft.ifftshift(out, axes=tuple(range(nax)))
        return out[..., 0] if single else out


# ---------------------------------------------------------------------------
# reconstruction pipeline (recon.py:200-379)
# ---------------------------------------------------------------------------

def wrapped_freqs(n: int, scale: float = 1.0):
    """fftfreq(n)*n*scale, with the reference's rounding (recon.py:211,282)."""
    return sfft.fftfreq(n) * n * scale


def lateral_freq_sq(n_lateral, ratios):
    """sum_ax (j_ax*ratio_ax)^2 on the wrapped lateral grid (recon.py:200-215)."""
    j2 = np.zeros(n_lateral)
    for ax, n in enumerate(n_lateral):
        shape = [1] * len(n_lateral)
        shape[ax] = n
        j2 = j2 + (wrapped_freqs(n, ratios[ax]) ** 2).reshape(shape)
    return j2


def even_extension(gh):
    """[g_0..g_{N-1}, 0, g_{N-1}..g_1] along the last axis (recon.py:263-271)."""
    pad = np.zeros(gh.shape[:-1] + (1,), dtype=gh.dtype)
    return np.concatenate([gh, pad, gh[..., :0:-1]], axis=-1)


def ner_targets(j2, nt):
    """kappa_e = 2*kappa on the band, 0 off it; and amp*band (recon.py:282-293).

    ``j2`` holds the squared lateral frequency of each row (any shape); the
    returned arrays have shape ``j2.shape + (nt,)``.
    """
    lv = wrapped_freqs(nt)
    j2 = np.asarray(j2)[..., None]
    kap = np.sign(lv) * np.sqrt(j2 + lv ** 2)
    band = (j2 + lv ** 2) <= (nt / 2.0) ** 2
    amp = np.zeros(kap.shape)
    np.divide(2.0 * lv, kap, out=amp, where=kap != 0)
    return np.where(band, 2.0 * kap, 0.0), amp * band


def fhat_rows(gh_rows, j2_rows, nt, spec):
    """Steps 2-3 for a set of lateral rows (recon.py:282-308, 'nufft' branch).

    gh_rows: (R, nt) lateral spectra; j2_rows: (R,) squared lateral frequency.
    """
    kap_e, scale = ner_targets(j2_rows, nt)
    ext = even_extension(gh_rows)
    phi = NerOracle(2 * nt, *spec).rows(ext, kap_e)
    return 0.5 * phi * scale


def fhat_rows_interp(gh_rows, j2_rows, nt):
    """Steps 2-3 with linear interpolation of the 2T FFT (recon.py:297-303)."""
    kap_e, scale = ner_targets(j2_rows, nt)
    spect = sfft.fft(even_extension(gh_rows), axis=-1)
    i0 = np.floor(kap_e).astype(np.int64)
    frac = kap_e - i0
    r = np.arange(spect.shape[0])[:, None]
    phi = spect[r, i0 % (2 * nt)] * (1.0 - frac) + spect[r, (i0 + 1) % (2 * nt)] * frac
    return 0.5 * phi * scale


def assemble_fhat(gh, nt, spec, ratios, time_eval="nufft"):
    """Warped time-axis NER + amplitude + band over the whole lateral grid (recon.py:274-308)."""
    n_lateral = gh.shape[:-1]
    nrows = int(np.prod(n_lateral)) if n_lateral else 1
    j2 = lateral_freq_sq(n_lateral, ratios).reshape(nrows)
    if time_eval == "interp":
        return fhat_rows_interp(gh.reshape(nrows, nt), j2, nt).reshape(gh.shape)
    return fhat_rows(gh.reshape(nrows, nt), j2, nt, spec).reshape(gh.shape)


def hermitian_part(a):
    """0.5*(a + conj(a[-k])) with wrapped negation on every axis (recon.py:218-222)."""
    b = a
    for ax in range(a.ndim):
        b = np.roll(np.flip(b, axis=ax), 1, axis=ax)
    return 0.5 * (a + np.conj(b))


def zero_pad_axis(a, ax, up):
    """Spectral zero-padding with Nyquist split (recon.py:225-246)."""
    n = a.shape[ax]
    m = up * n
    shape = list(a.shape)
    shape[ax] = m
    out = np.zeros(shape, dtype=a.dtype)

    def sl(s):
        idx = [slice(None)] * a.ndim
        idx[ax] = s
        return tuple(idx)

    out[sl(slice(0, n // 2))] = a[sl(slice(0, n // 2))]
    out[sl(slice(m - n // 2 + 1, m))] = a[sl(slice(n // 2 + 1, n))]
    out[sl(n // 2)] = 0.5 * a[sl(n // 2)]
    out[sl(m - n // 2)] = 0.5 * a[sl(n // 2)]
    return out


def invert_spectrum(fhat, upsample):
    """Symmetrise, pad, inverse FFT, lateral fftshift, real part (recon.py:249-260).

    Returns (image, imag_residual).
    """
    fhat = hermitian_part(fhat)
    if upsample > 1:
        for ax in range(fhat.ndim):
            fhat = zero_pad_axis(fhat, ax, upsample)
    img = sfft.ifftn(fhat) * upsample ** fhat.ndim
    peak = np.max(np.abs(img.real))
    resid = float(np.max(np.abs(img.imag)) / peak) if peak > 0 else 0.0
    img = np.fft.fftshift(img.real, axes=tuple(range(img.ndim - 1)))
    return img, resid


def lateral_ratios(nt, dt, sound_speed, dx, n_lateral):
    """Depth extent over aperture extent per lateral axis (recon.py:340-342)."""
    depth = nt * (sound_speed * dt)
    return tuple(depth / (n * dx) for n in n_lateral)


def reconstruct_nedner(positions, weights, samples, dt, sound_speed, dx, n_lateral,
                       out_dims=None, upsample=1, spec=(2.0, 6, None, None)):
    """NEDNER reconstruction (recon.py:358-379).  Returns (image, imag_residual).

    ``spec`` is (c, K, alpha, beta) with None for "resolve at plan time".
    Inputs are assumed validated (the product's SensorRecord does that).
    """
    positions = np.atleast_2d(np.asarray(positions, dtype=np.float64))
    samples = np.asarray(samples, dtype=np.float64)
    weights = np.asarray(weights, dtype=np.float64).ravel()
    n_lateral = tuple(int(n) for n in np.atleast_1d(n_lateral))
    if positions.shape[1] != len(n_lateral):
        positions = positions.T
    out_dims = n_lateral if out_dims is None else tuple(int(n) for n in np.atleast_1d(out_dims))
    nt = samples.shape[1]
    scaled = samples * (weights / dx ** len(out_dims))[:, None]                 # recon.py:374
    ned = NedOracle(out_dims, *spec)                                              # recon.py:375
    pos = (positions / dx) * (np.asarray(out_dims, float) / np.asarray(n_lateral, float))  # recon.py:376
    gh = ned.execute(pos, scaled.astype(np.complex128), wrapped=True)            # recon.py:377
    ratios = lateral_ratios(nt, dt, sound_speed, dx, n_lateral)
    fhat = assemble_fhat(gh, nt, spec, ratios)                                    # recon.py:378
    return invert_spectrum(fhat, upsample)                                        # recon.py:379


def full_grid_cube(positions, samples, dx, n_lateral):
    """Samples placed on the complete lateral grid, centred (recon.py:311-333)."""
    pos = np.atleast_2d(np.asarray(positions, dtype=np.float64)) / dx
    if pos.shape[1] != len(n_lateral):
        pos = pos.T
    idx = np.rint(pos).astype(np.int64)
    if np.max(np.abs(pos - idx)) > 1e-6:
        raise ValueError("record positions do not form the complete sensor grid")
    for ax, n in enumerate(n_lateral):
        idx[:, ax] += n // 2
    flat = np.ravel_multi_index(tuple(idx.T), n_lateral)
    if len(np.unique(flat)) != int(np.prod(n_lateral)) or flat.size != int(np.prod(n_lateral)):
        raise ValueError("record positions do not form the complete sensor grid")
    cube = np.empty((int(np.prod(n_lateral)), samples.shape[1]))
    cube[flat] = samples
    return cube.reshape(tuple(n_lateral) + (samples.shape[1],))


def reconstruct_equispaced(positions, samples, dt, sound_speed, dx, n_lateral, upsample=1,
                           spec=(2.0, 6, None, None), time_eval="nufft"):
    """reconstruct_equispaced (recon.py:345-355) / reconstruct_interp_fft (recon.py:382-389)."""
    n_lateral = tuple(int(n) for n in np.atleast_1d(n_lateral))
    samples = np.asarray(samples, dtype=np.float64)
    cube = full_grid_cube(positions, samples, dx, n_lateral)
    lat = tuple(range(cube.ndim - 1))
    gh = sfft.fftn(np.fft.ifftshift(cube, axes=lat).astype(np.complex128), axes=lat)
    nt = samples.shape[1]
    ratios = lateral_ratios(nt, dt, sound_speed, dx, n_lateral)
    fhat = assemble_fhat(gh, nt, spec, ratios, time_eval=time_eval)
    return invert_spectrum(fhat, upsample)


def out_spacing(dx, dt, sound_speed, nlat, upsample):
    """Output pitch per axis (recon.py:336-337, 259)."""
    return tuple(s / upsample for s in ((dx,) * nlat + (sound_speed * dt,)))
