"""Standalone GPU non-equispaced-range NUFFT: ``NerPlan`` / ``nufft_ner``.

Mirrors the reference's API (/root/reference/pkg/src/patfft/nufft.py:270-423):

    NerPlan(n, spec=None).execute(u, kappas)  ->  complex128 array
    nufft_ner(u, kappas, spec=None)

``u`` has shape (..., n); ``kappas`` is (M,) for targets shared by every row
or (..., M) matching u's batch shape for per-row targets; the result
approximates sum_k u[..., k] exp(-2 pi i kappa k / n).  Validation and error
classes follow nufft.py:301-311.  Execution is the sm_100a kernel of
csrc/ner_api.cu behind the C ABI (no CPU fallback).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .errors import ParameterError
from .window import WindowSpec

__all__ = ["NerPlan", "nufft_ner", "NedPlan", "nufft_ned"]


def _even_fast_len(target: float) -> int:
    """Reference oversampled length (nufft.py:83-89): used for kappa_max."""

    def smooth(n):
        for p in (2, 3, 5, 7, 11):
            while n % p == 0:
                n //= p
        return n == 1

    n = max(2, int(math.ceil(target)))
    while not (smooth(n) and n % 2 == 0):
        n += 1
    return n


class NerPlan:
    """Precomputed device state for non-equispaced-range transforms of length n."""

    def __init__(self, n: int, spec: WindowSpec | None = None, device: int = 0):
        if n < 2:
            raise ParameterError("input length must be >= 2")  # nufft.py:274-275
        spec = spec if spec is not None else WindowSpec()
        if not isinstance(spec, WindowSpec):
            spec = WindowSpec(c=spec.c, K=spec.K, alpha=spec.alpha, beta=spec.beta)
        self.n = int(n)
        self.spec = spec
        # the reference's range bound (nufft.py:278, 285)
        self.n_over = _even_fast_len(spec.c * n)
        self.c_eff = self.n_over / self.n
        self.kappa_max = self.n_over / 2.0
        lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(lib.patfft_ner_plan_create(int(n), float(spec.c), int(spec.K),
                                              math.nan if spec.alpha is None else float(spec.alpha),
                                              math.nan if spec.beta is None else float(spec.beta), int(device),
                                              ctypes.byref(h)))
        self._lib = lib
        self._h = h

    def execute(self, u, kappas, block_rows: int | None = None):
        """Evaluate the length-n DFT of each row of ``u`` at ``kappas`` (nufft.py:295-332)."""
        u = np.asarray(u, dtype=np.complex128)
        if u.shape[-1] != self.n:
            raise ParameterError(f"plan built for length {self.n}, got {u.shape[-1]}")
        kappas = np.asarray(kappas, dtype=np.float64)
        if not np.all(np.isfinite(kappas)):
            raise ParameterError("kappas must be finite")
        if np.any(np.abs(kappas) > self.kappa_max):
            raise ParameterError(f"|kappa| must not exceed {self.kappa_max}")
        shared = kappas.ndim == 1
        if not shared and kappas.shape[:-1] != u.shape[:-1]:
            raise ParameterError("per-row kappas must match the batch shape of u")
        m = kappas.shape[-1]
        batch = u.shape[:-1]
        ub = np.ascontiguousarray(u.reshape(-1, self.n))
        kb = np.ascontiguousarray(kappas.reshape(-1))
        rows = ub.shape[0]
        out = np.empty((rows, m), dtype=np.complex128)
        _lib.check(self._lib.patfft_ner_execute(self._h, _lib.ptr(ub), _lib.ptr(kb), rows, m, 1 if shared else 0,
                                                _lib.ptr(out)))
        return out.reshape(batch + (m,)) if shared else out.reshape(kappas.shape)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.patfft_ner_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nufft_ner(u, kappas, spec: WindowSpec | None = None):
    """Fast non-equispaced-range transform (nufft.py:335-338)."""
    u = np.asarray(u, dtype=np.complex128)
    return NerPlan(u.shape[-1], spec).execute(u, kappas)


def _check_ned_inputs(positions, values, out_dims):  # nufft.py:243-263
    positions = np.asarray(positions, dtype=np.float64)
    if positions.ndim == 1:
        positions = positions[:, None]
    if positions.ndim != 2:
        raise ParameterError("positions must be (M,) or (M, d)")
    out_dims = tuple(int(n) for n in np.atleast_1d(out_dims))
    if len(out_dims) != positions.shape[1]:
        raise ParameterError("out_dims length must match position dimensionality")
    if not 1 <= len(out_dims) <= 2:
        raise ParameterError("NED transforms support 1 or 2 position axes")
    for n in out_dims:
        if n < 2 or n % 2:
            raise ParameterError("centered grid lengths must be even and >= 2")
    for ax, n in enumerate(out_dims):
        if np.any(np.abs(positions[:, ax]) > n / 2):
            raise ParameterError("positions fall outside the centered domain")
    values = np.asarray(values, dtype=np.complex128)
    if values.shape[0] != positions.shape[0]:
        raise ParameterError("values and positions disagree on sample count")
    return positions, values, out_dims


class NedPlan:
    """Non-equispaced-data NUFFT onto a centred grid (nufft.py:345-418) on the GPU.

    Output grids follow the centred convention (index 0 along axis i is
    frequency -N_i/2) unless ``order="wrapped"``.
    """

    def __init__(self, out_dims, spec: WindowSpec | None = None, device: int = 0):
        spec = spec if spec is not None else WindowSpec()
        if not isinstance(spec, WindowSpec):
            spec = WindowSpec(c=spec.c, K=spec.K, alpha=spec.alpha, beta=spec.beta)
        self.out_dims = tuple(int(n) for n in np.atleast_1d(out_dims))
        if not 1 <= len(self.out_dims) <= 2:
            raise ParameterError("NED transforms support 1 or 2 position axes")  # nufft.py:355-356
        for n in self.out_dims:
            if n < 2 or n % 2:
                raise ParameterError("centered grid lengths must be even and >= 2")
        self.spec = spec
        self.device = int(device)
        self._lib = _lib.load()
        self._key = None
        self._h = None

    def _plan(self, positions, nvals):
        key = (positions.shape, hash(positions.tobytes()), nvals)
        if key == self._key and self._h is not None:
            return self._h
        self.close()
        dims = (ctypes.c_int32 * 2)(*(self.out_dims + (0,))[:2])
        h = ctypes.c_void_p()
        s = self.spec
        _lib.check(self._lib.patfft_ned_plan_create(
            len(self.out_dims), dims, int(nvals), float(s.c), int(s.K),
            math.nan if s.alpha is None else float(s.alpha), math.nan if s.beta is None else float(s.beta),
            positions.ctypes.data_as(_lib._D), positions.shape[0], self.device, ctypes.byref(h)))
        self._h, self._key = h, key
        return h

    def execute(self, positions, values, order: str = "centered"):
        positions, values, out_dims = _check_ned_inputs(positions, values, self.out_dims)
        if order not in ("centered", "wrapped"):
            raise ParameterError("order must be 'centered' or 'wrapped'")  # nufft.py:416-417
        single = values.ndim == 1
        vb = values[:, None] if single else values.reshape(values.shape[0], -1)
        positions = np.ascontiguousarray(positions)
        vb = np.ascontiguousarray(vb)
        h = self._plan(positions, vb.shape[1])
        out = np.empty(out_dims + (vb.shape[1],), dtype=np.complex128)
        _lib.check(self._lib.patfft_ned_execute(h, _lib.ptr(vb), _lib.ptr(out), 1 if order == "centered" else 0))
        if single:
            return out[..., 0]
        return out.reshape(out_dims + values.shape[1:])

    def close(self):
        if getattr(self, "_h", None):
            self._lib.patfft_nedner_plan_destroy(self._h)
        self._h = None
        self._key = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nufft_ned(positions, values, out_dims, spec: WindowSpec | None = None):
    """Fast non-equispaced-data transform (nufft.py:421-423)."""
    return NedPlan(out_dims, spec).execute(positions, values)
