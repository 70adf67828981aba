"""Standalone GPU non-equispaced-range NUFFT: ``NerPlan`` / ``nufft_ner``.

Mirrors the reference's API (/root/reference/pkg/src/patfft/nufft.py:270-338):

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

__all__ = ["NerPlan", "nufft_ner"]


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
