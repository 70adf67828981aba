"""``WindowSpec``: Kaiser-Bessel gridding window parameters.

Mirrors the reference's dataclass (/root/reference/pkg/src/patfft/nufft.py:92-156):
same fields, defaults, validation and ``resolved`` semantics, so a spec
built for the reference can be passed unchanged.  The device plan
re-resolves alpha/beta per transform for the oversampling it actually uses
(exactly as the reference resolves them for its own rounded FFT lengths).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

from .errors import ParameterError

_ALPHA_FRACTION = 0.999  # nufft.py:61


@dataclass(frozen=True)
class WindowSpec:
    c: float = 2.0
    K: int = 6
    alpha: float | None = None
    beta: float | None = None

    def __post_init__(self):  # nufft.py:114-122
        if not math.isfinite(self.c) or self.c <= 1.0:
            raise ParameterError(f"oversampling factor must exceed 1, got {self.c}")
        if int(self.K) != self.K or self.K < 1:
            raise ParameterError(f"interpolation half-width K must be an integer >= 1, got {self.K}")
        if self.alpha is not None:
            self._check_alpha(self.alpha, self.c)
        if self.beta is not None and (not math.isfinite(self.beta) or self.beta <= 0):
            raise ParameterError(f"window shape beta must be positive, got {self.beta}")

    @staticmethod
    def _check_alpha(alpha: float, c: float) -> None:  # nufft.py:124-131
        hi = math.pi * (2.0 * c - 1.0)
        if not (alpha > c and alpha < hi):
            raise ParameterError(f"window support alpha={alpha} outside admissible range ({c}, {hi})")
        if alpha <= math.pi:
            raise ParameterError(f"window support alpha={alpha} must exceed pi")

    def resolved(self, c_eff: float | None = None) -> "WindowSpec":  # nufft.py:133-149
        c = self.c if c_eff is None else c_eff
        if c_eff is not None and c_eff < self.c:
            raise ParameterError("effective oversampling below requested factor")
        alpha = self.alpha
        if alpha is None:
            alpha = _ALPHA_FRACTION * math.pi * (2.0 * c - 1.0)
        self._check_alpha(alpha, c)
        beta = self.beta
        if beta is None:
            rad = (self.K / c) ** 2 - (math.pi / alpha) ** 2
            beta = math.sqrt(rad) if rad > 0 else math.pi * self.K * (2.0 - 1.0 / c) / alpha
        return replace(self, c=c, alpha=alpha, beta=beta)
