"""GPU forward model: ``forward_fourier`` (full-grid sensor data of a field).

Mirrors the reference's ``patfft.forward.forward_fourier(f, sound_speed,
spec=None) -> SensorRecord`` (/root/reference/pkg/src/patfft/forward.py:105-166):
same arguments, validation, error classes and returned record (grid-node
positions, weights dx^(d-1), dt = dz / c, one trace of N_t samples per
lateral grid node).  The transform runs on the sm_100a kernels behind
``patfft_forward_*`` in include/patfft_b200.h (cuFFT for the uniform lateral
FFTs, a fused NER + depth-IFFT kernel per lateral frequency row); there is
no CPU fallback.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import ParameterError
from .recon import ScalarField, SensorRecord
from .window import WindowSpec

__all__ = ["ForwardPlan", "forward_fourier", "grid_node_positions"]


def lateral_freq_sq(n_lateral, ratios):
    """sum_ax (fftfreq(n)*n*ratio)^2 on the wrapped lateral grid (recon.py:200-215)."""
    j2 = np.zeros(n_lateral)
    for ax, n in enumerate(n_lateral):
        f = (np.fft.fftfreq(n) * n * ratios[ax]) ** 2
        shape = [1] * len(n_lateral)
        shape[ax] = n
        j2 = j2 + f.reshape(shape)
    return j2


def grid_node_positions(n_lateral, dx):
    """Sensor positions of the full grid, C order (forward.py:169-172)."""
    axes = [(np.arange(n) - n // 2) * dx for n in n_lateral]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.ravel() for m in mesh], axis=-1)


def _check_field(vals, sound_speed):  # forward.py:112-119
    if sound_speed <= 0:
        raise ParameterError("sound speed must be positive")
    if vals.ndim not in (2, 3):
        raise ParameterError("forward operator supports 2D and 3D fields")
    if vals.shape[-1] % 2 or any(n % 2 for n in vals.shape[:-1]):
        raise ParameterError("grid sizes must be even")


class ForwardPlan:
    """Device plan of the forward model for one grid shape and spacing."""

    def __init__(self, shape, spacing, spec: WindowSpec | None = None, device: int = 0):
        shape = tuple(int(n) for n in shape)
        spacing = tuple(float(s) for s in spacing)
        n_lateral, nt = shape[:-1], shape[-1]
        spec = spec if spec is not None else WindowSpec()
        depth_extent = nt * spacing[-1]                                       # forward.py:140
        ratios = tuple(depth_extent / (n * spacing[ax]) for ax, n in enumerate(n_lateral))
        j2 = np.ascontiguousarray(lateral_freq_sq(n_lateral, ratios), dtype=np.float64)
        self.shape = shape
        self.device = device
        lib = _lib.load()
        dims = (ctypes.c_int32 * 2)(*n_lateral, *([0] * (2 - len(n_lateral))))
        h = ctypes.c_void_p()
        nan = float("nan")
        _lib.check(lib.patfft_forward_plan_create(
            len(n_lateral), dims, nt, j2.ctypes.data_as(_lib._D), float(spec.c), int(spec.K),
            nan if spec.alpha is None else float(spec.alpha), nan if spec.beta is None else float(spec.beta),
            device, ctypes.byref(h)), "forward plan")
        self._h = h

    def execute(self, values: np.ndarray) -> np.ndarray:
        """Traces (prod n_lateral, N_t) float64 of a field of the plan's shape."""
        vals = np.ascontiguousarray(values, dtype=np.float64)
        if vals.shape != self.shape:
            raise ParameterError(f"plan built for shape {self.shape}, got {vals.shape}")
        out = np.empty(vals.shape, dtype=np.float64)
        _lib.check(_lib.load().patfft_forward_execute(self._h, _lib.ptr(vals), _lib.ptr(out)), "forward execute")
        return out.reshape(-1, self.shape[-1])

    def execute_device(self, field_ptr: int, traces_ptr: int, stream: int = 0) -> None:
        """float32 device buffers (may alias); enqueues on ``stream``."""
        _lib.check(_lib.load().patfft_forward_execute_device(self._h, ctypes.c_void_p(field_ptr),
                                                             ctypes.c_void_p(traces_ptr),
                                                             ctypes.c_void_p(stream or None)), "forward execute")

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().patfft_forward_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def forward_fourier(f: ScalarField, sound_speed: float, spec: WindowSpec | None = None, *,
                    device: int = 0) -> SensorRecord:
    """Simulate full-grid sensor data from an initial pressure field (forward.py:105-166).

    The time step is tied to the depth pitch by dt = dz / sound_speed, so the
    returned record has as many time samples as the field has depth samples.
    """
    vals = np.asarray(f.values, dtype=np.float64)
    _check_field(vals, sound_speed)
    n_lateral = vals.shape[:-1]
    plan = ForwardPlan(vals.shape, f.spacing, spec, device)
    try:
        traces = plan.execute(vals)
    finally:
        plan.close()
    dx = f.spacing[0]                                                         # forward.py:159-161
    rows = int(np.prod(n_lateral))
    return SensorRecord(positions=grid_node_positions(n_lateral, dx), weights=np.full(rows, dx ** len(n_lateral)),
                        samples=traces, dt=f.spacing[-1] / sound_speed, sound_speed=sound_speed, dx=dx,
                        n_lateral=n_lateral)
