"""B200-native NEDNER-NUFFT planar photoacoustic reconstruction.

Drop-in for ``patfft.recon.reconstruct_nedner`` of the reference
(arXiv 1501.02946, /root/reference/pkg/src/patfft/recon.py:358-379): same
Python signature and types, executed by hand-written sm_100a CUDA kernels
behind the C ABI in ``include/patfft_b200.h``.
"""

from .errors import DataValidationError, DeviceError, NumericalError, ParameterError
from .recon import (
    EquispacedPlan,
    NedNerPlan,
    ScalarField,
    SensorRecord,
    amplitude_factor,
    kappa,
    reconstruct_equispaced,
    reconstruct_interp_fft,
    reconstruct_nedner,
)
from .nufft import NedPlan, NerPlan, nufft_ned, nufft_ner
from .forward import ForwardPlan, forward_fourier
from .arrayfile import open_array, read_array, reconstruct_frames_file, write_array
from .window import WindowSpec

__version__ = "0.1.0"

__all__ = [
    "DataValidationError",
    "DeviceError",
    "NumericalError",
    "ParameterError",
    "EquispacedPlan",
    "ForwardPlan",
    "NedNerPlan",
    "NedPlan",
    "NerPlan",
    "ScalarField",
    "SensorRecord",
    "WindowSpec",
    "amplitude_factor",
    "forward_fourier",
    "open_array",
    "read_array",
    "reconstruct_frames_file",
    "write_array",
    "nufft_ned",
    "nufft_ner",
    "kappa",
    "reconstruct_equispaced",
    "reconstruct_interp_fft",
    "reconstruct_nedner",
    "__version__",
]
