"""B200-native SFT/ASFT Gaussian smoothing and Morlet wavelet transforms.

The hot path (window-recurrence scan + coefficient combine) runs as hand-written
sm_100a CUDA kernels in ``libsftgpu.so`` behind the C ABI of ``include/sftgpu.h``;
``sft`` mirrors the reference library's public API (namespace ``sft``).
"""
from . import sft  # noqa: F401
from .sft import *  # noqa: F401,F403

__version__ = "0.1.0"
