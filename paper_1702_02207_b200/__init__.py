"""B200-native RK4 time stepping of M x'' + K x = 0 (arXiv 1702.02207).

Drop-in for the hot path of the reference package ``oscbench``
(/root/reference/pkg/src/oscbench/oscillator.py:152-276): the same public
names (``__init__.py:9-23`` of the reference), with the arithmetic executed by
hand-written sm_100a kernels in ``libosc_b200.so`` (C ABI: include/osc_b200.h).

Importing this package needs no GPU; calling into it does, and fails loudly
(:class:`NativeUnavailableError`) when the library or the device is missing.
"""

from ._native import NativeUnavailableError
from .oscillator import (
    DimensionMismatchError,
    LengthMismatchError,
    NonFiniteStateError,
    NonPositiveParameterError,
    OscillatorSystem,
    PhaseDerivative,
    PhaseState,
    Trajectory,
    build_chain,
    derivative,
    energy,
    integrate,
    rk4_step,
)

__version__ = "0.1.0"

__all__ = [
    "DimensionMismatchError",
    "LengthMismatchError",
    "NativeUnavailableError",
    "NonFiniteStateError",
    "NonPositiveParameterError",
    "OscillatorSystem",
    "PhaseDerivative",
    "PhaseState",
    "Trajectory",
    "build_chain",
    "derivative",
    "energy",
    "integrate",
    "rk4_step",
]
