"""Error hierarchy of the drop-in API.

Mirrors the reference's exception tree (``pkg/src/gpukalc/errors.py:4-34``) so
callers that catch ``ScheduleError`` / ``EnsembleError`` / ``ProfileError`` keep
working.  ``DeviceError`` is new: it is raised when the sm_100a library is
missing or a CUDA call through the C-ABI fails (there is no CPU fallback).
"""

from __future__ import annotations


class GpukalcError(Exception):
    """Base class (reference ``errors.py:4``)."""


class PtxParseError(GpukalcError):
    """Malformed PTX (reference ``errors.py:8-18``); carries the 1-based line."""

    def __init__(self, message, line=None):
        self.line = line
        if line is not None:
            message = f"line {line}: {message}"
        super().__init__(message)


class ProfileError(GpukalcError):
    """Missing / malformed / inconsistent arch profile (reference ``errors.py:21``)."""


class ScheduleError(GpukalcError):
    """Kernel cannot be scheduled under a launch config (reference ``errors.py:25``)."""


class FitError(GpukalcError):
    """Reference ``errors.py:29`` (profile fitting; kept for API parity)."""


class EnsembleError(GpukalcError):
    """Malformed ensemble or manifest mismatch (reference ``errors.py:33``)."""


class TrainerError(Exception):
    """Trainer-side error (reference ``trainer/src/gpukalc_trainer/errors.py``)."""


class DeviceError(GpukalcError):
    """The CUDA library is missing, failed to load, or a device call failed."""
