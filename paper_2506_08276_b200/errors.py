"""Error hierarchy, mirroring the reference's (errors.py:11-93).

``code`` is one of usage / data / provider / internal; the C-ABI status codes
(include/leann_b200.h LV_ERR_*) map one-to-one onto these classes.
"""
from __future__ import annotations


class SlimvecError(Exception):
    code = "internal"


class InvalidArgumentError(SlimvecError, ValueError):
    code = "usage"


class FormatError(SlimvecError):
    code = "data"

    def __init__(self, section: str, message: str) -> None:
        super().__init__(f"{section}: {message}")
        self.section = section


class BuildError(SlimvecError):
    code = "data"


class ProviderError(SlimvecError):
    code = "provider"

    def __init__(self, message: str, retries: int = 0) -> None:
        super().__init__(message)
        self.retries = retries


class ProviderMismatchError(SlimvecError):
    code = "usage"


class SearchError(SlimvecError):
    code = "provider"

    def __init__(self, message: str, partial_report=None) -> None:
        super().__init__(message)
        self.partial_report = partial_report


class DeviceError(SlimvecError):
    """The CUDA library failed (LV_ERR_INTERNAL) or is missing."""

    code = "internal"


def raise_for(rc: int, message: str) -> None:
    """Map an LV_ERR_* return code onto the hierarchy."""
    if rc == 0:
        return
    if rc == 2:
        raise InvalidArgumentError(message)
    if rc == 3:
        raise FormatError("device", message)
    if rc == 4:
        raise SearchError(message)
    raise DeviceError(message)
