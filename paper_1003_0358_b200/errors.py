"""Exception types of the reference API (same names and bases)."""


class SizeMismatch(Exception):
    """network.py:20-21."""


class CheckpointError(Exception):
    """network.py:24-25."""


class CorruptHeader(CheckpointError):
    pass


class VersionMismatch(CheckpointError):
    pass


class PayloadLengthMismatch(CheckpointError):
    pass


class InvalidSigma(ValueError):
    """deform.py:26-27."""


class EvenSize(ValueError):
    """deform.py:30-31."""
