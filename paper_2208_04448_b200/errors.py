"""Exception types mirroring svcodec.errors (errors.py:4-63).

When the reference package is importable its classes are re-used, so code
catching ``svcodec.errors.SvcodecError`` also catches errors raised here.
"""

try:  # pragma: no cover - depends on the environment
    from svcodec.errors import EncodeError, OutOfCoverageError, SvcodecError  # type: ignore
except Exception:  # noqa: BLE001
    class SvcodecError(Exception):
        """Base class for codec errors (errors.py:4)."""

    class OutOfCoverageError(SvcodecError):
        """A point outside every gate (errors.py:20-21)."""

    class EncodeError(SvcodecError):
        """Training failure, optionally naming the expert (errors.py:28-35)."""

        def __init__(self, msg: str, expert_id=None):
            self.expert_id = expert_id
            super().__init__(msg if expert_id is None else f"expert {expert_id}: {msg}")

__all__ = ["SvcodecError", "OutOfCoverageError", "EncodeError"]
