"""Exception hierarchy of the drop-in API.

Names and bases match the reference's ``moeplan.errors``
(``/root/reference/pkg/src/moeplan/errors.py:4-41``) so callers that catch
``StrategyError`` / ``CapacityError`` / ``VerificationError`` keep working.
The C-ABI error codes map onto these in ``_native.check``.
"""

__all__ = ["MoeplanError", "ConfigError", "GrammarError", "StrategyError",
           "SaturationError", "CalibrationError", "AnalyzerError",
           "CapacityError", "SchedulingError", "VerificationError"]


class MoeplanError(Exception):
    """Root of every error raised by this package."""


# input validation errors (also ValueError for generic callers)
class ConfigError(MoeplanError, ValueError):
    """A configuration value or file violates its schema or invariants."""


class GrammarError(MoeplanError, ValueError):
    """A strategy string does not follow the parallel-strategy grammar."""


class StrategyError(MoeplanError, ValueError):
    """Well-formed strategy or shapes that do not fit the other inputs
    (cluster size, token divisibility, partial shapes); MX_ERR_INVALID."""


class CalibrationError(MoeplanError, ValueError):
    """A least-squares coefficient fit is degenerate."""


# runtime conditions
class SaturationError(MoeplanError, ArithmeticError):
    """M/M/1 utilisation reached or exceeded one."""


class AnalyzerError(MoeplanError, RuntimeError):
    """No strategy survives the memory bound and SLO filters."""


class CapacityError(MoeplanError, RuntimeError):
    """A host group would receive more routed slots than its receive
    buffer holds (MX_ERR_CAPACITY); tokens are never dropped."""


class SchedulingError(MoeplanError, RuntimeError):
    """A trace dependency graph cannot be scheduled (cycle)."""


class VerificationError(MoeplanError, AssertionError):
    """Layer output disagrees with the dense reference beyond tolerance."""
