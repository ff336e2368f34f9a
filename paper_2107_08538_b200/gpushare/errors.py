"""Exception hierarchy of the drop-in (mirrors gpushare/errors.py:10-73).

ConfigError covers bad input and maps to exit code 2; ContractViolation
covers protocol misuse (stale plans, unknown releases) and maps to exit
code 3.  libgs status codes -2 / -3 map onto these two.
"""


class GpuShareError(Exception):
    pass


class ConfigError(GpuShareError):
    """Bad user input: specs, policies, requests."""

    exit_code = 2


class ContractViolation(GpuShareError):
    """An operation was called in a state its contract forbids."""

    exit_code = 3


class AnalysisError(ConfigError):
    """Probe construction failed (byte overflow, undeclared buffer)."""


class LazyBindingError(ContractViolation):
    """Lazy probe assembly was driven outside its protocol."""
