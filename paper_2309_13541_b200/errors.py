"""Error classes of the drop-in surface.

When the reference package ``a2aflow`` is importable (the drop-in situation:
a caller of the reference swaps in this executor), ``EvalError`` and
``RouteError`` subclass the reference's own classes
(``a2aflow.evaluate.EvalError``, pkg/src/a2aflow/evaluate.py:30-31;
``a2aflow.paths.RouteError``, pkg/src/a2aflow/paths.py:45-46), so code that
catches the reference's exceptions catches ours unchanged.  Without it they
keep the reference's bases (``RuntimeError`` / ``ValueError``).
"""
from __future__ import annotations

__all__ = ["EvalError", "RouteError", "REFERENCE_CLASSES"]

try:  # pragma: no cover - depends on the caller's environment
    from a2aflow.evaluate import EvalError as _RefEvalError
    from a2aflow.paths import RouteError as _RefRouteError
    REFERENCE_CLASSES = True
except Exception:  # noqa: BLE001 - any import failure means "standalone"
    _RefEvalError, _RefRouteError = RuntimeError, ValueError
    REFERENCE_CLASSES = False


class EvalError(_RefEvalError):
    """A schedule the reference replay would reject; same messages
    (reference pkg/src/a2aflow/evaluate.py:30-31)."""


class RouteError(_RefRouteError):
    """A path that does not join its commodity, is not simple, or uses a
    missing edge (reference pkg/src/a2aflow/paths.py:45-57)."""
