"""Exception types of the drop-in, mirroring trident/errors.py.

Same class names, hierarchy, constructor arguments and messages as the
reference (trident/errors.py:10-100).  When ``run`` is handed a reference
``TypedProgram`` it raises the REFERENCE's classes instead (resolved from
the program object's own package, see ``errors_for``), so callers' existing
``except trident.errors.NonConvergenceError`` clauses keep working.
"""

from __future__ import annotations

import sys
import types


class TridentError(Exception):
    """Base class for all toolchain errors (errors.py:10-11)."""


class GraphError(TridentError):
    """Graph loading and query errors (errors.py:53-54)."""


class GraphIoError(GraphError):
    pass


class FormatError(GraphError):
    """Malformed line in an edge-list file (errors.py:61-66)."""

    def __init__(self, lineno: int, message: str):
        super().__init__(f"line {lineno}: {message}")
        self.lineno = lineno


class RangeError(GraphError):
    """lo > hi passed to the random weight assigner."""


class ArgError(GraphError):
    """Invalid partitioning argument (e.g. zero ranks)."""


class EmptyGraphError(GraphError):
    """Aggregate weight query on a graph with no edges."""


class ExecError(TridentError):
    """Runtime failure inside the executor (errors.py:81-82)."""


class NonConvergenceError(ExecError):
    """A fixedPoint exceeded its iteration cap (errors.py:85-92)."""

    def __init__(self, flag: str, cap: int):
        super().__init__(
            f"fixedPoint '{flag}' did not converge within {cap} iterations")
        self.flag = flag
        self.cap = cap


class PartitionError(ExecError):
    """Invalid rank count or rank order."""


class SizeError(TridentError):
    """Input beyond a size bound."""


class UnsupportedProgramError(ExecError):
    """The program is not one of the corpus programs this backend runs on
    the GPU.  There is deliberately no CPU fallback."""


class BackendError(RuntimeError):
    """CUDA / device failure reported by the native library."""


_OURS = types.SimpleNamespace(
    TridentError=TridentError, GraphError=GraphError, GraphIoError=GraphIoError,
    FormatError=FormatError, RangeError=RangeError, ArgError=ArgError,
    EmptyGraphError=EmptyGraphError, ExecError=ExecError,
    NonConvergenceError=NonConvergenceError, PartitionError=PartitionError,
    SizeError=SizeError)


def errors_for(obj) -> types.SimpleNamespace:
    """Exception namespace matching ``obj``'s origin: the reference package's
    ``errors`` module when obj is a trident object, else this module."""
    mod = type(obj).__module__ or ""
    pkg = mod.rsplit(".", 1)[0] if "." in mod else ""
    ref = sys.modules.get(pkg + ".errors") if pkg else None
    if ref is not None and ref is not sys.modules[__name__] and \
            hasattr(ref, "NonConvergenceError"):
        return types.SimpleNamespace(**{k: getattr(ref, k, getattr(_OURS, k))
                                        for k in vars(_OURS)})
    return _OURS
