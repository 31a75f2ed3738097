"""Program identity: which corpus function a TypedProgram holds.

The backend runs exactly the corpus programs of the reference
(trident/corpus/programs/{sssp,sssp_pull,pr,bc,tc}.sp) on hand-written
kernels.  A reference ``TypedProgram`` is recognised structurally: the
reference's own ``to_sexpr`` dump (trident/syntax.py:303-320; spans and
sem_* annotations excluded) of the function's parameters and body is hashed
and looked up below (tools/make_fingerprints.py regenerates the table).
Anything else raises UnsupportedProgramError -- there is no CPU fallback.

``Program`` objects (``SSSP``, ``PR``, ...) can also be passed to ``run``
directly in place of a TypedProgram, e.g. where the reference frontend is
not installed (the GPU box).
"""

from __future__ import annotations

import hashlib
import sys
from dataclasses import dataclass

from .errors import UnsupportedProgramError

FINGERPRINTS = {
    "sssp": "0afbd6f73011e0255bec041c3f6375fe17202cf4f85e01e43c0ed2914cdaebdb",
    "sssp_pull": "b1490c6d27cd305c18eada7d4e9c327a25b8594b557f052a5ca6bd02b31c0732",
    "pr": "a33949c2ad8e09dc92baa40f5c8346ea342991540c9fd4e92d36dce2c2b48cdc",
    "bc": "fe91f9b5fbe40d6a1d2a0b614d162bfa9b09470fea4e1c9ce877ccfe999e7172",
    "tc": "28f098b022be174a0cb41954159d8d5a3d04b6bb473db20181a9ab7c7dca9aaa",
    "reduction": "08246c459994266f33ec2ab393b539a180995d24fc199b3e6e981ad69cd5325f",
}


@dataclass(frozen=True)
class Program:
    """A corpus program: its formals (name, kind) in declaration order and
    the fixedPoint flag it reports (None if it has no fixedPoint)."""

    key: str
    name: str
    params: tuple
    flag: str | None

    # TypedProgram-like surface so a Program can stand in for ``tp``
    def function(self, name=None):
        if name not in (None, self.name):
            raise KeyError(name)
        return self


SSSP = Program("sssp", "Compute_SSSP", (("g", "Graph"), ("src", "node")), "finished")
SSSP_PULL = Program("sssp_pull", "Compute_SSSP_Pull", (("g", "Graph"), ("src", "node")),
                    "finished")
PR = Program("pr", "Compute_PR", (("g", "Graph"), ("damping", "double"),
                                  ("epsilon", "double"), ("maxIter", "int")), "converged")
BC = Program("bc", "Compute_BC", (("g", "Graph"), ("sourceSet", "SetN")), None)
TC = Program("tc", "Compute_TC", (("g", "Graph"),), None)
# reduction.sp: the generic forall / neighbour-reduction shape (sp_forall.cu)
REDUCTION = Program("reduction", "Sum_Neighbor_Props", (("g", "Graph"),), None)

BY_KEY = {p.key: p for p in (SSSP, SSSP_PULL, PR, BC, TC, REDUCTION)}
_BY_PRINT = {v: BY_KEY[k] for k, v in FINGERPRINTS.items()}


def fingerprint(fn) -> str:
    """sha256 of the reference's structural dump of (params, body)."""
    mod = sys.modules.get(type(fn).__module__)
    to_sexpr = getattr(mod, "to_sexpr", None)
    if to_sexpr is None:
        raise UnsupportedProgramError(
            f"cannot fingerprint {type(fn).__name__}: its module has no to_sexpr")
    s = to_sexpr(fn.params) + "|" + to_sexpr(fn.body)
    return hashlib.sha256(s.encode()).hexdigest()


def identify(tp, function: str | None = None) -> Program:
    """Map (tp, function) to a corpus Program or raise."""
    if isinstance(tp, Program):
        return tp.function(function)
    if isinstance(tp, str):
        try:
            return BY_KEY[tp]
        except KeyError:
            raise UnsupportedProgramError(f"unknown corpus program {tp!r}") from None
    if getattr(tp, "key", None) == "forall":  # an already recognised ForallProgram
        return tp.function(function)
    fn = tp.function(function)  # KeyError for an unknown name, like interp.run
    prog = _BY_PRINT.get(fingerprint(fn))
    if prog is None:
        # not a corpus program: the generic forall / neighbour-reduction shape
        # (forall.py), or UnsupportedProgramError -- there is no CPU fallback
        from . import forall
        return forall.match(fn)
    return prog
