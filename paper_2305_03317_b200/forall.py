"""Generic forall / neighbour-reduction programs.

The reference executes any typed program with its tree-walking
interpreter (trident/interp.py); the B200 backend has hand-written kernels
for the corpus programs and, for the *shape* of corpus/programs/
reduction.sp, this generic form: a program is accepted when its AST (the
reference's own ``trident.syntax`` nodes, matched by class name) is

    function F(Graph g) {
      propNode<T> P, ...;  g.attachNodeProperty(P = <literal>, ...);
      T2 A = <literal>; ...                       // function-level scalars
      forall (v in g.nodes()) {                   // no filter
        <T3 local = <literal>;> ...               // forall-locals (not results)
        forall (u in g.neighbors(v) | g.nodesTo(v)) {   // no filter; one or more
          A += term;  v.Q += term;  A++;  v.Q++;
          <A> = <Min|Max(A, term)>;  <v.Q> = <Min|Max(v.Q, term)>;
          local += ...;  local++;                 // ignored: locals are not results
        }
      }
    }

with ``term`` a literal, ``u.P`` or ``v.P`` where P is a property no
reduction writes (so every slot's term is the constant P was attached
with).  Every such reduction is order-independent (integer sums; min / max
in any type), so the GPU result equals the reference's sequential loop bit
for bit.  Each reduction runs one ``sp_neighbor_reduce`` kernel over the
rows (interp.py:347-359 semantics for ``+=`` / ``++``, interp.py:401-421 for
Min/Max).  ``+=`` on a float/double target is order-dependent and is
rejected (UnsupportedProgramError), as is anything else outside the shape.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import UnsupportedProgramError

_INT_TYPES = ("int", "long")
_NUM_TYPES = ("int", "long", "float", "double")


@dataclass(frozen=True)
class Reduction:
    target: tuple   # ("scalar", A) | ("prop", Q)
    op: str         # "+=" | "Min" | "Max"
    term: tuple     # ("lit", value) | ("prop", P)
    reverse: bool   # nodesTo(v) rows


@dataclass
class ForallProgram:
    """A recognised program of the shape above (a Program-like object:
    ``key``, ``name``, ``params``, ``flag``)."""
    name: str
    props: dict = field(default_factory=dict)    # P -> (type name, initial value)
    scalars: dict = field(default_factory=dict)  # A -> (type name, initial value)
    reductions: list = field(default_factory=list)
    key: str = "forall"
    params: tuple = (("g", "Graph"),)
    flag: str | None = None

    def function(self, name=None):
        if name not in (None, self.name):
            raise KeyError(name)
        return self


def _cls(x) -> str:
    return type(x).__name__


def _typename(t) -> str | None:
    """'int'/'long'/'float'/'double'/'bool' of a PrimType or PropNodeType."""
    for attr in ("name", "kind", "prim"):
        v = getattr(t, attr, None)
        if isinstance(v, str):
            return v
    elem = getattr(t, "elem", None) or getattr(t, "elem_type", None)
    if elem is not None:
        return _typename(elem)
    s = str(t)
    for n in ("double", "float", "long", "int", "bool"):
        if n in s:
            return n
    return None


def _literal(e):
    if _cls(e) != "Literal":
        return None
    return e.value


def _fail(why: str):
    raise _NoMatch(why)


class _NoMatch(Exception):
    pass


def match(fn) -> ForallProgram:
    """ForallProgram for a reference Function AST of the shape above, else
    UnsupportedProgramError."""
    try:
        return _match(fn)
    except _NoMatch as e:
        raise UnsupportedProgramError(
            f"function '{getattr(fn, 'name', '?')}' is neither a corpus program nor a "
            f"neighbour reduction the generic forall kernel runs ({e}); there is no CPU "
            "fallback") from None


def _match(fn) -> ForallProgram:
    params = list(getattr(fn, "params", []))
    if len(params) != 1 or _cls(params[0].dsl_type) != "GraphType":
        _fail("parameters other than (Graph g)")
    g = params[0].name
    prog = ForallProgram(name=fn.name)
    declared_props = {}
    outer_seen = False
    for s in fn.body.stmts:
        c = _cls(s)
        if c == "DeclStmt" and _cls(s.dsl_type) == "PropNodeType":
            declared_props[s.name] = _typename(s.dsl_type)
        elif c == "DeclStmt" and _cls(s.dsl_type) == "PrimType":
            t = _typename(s.dsl_type)
            v = _literal(s.init) if s.init is not None else 0
            if t not in _NUM_TYPES or v is None or outer_seen:
                _fail(f"scalar '{s.name}'")
            prog.scalars[s.name] = (t, v)
        elif c == "ExprStmt" and _cls(s.expr) == "ProcCall" and \
                s.expr.method == "attachNodeProperty" and _cls(s.expr.receiver) == "Identifier" \
                and s.expr.receiver.name == g:
            for a in s.expr.args:
                v = _literal(a.value)
                if a.name not in declared_props or v is None:
                    _fail(f"attachNodeProperty({a.name})")
                prog.props[a.name] = (declared_props[a.name], v)
        elif c == "ForallStmt" and not outer_seen:
            outer_seen = True
            _match_outer(prog, s, g)
        else:
            _fail(f"statement {c}")
    if not outer_seen:
        _fail("no forall over g.nodes()")
    for P in declared_props:
        if P not in prog.props:
            _fail(f"property '{P}' is never attached")
    written = {r.target[1] for r in prog.reductions if r.target[0] == "prop"}
    for r in prog.reductions:
        if r.term[0] == "prop" and r.term[1] in written:
            _fail(f"a term reads '{r.term[1]}', which the loop writes")
        ttype = (prog.scalars if r.target[0] == "scalar" else prog.props)[r.target[1]][0]
        if r.op == "+=" and ttype not in _INT_TYPES:
            _fail(f"'+=' on {ttype} '{r.target[1]}' (order-dependent)")
        if ttype not in _NUM_TYPES:
            _fail(f"target type {ttype}")
    return prog


def _range(e, g, it=None):
    """('nodes',) / ('neighbors'|'nodesTo', arg) of g.<method>(...)"""
    if _cls(e) != "ProcCall" or _cls(e.receiver) != "Identifier" or e.receiver.name != g:
        return None
    if e.method == "nodes" and not e.args:
        return ("nodes",)
    if e.method in ("neighbors", "nodesTo") and len(e.args) == 1 and \
            _cls(e.args[0].value) == "Identifier" and e.args[0].value.name == it:
        return (e.method,)
    return None


def _match_outer(prog, s, g):
    if s.filter is not None or _range(s.range_call, g) != ("nodes",):
        _fail("outer forall is not over g.nodes() without a filter")
    v = s.iterator
    locals_ = set()
    inner = 0
    for t in s.body.stmts:
        c = _cls(t)
        if c == "DeclStmt" and _cls(t.dsl_type) == "PrimType":
            if t.init is not None and _literal(t.init) is None:
                _fail(f"local '{t.name}'")
            locals_.add(t.name)
        elif c == "ForallStmt":
            rng = _range(t.range_call, g, v)
            if t.filter is not None or rng is None or rng[0] == "nodes":
                _fail("inner forall is not over g.neighbors(v) / g.nodesTo(v)")
            inner += 1
            _match_inner(prog, t, v, locals_, rng[0] == "nodesTo")
        else:
            _fail(f"outer-loop statement {c}")
    if not inner:
        _fail("no inner forall")


def _target(e, v, prog, locals_):
    if _cls(e) == "Identifier":
        if e.name in locals_:
            return ("local", e.name)
        if e.name in prog.scalars:
            return ("scalar", e.name)
    if _cls(e) == "MemberAccess" and _cls(e.obj) == "Identifier" and e.obj.name == v and \
            e.prop in prog.props:
        return ("prop", e.prop)
    _fail("reduction target")


def _term(e, v, u, prog):
    lit = _literal(e)
    if lit is not None:
        return ("lit", lit)
    if _cls(e) == "MemberAccess" and _cls(e.obj) == "Identifier" and e.obj.name in (v, u) \
            and e.prop in prog.props:
        return ("prop", e.prop)
    _fail("term is not a literal, u.P or v.P")


def _match_inner(prog, t, v, locals_, reverse):
    u = t.iterator
    for r in t.body.stmts:
        c = _cls(r)
        if c == "ReductionAssign" and r.op in ("+=", "++"):
            tgt = _target(r.lvalue, v, prog, locals_)
            if tgt[0] == "local":
                continue  # forall-locals are not part of the result
            term = ("lit", 1) if r.op == "++" else _term(r.expr, v, u, prog)
            prog.reductions.append(Reduction(tgt, "+=", term, reverse))
        elif c == "MinMaxAssign" and len(r.targets) == 1 and not r.companions:
            tgt = _target(r.targets[0], v, prog, locals_)
            if tgt[0] == "local":
                continue
            first = _target(r.first, v, prog, locals_) if r.first is not None else tgt
            if first != tgt:
                _fail("Min/Max whose first argument is not its target")
            prog.reductions.append(Reduction(tgt, r.op, _term(r.candidate, v, u, prog), reverse))
        else:
            _fail(f"inner-loop statement {c}")


def _value(prog, term):
    return term[1] if term[0] == "lit" else prog.props[term[1]][1]


def _np_type(t):
    return np.int64 if t in _INT_TYPES or t == "bool" else np.float64


def execute(prog: ForallProgram, dg, mem_host=True):
    """Run the reductions on the device graph; -> (node_props, scalars, stats)."""
    L = _lib.lib()
    n = dg.n
    props = {P: np.full(n, v, dtype=_np_type(t)) for P, (t, v) in prog.props.items()}
    scalars = {A: v for A, (t, v) in prog.scalars.items()}
    stats = {"kernel_launches": 0, "device_ms": 0.0, "edges_visited": 0}
    for r in prog.reductions:
        c = _value(prog, r.term)
        st = _lib.Stats()
        want_pv = r.target[0] == "prop"
        if r.op == "+=":
            if not float(c).is_integer():
                raise UnsupportedProgramError("'+=' of a non-integral term")
            pv = np.empty(max(1, n), dtype=np.int64) if want_pv else None
            tot = C.c_int64()
            rc = L.sp_neighbor_reduce(dg.handle, _lib.SP_REDUCE_SUM_I64, int(r.reverse), int(c),
                                      0.0, None, _lib.SP_MEM_HOST,
                                      pv.ctypes.data_as(C.c_void_p) if want_pv else None,
                                      C.byref(tot), C.byref(st))
            _check(rc)
            if want_pv:
                props[r.target[1]] = props[r.target[1]] + pv[:n]
            else:
                scalars[r.target[1]] = scalars[r.target[1]] + int(tot.value)
        else:
            op = _lib.SP_REDUCE_MIN_F64 if r.op == "Min" else _lib.SP_REDUCE_MAX_F64
            pv = np.empty(max(1, n), dtype=np.float64) if want_pv else None
            tot = C.c_double()
            rc = L.sp_neighbor_reduce(dg.handle, op, int(r.reverse), 0, float(c), None,
                                      _lib.SP_MEM_HOST,
                                      pv.ctypes.data_as(C.c_void_p) if want_pv else None,
                                      C.byref(tot), C.byref(st))
            _check(rc)
            f = np.minimum if r.op == "Min" else np.maximum
            if want_pv:
                cur = props[r.target[1]]
                got = pv[:n]
                has = np.isfinite(got)  # rows with at least one slot
                cur[has] = f(cur[has], got[has].astype(cur.dtype))
            elif np.isfinite(tot.value):
                t = prog.scalars[r.target[1]][0]
                best = f(scalars[r.target[1]], tot.value)
                scalars[r.target[1]] = int(best) if t in _INT_TYPES else float(best)
        stats["kernel_launches"] += st.kernel_launches
        stats["device_ms"] += st.device_ms
        stats["edges_visited"] += st.edges_visited
    for A, (t, _) in prog.scalars.items():  # reference value types
        scalars[A] = int(scalars[A]) if t in _INT_TYPES else float(scalars[A])
    return props, scalars, stats


def _check(rc):
    if rc != _lib.SP_OK:
        raise RuntimeError(f"sp_neighbor_reduce failed ({rc}): {_lib.last_error()}")


def from_dict(d: dict) -> ForallProgram:
    """A ForallProgram from its dataclasses.asdict() / JSON form (the golden
    fixtures carry the matched spec, so the GPU tests need no frontend)."""
    return ForallProgram(
        name=d["name"],
        props={k: (v[0], v[1]) for k, v in d["props"].items()},
        scalars={k: (v[0], v[1]) for k, v in d["scalars"].items()},
        reductions=[Reduction(tuple(r["target"]), r["op"], tuple(r["term"]), bool(r["reverse"]))
                    for r in d["reductions"]])
