"""The generic forall / neighbour-reduction form (paper_2305_03317_b200/
forall.py): the matcher on programs parsed by the
reference's own frontend, and the semantics of the matched spec against
the reference interpreter's outputs (tests/golden/forall, written by
tests/golden/make_forall_golden.py) -- on the CPU through a NumPy model of
the spec (test infrastructure), on the GPU through the native kernel."""

import glob
import json
import os

import numpy as np
import pytest

from conftest import REPO  # noqa: F401
from paper_2305_03317_b200 import forall
from paper_2305_03317_b200.errors import UnsupportedProgramError

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FA = os.path.join(GOLD, "forall")
REF = "/root/reference/pkg/src"
PROGS = sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(FA, "*.json")))
GRAPHS = ["fx_rand200_a_d", "fx_rand200_b_u", "fx_star13_d", "fx_isolated4_d", "fx_grid5x5_u",
          "syn_rmat10_d", "syn_unif1k_u"]


def _spec(name):
    return forall.from_dict(json.load(open(os.path.join(FA, name + ".json"))))


def _model(spec, off, roff):
    """NumPy restatement of a matched spec (the rows' slot counts times the
    constant term; min/max where the row is non-empty)."""
    deg = np.diff(np.asarray(off))
    rdeg = np.diff(np.asarray(roff))
    props = {P: np.full(len(deg), v, dtype=np.int64 if t in ("int", "long") else np.float64)
             for P, (t, v) in spec.props.items()}
    scal = dict((A, v) for A, (t, v) in spec.scalars.items())
    for r in spec.reductions:
        c = r.term[1] if r.term[0] == "lit" else spec.props[r.term[1]][1]
        d = rdeg if r.reverse else deg
        if r.op == "+=":
            if r.target[0] == "prop":
                props[r.target[1]] = props[r.target[1]] + d * int(c)
            else:
                scal[r.target[1]] += int(d.sum()) * int(c)
        else:
            f = min if r.op == "Min" else max
            if r.target[0] == "prop":
                a = props[r.target[1]]
                a[d > 0] = np.array([f(x, c) for x in a[d > 0]], dtype=a.dtype)
            elif d.sum() > 0:
                scal[r.target[1]] = f(scal[r.target[1]], c)
    return props, scal


@pytest.mark.parametrize("name", PROGS)
def test_spec_model_matches_reference_goldens(name):
    spec = _spec(name)
    gold = np.load(os.path.join(FA, name + ".npz"))
    for gname in GRAPHS:
        z = np.load(os.path.join(GOLD, gname + ".npz"))
        props, scal = _model(spec, z["csr_off"], z["csr_roff"])
        for P, a in props.items():
            assert np.array_equal(a, gold[f"{gname}/prop/{P}"]), (gname, P)
        for A, v in scal.items():
            assert v == gold[f"{gname}/scalar/{A}"].item(), (gname, A)


def _reference():
    if not os.path.isdir(REF):
        pytest.skip("reference frontend not present")
    import sys
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from trident.parser import parse_source
    from trident.sema import analyze
    return parse_source, analyze


@pytest.mark.parametrize("name", PROGS)
def test_matcher_on_reference_ast(name):
    parse_source, analyze = _reference()
    tp = analyze(parse_source(open(os.path.join(FA, name + ".sp")).read()))
    from paper_2305_03317_b200 import corpus
    spec = corpus.identify(tp)
    assert spec.key == "forall"
    assert spec == _spec(name)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(FA, "rejected_*.sp"))))
def test_matcher_rejects_order_dependent_or_unsupported(path):
    parse_source, analyze = _reference()
    tp = analyze(parse_source(open(path).read()))
    from paper_2305_03317_b200 import corpus
    with pytest.raises(UnsupportedProgramError):
        corpus.identify(tp)


@pytest.mark.gpu
@pytest.mark.parametrize("name", PROGS)
def test_forall_kernel_matches_reference(name):
    import paper_2305_03317_b200 as sp
    spec = _spec(name)
    gold = np.load(os.path.join(FA, name + ".npz"))
    for gname in GRAPHS:
        z = np.load(os.path.join(GOLD, gname + ".npz"))
        g = sp.from_arrays(z["u"], z["v"], z["w"], directed=bool(z["directed"]), n=int(z["n"]))
        r = sp.run(spec, g, {})
        for P, a in r.env.node_props.items():
            assert np.array_equal(a, gold[f"{gname}/prop/{P}"]), (gname, P)
        for A, v in r.env.scalars.items():
            want = gold[f"{gname}/scalar/{A}"].item()
            assert v == want and type(v) is type(want), (gname, A, v, want)
        lists = sp.run(spec, g, {}, as_lists=True).env.node_props
        assert all(isinstance(x, list) for x in lists.values())
