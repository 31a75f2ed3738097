"""CPU-only tests of the boundary and host logic (no GPU calls).

* the C-ABI library loads and exports every symbol include/starplat_b200.h
  declares, and the ctypes table binds exactly those symbols;
* program identity: the structural fingerprints re-derive from the
  reference corpus (when the reference is importable here);
* argument checking, loader errors, partitioning and error classes match
  the reference's behaviour (compared against the reference when present);
* the host generators are deterministic and produce what they promise.
"""

import os
import re
import subprocess
import sys

import numpy as np
import pytest

from conftest import REPO

from paper_2305_03317_b200 import _lib, corpus, gen
from paper_2305_03317_b200 import graph as spg
from paper_2305_03317_b200 import interp as spi
from paper_2305_03317_b200.errors import (ArgError, ExecError, FormatError,
                                          GraphIoError, UnsupportedProgramError,
                                          errors_for)

REF = os.environ.get("TRIDENT_REF", "/root/reference/pkg/src")
HAVE_REF = os.path.isdir(os.path.join(REF, "trident"))


def header_symbols():
    txt = open(_lib.HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z_]+)\s*\(", txt)) - {"sp_iter_cb"})


def test_header_matches_ctypes_table():
    assert header_symbols() == sorted(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (sp_\w+)", out))
    missing = set(header_symbols()) - exported
    assert not missing, missing
    L = _lib.lib()  # binds every signature
    assert L.sp_abi_version() == _lib.ABI_VERSION == 8


def test_library_has_no_unresolved_internal_symbols():
    """Every internal (sp::) function the library calls is defined in it --
    a declaration whose definition landed in an anonymous namespace would
    only fail at dlopen on the GPU box."""
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    out = subprocess.run(["nm", "-D", "--undefined-only", _lib.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert not re.findall(r"_ZN2sp\w+", out)


def test_no_gpu_means_loud_failure():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        spg.from_edges([(0, 1)])


def test_oracle_not_imported_by_product():
    code = ("import sys; import paper_2305_03317_b200 as p; "
            "print(any(m == 'oracle' or m.startswith('oracle.') for m in sys.modules))")
    out = subprocess.run([sys.executable, "-c", code], cwd=REPO, capture_output=True,
                         text=True, check=True).stdout.strip()
    assert out == "False"
    for root, _, files in os.walk(os.path.join(REPO, "paper_2305_03317_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(root, f)).read()
                assert "import oracle" not in src and "from oracle" not in src
                assert "cpu_ref" not in src


# ---------------------------------------------------------------------------
# program identity


def test_identify_descriptors():
    assert corpus.identify(corpus.SSSP) is corpus.SSSP
    assert corpus.identify("pr") is corpus.PR
    assert corpus.identify("reduction") is corpus.REDUCTION
    with pytest.raises(UnsupportedProgramError):
        corpus.identify("bfs")


@pytest.mark.skipif(not HAVE_REF, reason="reference not importable here")
def test_fingerprints_rederive_from_reference():
    sys.path.insert(0, REF)
    from trident.parser import parse_source
    from trident.sema import analyze
    progs = os.path.join(REF, "trident", "corpus", "programs")
    for key in ("sssp", "sssp_pull", "pr", "bc", "tc", "reduction"):
        tp = analyze(parse_source(open(os.path.join(progs, key + ".sp")).read()))
        assert corpus.identify(tp) is corpus.BY_KEY[key]
        assert corpus.fingerprint(tp.function()) == corpus.FINGERPRINTS[key]
    # reformatting / renaming the function does not matter; changing code does
    src = open(os.path.join(progs, "tc.sp")).read()
    tp = analyze(parse_source(src.replace("Compute_TC", "MyTriangles").replace("  ", " ")))
    assert corpus.identify(tp) is corpus.TC
    tp = analyze(parse_source(src.replace("triangle_count += 1", "triangle_count += 2")))
    with pytest.raises(UnsupportedProgramError):
        corpus.identify(tp)
    red = open(os.path.join(progs, "reduction.sp")).read()
    tp = analyze(parse_source(red.replace("accum += nbr.prop", "accum += 2 * nbr.prop")))
    with pytest.raises(UnsupportedProgramError):
        corpus.identify(tp)
    with pytest.raises(KeyError):
        corpus.identify(tp, "nope")


@pytest.mark.skipif(not HAVE_REF, reason="reference not importable here")
def test_errors_follow_the_program_origin():
    sys.path.insert(0, REF)
    import trident.errors as te
    from trident.parser import parse_source
    from trident.sema import analyze
    progs = os.path.join(REF, "trident", "corpus", "programs")
    tp = analyze(parse_source(open(os.path.join(progs, "sssp.sp")).read()))
    E = errors_for(tp)
    assert E.NonConvergenceError is te.NonConvergenceError
    assert E.ExecError is te.ExecError
    assert errors_for(corpus.SSSP).ExecError is ExecError


class _FakeGraph:
    def __init__(self, n):
        self.n = n


@pytest.mark.skipif(not HAVE_REF, reason="reference not importable here")
@pytest.mark.parametrize("key,args", [
    ("sssp", {}), ("sssp", {"src": 7}), ("sssp", {"src": -1}), ("sssp", {"src": "3"}),
    ("pr", {"damping": 0.85, "epsilon": 1e-6}), ("pr", {"damping": "x", "epsilon": 1, "maxIter": 3}),
    ("bc", {"sourceSet": [0, 9]}), ("bc", {"sourceSet": [1, 1, 2]}), ("tc", {})])
def test_check_args_matches_reference(key, args):
    sys.path.insert(0, REF)
    from trident.graph import from_edges
    from trident.interp import check_args
    from trident.parser import parse_source
    from trident.sema import analyze
    progs = os.path.join(REF, "trident", "corpus", "programs")
    tp = analyze(parse_source(open(os.path.join(progs, key + ".sp")).read()))
    rg = from_edges([(0, 1), (1, 2), (2, 3), (3, 4)])
    try:
        want = check_args(tp.info(), rg, args)
        want = {k: v for k, v in want.items() if k != "g"}
        werr = None
    except Exception as e:  # noqa: BLE001
        werr = (type(e).__name__, str(e))
    try:
        got = spi.check_args(corpus.BY_KEY[key], _FakeGraph(rg.n), args, errors_for(tp))
        gerr = None
    except Exception as e:  # noqa: BLE001
        gerr = (type(e).__name__, str(e))
    if werr is None:
        assert gerr is None and got == want
    else:
        assert gerr == werr


# ---------------------------------------------------------------------------
# loader errors (raised before any device work)


@pytest.mark.parametrize("text,lineno,msg", [
    ("0 1\n1 x\n", 2, "non-integer field"),
    ("# c\n\n0 1 2 3\n", 3, "expected 2 or 3 fields, got 4"),
    ("0 -1\n", 1, "negative vertex id"),
    ("5\n", 1, "expected 2 or 3 fields, got 1"),
])
def test_loader_format_errors(tmp_path, text, lineno, msg):
    p = tmp_path / "g.txt"
    p.write_text(text)
    with pytest.raises(FormatError) as ei:
        spg.load_edge_list(str(p))
    assert ei.value.lineno == lineno and msg in str(ei.value)
    if HAVE_REF:
        sys.path.insert(0, REF)
        from trident.errors import FormatError as RFE
        from trident.graph import load_edge_list
        with pytest.raises(RFE) as er:
            load_edge_list(str(p))
        assert str(er.value) == str(ei.value)


_TRICKY = [
    b"0 1\r\n1 2\r\n2 x\r\n",                    # CRLF, error on line 3
    b"0 1\r1 2\r-3 4\r",                           # bare CR terminators
    b"0 1\n\r\n1 2 3 4\n",                         # \n then \r\n: line 3
    b"  # comment\n\t\n0\t1\x0b\n1 1_0\n2 1__0\n",  # \v whitespace, underscores
    b"0 1\n2 _3\n",
    b"0 1\n3_ 4\n",
    b"0 1\n+\n",
    b"0 +1 -2\n1 2 0x10\n",
    b"0 1 2\n1.5 2\n",
    b"0 1\n\x0c\x1c\n5 -0\n-0 3\n 7\n",           # \f, \x1c whitespace; -0 is 0
    b"0 1 99999999999999999999\n1 2 x\n",           # huge weight parses, then error
    b"0 1",                                          # no final newline, valid
]


@pytest.mark.parametrize("k", range(len(_TRICKY)))
def test_native_parser_errors_match_reference(tmp_path, k):
    """The native parser raises FormatError on the same line with the same
    message as the reference (or parses the file the reference accepts)."""
    p = tmp_path / "g.txt"
    p.write_bytes(_TRICKY[k])
    ours = ref = None
    try:
        spg.load_edge_list(str(p))
    except FormatError as e:
        ours = str(e)
    except (RuntimeError, ArgError):
        ours = "parsed"  # no GPU here (or out of int32 range): the text parsed
    if not HAVE_REF:
        return
    sys.path.insert(0, REF)
    from trident.errors import FormatError as RFE
    from trident.graph import load_edge_list
    try:
        load_edge_list(str(p))
        ref = "parsed"
    except RFE as e:
        ref = str(e)
    assert ours == ref


def test_native_parser_multithreaded_error_line(tmp_path):
    """A > 1 MiB file is cut into per-thread parts; the reported line is the
    global first failing line."""
    good = "".join(f"{i} {i + 1} {i % 7}\n" for i in range(120000))
    text = "# header\n" + good + "12 oops\n" + good + "bad line here now\n"
    p = tmp_path / "big.txt"
    p.write_text(text)
    with pytest.raises(FormatError) as ei:
        spg.load_edge_list(str(p))
    assert ei.value.lineno == 1 + 120000 + 1
    assert "non-integer field in '12 oops'" in str(ei.value)


def test_loader_io_error(tmp_path):
    with pytest.raises(GraphIoError):
        spg.load_edge_list(str(tmp_path / "missing.txt"))


def test_from_arrays_rejects_out_of_domain():
    with pytest.raises(ArgError):
        spg.from_arrays([0], [1], [2 ** 31])
    with pytest.raises(ArgError):
        spg.from_arrays([-1], [1], [1])


# ---------------------------------------------------------------------------
# partitioning (graph.py:193-249)


def test_block_partition_spec_examples():
    parts = spg.block_partition(_FakeGraph(10), 3)
    assert [(p.local_begin, p.local_end, p.padded) for p in parts] == \
        [(0, 4, 0), (4, 8, 0), (8, 12, 2)]
    assert [p.real_range() for p in parts] == [range(0, 4), range(4, 8), range(8, 10)]
    assert [(p.local_begin, p.local_end) for p in spg.block_partition(_FakeGraph(4), 4)] == \
        [(0, 1), (1, 2), (2, 3), (3, 4)]
    with pytest.raises(ArgError):
        spg.block_partition(_FakeGraph(4), 0)
    assert [spg.owner_of(v, 3, 10) for v in range(10)] == [0] * 4 + [1] * 4 + [2] * 2


@pytest.mark.skipif(not HAVE_REF, reason="reference not importable here")
@pytest.mark.parametrize("n,k", [(10, 3), (0, 2), (7, 7), (5, 8), (1000, 7)])
def test_block_partition_matches_reference(n, k):
    sys.path.insert(0, REF)
    from trident.graph import block_partition, owner_of
    ref = block_partition(_FakeGraph(n), k)
    ours = spg.block_partition(_FakeGraph(n), k)
    assert [(p.rank, p.local_begin, p.local_end, p.padded) for p in ref] == \
        [(p.rank, p.local_begin, p.local_end, p.padded) for p in ours]
    if n:
        assert [owner_of(v, k, n) for v in range(n)] == [spg.owner_of(v, k, n) for v in range(n)]


# ---------------------------------------------------------------------------
# host generators


def test_generators_deterministic_and_clean():
    u1, v1, w1, n = gen.rmat(10, 16, seed=3)
    u2, v2, w2, _ = gen.rmat(10, 16, seed=3)
    assert (u1 == u2).all() and (v1 == v2).all() and (w1 == w2).all()
    assert n == 1024 and (u1 != v1).all()
    key = u1.astype(np.int64) << 32 | v1
    assert (np.diff(key) > 0).all()  # sorted, unique
    assert w1.min() >= 1 and w1.max() <= 100
    deg = np.bincount(u1, minlength=n)
    assert deg[0] == deg.max()  # no relabel: vertex 0 is the hub
    us, vs, ws, _ = gen.rmat(10, 16, seed=3, undirected=True)
    assert (us < vs).all()
    uu, vu, wu, nu = gen.uniform(4096, 20000, seed=1)
    assert (uu < vu).all() and len(uu) > 19900
    ug, vg, wg, ng = gen.grid(3, 4, seed=1)
    assert ng == 12 and len(ug) == 3 * 3 + 2 * 4


def test_rmat_thresholds():
    assert gen.rmat_thresholds() == (37356, 37356 + 12452, 37356 + 2 * 12452)


WEIGHT_CASES = sorted(f[:-4] for f in os.listdir(os.path.join(REPO, "tests", "golden", "weights"))
                      if f.endswith(".npz"))


@pytest.mark.parametrize("case", WEIGHT_CASES)
def test_random_weights_match_reference_golden(case):
    """assign_random_weights' draw order (graph.py:154-190) against weights
    the reference itself assigned (tests/golden/make_weights_golden.py):
    directed per slot; undirected per canonical slot, mirrored by position
    onto parallel copies; self-loops drawn once."""
    z = np.load(os.path.join(REPO, "tests", "golden", "weights", case + ".npz"))
    w = spg.random_weights(z["off"], z["adj"], bool(z["directed"]), int(z["lo"]), int(z["hi"]),
                           int(z["seed"]))
    np.testing.assert_array_equal(w, z["w"])


def test_random_weights_range_error():
    with pytest.raises(spg.RangeError):
        spg.random_weights(np.zeros(1, np.int64), np.zeros(0, np.int32), True, 5, 1, 0)
