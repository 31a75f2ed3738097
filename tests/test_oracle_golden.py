"""Pin the CPU oracle (oracle/cpu_ref.c) to the Python reference's own outputs
(tests/golden/*.npz, written by tests/golden/make_golden.py running
trident.graph / trident.interp.run).  Everything here is bit-exact,
including fixedPoint iteration counts: the oracle restates the
interpreter's sequential semantics exactly."""

import numpy as np
import pytest

from conftest import golden_cases, load_golden
from oracle import cpu_ref

CASES = golden_cases()


def _csr(z):
    return cpu_ref.build_csr(z["u"], z["v"], z["w"], bool(z["directed"]),
                             n=int(z["n"]))


@pytest.mark.parametrize("case", CASES)
def test_csr_matches_reference(case):
    z = load_golden(case)
    g = _csr(z)
    assert g.n == int(z["n"])
    np.testing.assert_array_equal(g.off, z["csr_off"])
    np.testing.assert_array_equal(g.adj, z["csr_adj"])
    np.testing.assert_array_equal(g.w, z["csr_w"])
    np.testing.assert_array_equal(g.roff, z["csr_roff"])
    np.testing.assert_array_equal(g.radj, z["csr_radj"])
    np.testing.assert_array_equal(g.reid, z["csr_reid"])


@pytest.mark.parametrize("case", CASES)
def test_sssp_matches_reference(case):
    z = load_golden(case)
    g = _csr(z)
    for i, s in enumerate(z["sssp_srcs"]):
        dist, iters, rc = cpu_ref.sssp(g, int(s))
        assert rc == 0
        np.testing.assert_array_equal(dist.astype(np.int64), z["sssp_dist"][i])
        assert iters == int(z["sssp_iters"][i])


@pytest.mark.parametrize("case", CASES)
def test_pagerank_matches_reference(case):
    z = load_golden(case)
    g = _csr(z)
    cap_err = int(z["pr_err_cap"])
    rank, it, diff, its, rc = cpu_ref.pagerank(g, 0.85, 1e-6, 100)
    if cap_err >= 0:
        assert rc == 1 and its == cap_err
        rank, it, diff, its, rc = cpu_ref.pagerank(g, 0.85, 1e-6, 100, cap=10 ** 6)
    assert rc == 0
    assert rank.tobytes() == z["pr_rank"].tobytes()      # bit-exact
    assert rank.tobytes() == z["pr_rank_nxt"].tobytes()
    assert it == int(z["pr_iter"]) and its == int(z["pr_iters"])
    assert diff == float(z["pr_diff"])


@pytest.mark.parametrize("case", CASES)
def test_pagerank_threads_bit_identical(case):
    z = load_golden(case)
    g = _csr(z)
    r1 = cpu_ref.pagerank(g, cap=10 ** 6, nthreads=1)
    r4 = cpu_ref.pagerank(g, cap=10 ** 6, nthreads=4)
    assert r1[0].tobytes() == r4[0].tobytes() and r1[1:] == r4[1:]


@pytest.mark.parametrize("case", CASES)
def test_bc_matches_reference(case):
    z = load_golden(case)
    g = _csr(z)
    srcs = z["bc_srcs"]
    for nt in (1, 3):
        bc, sg, dl = cpu_ref.bc(g, srcs, nthreads=nt)
        assert bc.tobytes() == z["bc"].tobytes()
        if len(srcs):
            assert sg.tobytes() == z["bc_sigma"].tobytes()
            assert dl.tobytes() == z["bc_delta"].tobytes()


@pytest.mark.parametrize("case", CASES)
def test_tc_matches_reference(case):
    z = load_golden(case)
    g = _csr(z)
    assert cpu_ref.tc(g) == int(z["tc"])
    assert cpu_ref.tc(g, nthreads=4) == int(z["tc"])


def test_dijkstra_oracle_matches_reference_sssp_goldens():
    """cr_sssp_dijkstra (trident/oracles.py:23-40 over w_eff) gives the
    reference interpreter's SSSP distances on every non-negative golden case
    (it certifies the cfg5a grid, where the interpreter-order oracle would
    need ~10^4 sweeps)."""
    import glob
    import os
    checked = 0
    for f in sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz"))):
        z = np.load(f)
        if "sssp_dist" not in z:
            continue
        o = cpu_ref.build_csr(z["u"], z["v"], z["w"], bool(z["directed"]), int(z["n"]))
        if (o.weff < 0).any():
            continue
        for i, s in enumerate(z["sssp_srcs"]):
            d, rc = cpu_ref.sssp_dijkstra(o, int(s))
            assert rc == 0
            np.testing.assert_array_equal(d, z["sssp_dist"][i])
            checked += 1
    assert checked >= 50
