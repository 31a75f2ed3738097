"""Golden vectors for the generic forall / neighbour-reduction programs
(paper_2305_03317_b200/forall.py), produced by the REFERENCE interpreter.

For every tests/golden/forall/*.sp program the reference frontend
(trident.parser / trident.sema) builds the typed program, our matcher turns
it into a ForallProgram spec (saved as JSON, so the GPU tests need no
reference), and trident.interp.run executes it on a set of golden graphs;
node properties and scalars are saved per graph.  Test infrastructure
only.  usage: python tests/golden/make_forall_golden.py [--ref /root/reference/pkg/src]
"""
import argparse
import dataclasses
import glob
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
GRAPHS = ["fx_rand200_a_d", "fx_rand200_b_u", "fx_star13_d", "fx_isolated4_d", "fx_grid5x5_u",
          "syn_rmat10_d", "syn_unif1k_u"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    a = ap.parse_args()
    sys.path.insert(0, a.ref)
    sys.path.insert(0, REPO)
    from trident.graph import CsrGraph
    from trident.interp import run
    from trident.parser import parse_source
    from trident.sema import analyze

    from paper_2305_03317_b200 import forall
    for path in sorted(glob.glob(os.path.join(HERE, "forall", "*.sp"))):
        name = os.path.basename(path)[:-3]
        if name.startswith("rejected_"):
            continue
        tp = analyze(parse_source(open(path).read()))
        spec = forall.match(tp.function(None))
        out = {}
        for gname in GRAPHS:
            z = np.load(os.path.join(HERE, gname + ".npz"))
            g = CsrGraph(n=len(z["csr_off"]) - 1, m=len(z["csr_adj"]), offsets=z["csr_off"].tolist(),
                         adj=z["csr_adj"].tolist(), weights=z["csr_w"].tolist(),
                         rev_offsets=z["csr_roff"].tolist(), rev_adj=z["csr_radj"].tolist(),
                         rev_eid=z["csr_reid"].tolist(), directed=bool(z["directed"]))
            r = run(tp, g, {})
            for k, v in r.env.node_props.items():
                out[f"{gname}/prop/{k}"] = np.asarray(v)
            for k, v in r.env.scalars.items():
                out[f"{gname}/scalar/{k}"] = np.asarray(v)
        np.savez_compressed(os.path.join(HERE, "forall", name + ".npz"), **out)
        d = dataclasses.asdict(spec)
        json.dump(d, open(os.path.join(HERE, "forall", name + ".json"), "w"), indent=1,
                  default=list)
        print(name, len(out), "arrays")


if __name__ == "__main__":
    main()
