"""PR layout A/B on the GPU box: relabelled (SP_PR_REL=1) vs hot-encoded
(SP_PR_REL=0) device time per run, RMAT scales from argv."""
import os
import statistics
import sys

sys.path.insert(0, '.')
import paper_2305_03317_b200 as sp  # noqa: E402
from paper_2305_03317_b200 import corpus  # noqa: E402

args = {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}
for scale in [int(x) for x in (sys.argv[1:] or ["22", "24"])]:
    for rel in ("1", "0"):
        os.environ["SP_PR_REL"] = rel
        g = sp.generate("rmat", scale, 16, seed=1)
        t = []
        for i in range(7):
            r = sp.run(corpus.PR, g, args, device_outputs=True)
            if i >= 2:
                t.append(r.stats["device_ms"])
        it = r.env.scalars["iter"]
        print(f"rmat{scale} rel={rel} iters {it} device ms median {statistics.median(t):.3f} "
              f"min {min(t):.3f}  per-iter {statistics.median(t) / it:.4f}  "
              f"frac {(12 * g.m + 36 * g.n) * it / (statistics.median(t) / 1e3) / 6470.5e9:.3f}",
              flush=True)
        g.close()
