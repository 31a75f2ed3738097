"""Host/device time breakdown of one PR call (GPU box diagnostic)."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_2305_03317_b200 as sp  # noqa: E402
from paper_2305_03317_b200 import _lib, corpus  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
g = sp.generate("rmat", scale, 16, seed=1)
args = {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}
for i in range(4):
    t0 = time.perf_counter()
    r = sp.run(corpus.PR, g, args, device_outputs=True)
    t1 = time.perf_counter()
    print(f"run(device_outputs) wall {(t1-t0)*1e3:.2f} ms  device {r.stats['device_ms']:.2f}"
          f"  iterations-kernels {r.stats['main_kernel_ms']:.2f}  iters {r.env.scalars['iter']}",
          flush=True)
L = _lib.lib()
rank = torch.empty(g.n, dtype=torch.float64, device="cuda")
it, its, diff, st = C.c_int64(), C.c_int64(), C.c_double(), _lib.Stats()
for i in range(3):
    t0 = time.perf_counter()
    rc = L.sp_pagerank(g.handle, 0.85, 1e-6, 100, 10 ** 9, 0, C.c_void_p(rank.data_ptr()), 1,
                       C.byref(it), C.byref(diff), C.byref(its), _lib.ITER_CB(), None, C.byref(st))
    t1 = time.perf_counter()
    print(f"native wall {(t1-t0)*1e3:.2f} ms  device {st.device_ms:.2f}  kernels "
          f"{st.main_kernel_ms:.2f}  rc {rc}", flush=True)

# per-step host overhead distribution of the bench's device-resident leg
import statistics  # noqa: E402
walls, devs = [], []
r = None
for i in range(60):
    t0 = time.perf_counter()
    r = sp.run(corpus.PR, g, args, device_outputs=True)
    walls.append((time.perf_counter() - t0) * 1e3)
    devs.append(r.stats["device_ms"])
gap = [w - d for w, d in zip(walls, devs)]
print("gap ms: median %.3f p90 %.3f max %.3f  device median %.3f" % (
    statistics.median(gap), sorted(gap)[54], max(gap), statistics.median(devs)))
print("gaps:", " ".join(f"{x:.2f}" for x in gap))
