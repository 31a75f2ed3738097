#!/usr/bin/env python3
"""Benchmark driver (one JSON line on rank 0).

Headline workload = BASELINE.json configs[1]: PageRank (d=0.85, eps=1e-6,
maxIter=100) on RMAT scale-22 (edge factor 16, seed 1, deduplicated, no
self-loops), metric GTEPS = iterations * m / time.  A "step" is one full
``pr.sp`` run to convergence on the device-resident graph.
  value : device-timed (CUDA events), graph already in HBM, ranks left in
          HBM (run(..., device_outputs=True)).
  e2e   : through the public API with host buffers every step: pinned host
          CSR -> sp.from_csr (H2D + on-device reverse CSR) -> sp.run(PR) ->
          ranks back to host.  This is the paper's CUDA timing convention
          (times include CPU<->GPU transfer).
  roofline : one PR iteration (k_pr_units + k_pr_fix + k_pr_epi, bracketed
          by CUDA events on the call's stream), algorithmic bytes 12 m + 36 n
           / its mean duration, against MEASURED_PEAKS.json
          hbm_gbs.
  cpu_baseline : the CPU oracle port (oracle/cpu_ref.c, OpenMP on all host
          threads) on a bounded sample of the same workload.
  algorithms : the other BASELINE configs at one GPU (SSSP cfg1, BC cfg4
          with 256 sources, TC cfg3), each with GTEPS and its roofline.
N > 1 (torchrun, one process per GPU): PR is block-partitioned
(graph.py:226-249 ownership); every iteration each rank updates its own
vertex block and the contrib slices are exchanged with an NCCL all-gather
(the reference's remote-read snapshot, bsp.py:182-185/287-288), diff with an
all-reduce(max).  Total work is fixed -> "strong" scaling.

--impl reference: the reference's algorithm on the host CPU (the oracle
port; the Python interpreter itself needs hours for this config, F6).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

BASELINE_METRIC = "GTEPS per algorithm (SSSP/PR/BC/TC) at 1/2/4/8 B200; % of HBM roofline"
PR_ARGS = {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}
SCALE, EF, SEED = 22, 16, 1


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kernel: str):
    """dram bytes per launch from the committed ncu summary, if any."""
    path = os.path.join(REPO, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        busy = [float(s[0]) for s in self.samples
                if s[0].replace(".", "").isdigit() and s[6].isdigit() and int(s[6]) > 0]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower() == "active"})
        use = busy or sm
        return {"sm_mhz": statistics.median(use) if use else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_pr_sample(off, roff, radj, n, m, budget_s=12.0, nthreads=None):
    """Oracle PR (OpenMP) on the full graph for a bounded number of
    iterations; returns (GTEPS, iterations, seconds, threads)."""
    from oracle import cpu_ref
    nt = nthreads or os.cpu_count() or 1
    g = cpu_ref.Csr(n, m, True, off, None, None, roff, radj, None, None)
    t0 = time.perf_counter()
    cpu_ref.pagerank(g, 0.85, 1e-6, 1, cap=10 ** 6, nthreads=nt)
    t1 = time.perf_counter() - t0
    k = int(max(1, min(20, budget_s / max(t1, 1e-3))))
    t0 = time.perf_counter()
    _, it, _, _, _ = cpu_ref.pagerank(g, 0.85, 1e-6, k, cap=10 ** 6, nthreads=nt)
    dt = time.perf_counter() - t0
    return it * m / dt / 1e9, it, dt, nt


# ---------------------------------------------------------------------------
# reference arm


def run_reference(a):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import cpu_ref
    from paper_2305_03317_b200 import gen
    u, v, w, n = gen.rmat(SCALE, EF, seed=SEED)
    o = cpu_ref.build_csr(u, v, w, True, n)
    del u, v, w
    nt = os.cpu_count() or 1
    # each step: a bounded sample of PR iterations on the full cfg2 graph
    _, _, t1, _ = cpu_pr_sample(o.off, o.roff, o.radj, o.n, o.m, budget_s=0.0, nthreads=nt)
    k = int(max(1, min(10, 20.0 / max(1, a.steps + a.warmup) / max(t1, 1e-3))))
    vals = []
    times = []
    for s in range(a.warmup + a.steps):
        t0 = time.perf_counter()
        _, it, _, _, _ = cpu_ref.pagerank(o, 0.85, 1e-6, k, cap=10 ** 6, nthreads=nt)
        dt = time.perf_counter() - t0
        if s >= a.warmup:
            vals.append(it * o.m / dt / 1e9)
            times.append(dt)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": BASELINE_METRIC, "value": value, "unit": "GTEPS",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1e3 * statistics.median(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic RMAT-{SCALE} ef{EF} seed {SEED} (host generator)",
        "config": {"workload": "pagerank_rmat22", "n": o.n, "m": o.m, **PR_ARGS,
                   "sample_iterations_per_step": k},
        "cpu_baseline": {"value": value, "unit": "GTEPS", "cores": nt, "kind": "port",
                         "sample": f"{k} PR iterations of cfg2 (full RMAT-22 graph) per step, "
                                   f"oracle/cpu_ref.c OpenMP x{nt}"},
        "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm


def run_ours(a):
    import torch
    import torch.distributed as dist

    import paper_2305_03317_b200 as sp
    from paper_2305_03317_b200 import _lib, corpus

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    hbm_peak, peak_kind = peaks()

    g = sp.generate("rmat", SCALE, EF, seed=SEED, undirected=False, device=local)
    n, m = g.n, g.m
    bytes_pull = 12 * m + 36 * n

    result = {}
    with ClockSampler(local) as clk:
        if world == 1:
            # warmup + timed steps (device-resident)
            for _ in range(a.warmup):
                sp.run(corpus.PR, g, PR_ARGS, device_outputs=True)
            torch.cuda.synchronize()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record()
            t_wall0 = time.perf_counter()
            main_ms = 0.0
            main_launches = launches = 0
            dev_ms = []
            for _ in range(a.steps):
                r = sp.run(corpus.PR, g, PR_ARGS, device_outputs=True)
                st = r.stats
                dev_ms.append(st["device_ms"])
                main_ms += st["main_kernel_ms"]
                main_launches += st["main_kernel_launches"]
                launches += st["kernel_launches"]
            ev1.record()
            torch.cuda.synchronize()
            t_wall = time.perf_counter() - t_wall0
            iters = r.env.scalars["iter"]
            # K steps bracketed by CUDA events after a device sync on both sides;
            # each call runs on its own stream and syncs before returning, so
            # this span holds all device work plus the per-iteration host reads
            total_ms = ev0.elapsed_time(ev1)
            result.update(iters=iters, total_ms=total_ms, wall_s=t_wall, main_ms=main_ms,
                          main_launches=main_launches, launches=launches,
                          call_device_ms=sum(dev_ms))
        else:
            total_ms, iters, launches, main_ms, main_launches = pr_distributed(
                sp, _lib, g, a, world, rank, local)
            result.update(iters=iters, total_ms=total_ms, main_ms=main_ms,
                          main_launches=main_launches, launches=launches)
    ms_per_step = result["total_ms"] / a.steps
    value = result["iters"] * m / (ms_per_step / 1e3) / 1e9
    mean_pull_ms = result["main_ms"] / max(1, result["main_launches"])
    achieved = bytes_pull / (mean_pull_ms / 1e3) / 1e9
    line = {
        "metric": BASELINE_METRIC, "value": value, "unit": "GTEPS", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic RMAT-{SCALE} (ef {EF}, seed {SEED}, dedup, no self-loops), "
                "generated on device",
        "config": {"workload": "pagerank_rmat22", "graph": f"rmat{SCALE}", "n": n, "m": m,
                   **PR_ARGS, "iterations": result["iters"],
                   "parallelism": f"block{world}" if world > 1 else "single",
                   "l2": "no flush: radj (4m = %.0f MB) + roff exceed the 126 MB L2; "
                         "contrib (8n = %.0f MB) is L2-resident by design"
                         % (4 * m / 1e6, 8 * n / 1e6)},
        "roofline": {"bound": "hbm", "kernel": "k_pr_units+k_pr_fix+k_pr_epi (one PR iteration)",
                     "achieved": achieved,
                     "peak": hbm_peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": ncu_traffic("pr_iteration"),
                     "algorithmic_bytes_per_launch": bytes_pull,
                     "mean_launch_ms": mean_pull_ms,
                     "note": "12 B/slot (radj 4 + contrib gather 8) + 36 B/vertex; gathers "
                             "hit L2, so frac > 1 is possible"},
        "gpu_launches": result["launches"],
        "call_device_ms_per_step": result.get("call_device_ms", result["total_ms"]) / a.steps,
        "clocks": clk.summary(),
    }
    if world == 1:
        line["e2e"] = e2e_pr(sp, corpus, g, a)
        if not a.no_cpu:
            line["cpu_baseline"] = cpu_baseline(g)
        if a.algos:
            line["algorithms"] = other_algorithms(sp, corpus, a, hbm_peak)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def e2e_pr(sp, corpus, g, a):
    """Public-API PR with host buffers each step (pinned CSR in, ranks out)."""
    import torch
    off = torch.from_numpy(np.asarray(g.offsets)).pin_memory().numpy()
    adj = torch.from_numpy(np.asarray(g.adj)).pin_memory().numpy()
    w = torch.from_numpy(np.asarray(g.weights)).pin_memory().numpy()
    h2d = off.nbytes + adj.nbytes + w.nbytes
    d2h = 8 * g.n

    def step():
        gg = sp.from_csr(off, adj, w, directed=True, device=g.device)
        r = sp.run(corpus.PR, gg, PR_ARGS)
        rank = r.env.node_props["rank"]
        gg.close()
        return r, rank

    for _ in range(max(1, min(a.warmup, 2))):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    k = max(1, min(a.steps, 3))
    for _ in range(k):
        r, _ = step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / k
    return {"value": r.env.scalars["iter"] * g.m / dt / 1e9, "unit": "GTEPS",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": dt * 1e3,
            "includes": "H2D CSR (pinned) + device reverse-CSR build + PR + D2H ranks"}


def cpu_baseline(g):
    try:
        gteps, it, dt, nt = cpu_pr_sample(np.asarray(g.offsets), np.asarray(g.rev_offsets),
                                          np.asarray(g.rev_adj), g.n, g.m)
        return {"value": gteps, "unit": "GTEPS", "cores": nt, "kind": "port",
                "sample": f"{it} PR iterations on the full RMAT-{SCALE} graph "
                          f"({dt:.1f} s), oracle/cpu_ref.c OpenMP x{nt}"}
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "GTEPS", "cores": None, "kind": "port",
                "sample": f"failed: {e}"}


def pr_distributed(sp, _lib, g, a, world, rank, local):
    """Block-partitioned PR over NCCL: local pull on the owned block, then
    all_gather of contrib slices + all_reduce(max) of diff per iteration."""
    import ctypes as C

    import torch
    import torch.distributed as dist
    parts = sp.block_partition(g, world)
    per = parts[0].size
    v0, v1 = parts[rank].real_range().start, parts[rank].real_range().stop
    L = _lib.lib()
    dev = torch.device("cuda", local)
    contrib_full = torch.zeros(per * world, dtype=torch.float64, device=dev)
    rank_local = torch.zeros(max(1, per), dtype=torch.float64, device=dev)
    contrib_local = torch.zeros(max(1, per), dtype=torch.float64, device=dev)
    diff = C.c_double()
    eps, max_iter = PR_ARGS["epsilon"], PR_ARGS["maxIter"]

    def one_run():
        torch.cuda.current_stream().synchronize()
        L.sp_pagerank_block_init(g.handle, v0, v1, C.c_void_p(rank_local.data_ptr()),
                                 C.c_void_p(contrib_local.data_ptr()))
        dist.all_gather_into_tensor(contrib_full, contrib_local)
        it = 0
        launches = 0
        kms = 0.0
        while True:
            st = _lib.Stats()
            torch.cuda.current_stream().synchronize()  # collectives done before the native step
            rc = L.sp_pagerank_block_step(g.handle, v0, v1, PR_ARGS["damping"],
                                          C.c_void_p(contrib_full.data_ptr()),
                                          C.c_void_p(rank_local.data_ptr()),
                                          C.c_void_p(contrib_local.data_ptr()),
                                          C.byref(diff), 0, C.byref(st))
            assert rc == 0, _lib.last_error()
            launches += st.kernel_launches
            kms += st.device_ms
            dt = torch.tensor([diff.value], dtype=torch.float64, device=dev)
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            dist.all_gather_into_tensor(contrib_full, contrib_local)
            it += 1
            if float(dt.item()) < eps or it >= max_iter:
                return it, launches, kms

    for _ in range(a.warmup):
        one_run()
    torch.cuda.synchronize()
    dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    launches = 0
    kms = 0.0
    for _ in range(a.steps):
        it, l, k = one_run()
        launches += l
        kms += k
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return float(ms.item()), it, launches, kms, it * a.steps


def other_algorithms(sp, corpus, a, hbm_peak):
    """SSSP cfg1, BC cfg4 (256 sources), TC cfg3 at one GPU."""
    out = {}
    reps = 3
    if "sssp" in a.algos:
        g = sp.generate("rmat", 16, 16, seed=SEED)
        for _ in range(2):
            sp.run(corpus.SSSP, g, {"src": 0})
        ms, R, F, km = [], 0, 0, 0.0
        for _ in range(reps):
            r = sp.run(corpus.SSSP, g, {"src": 0})
            ms.append(r.stats["device_ms"])
            R, F, km = r.stats["edges_visited"], r.stats["vertices_visited"], r.stats["main_kernel_ms"]
        t = statistics.median(ms) / 1e3
        offs = np.asarray(g.offsets)
        d = r.env.node_props["dist"]
        reached = d < 2147483647
        m_reached = int((offs[1:] - offs[:-1])[reached].sum())
        b = 12 * R + 20 * F
        out["sssp_cfg1"] = {"graph": "rmat16 directed", "n": g.n, "m": g.m,
                            "gteps": m_reached / t / 1e9, "relax_per_s": R / t / 1e9,
                            "ms": t * 1e3, "iterations": r.fixedpoint_iterations["finished"],
                            "roofline_frac": b / (km / 1e3) / 1e9 / hbm_peak,
                            "note": "launch/latency-bound (m ~ 1M)"}
        g.close()
    if "bc" in a.algos:
        g = sp.generate("rmat", 20, 16, seed=SEED, undirected=True)
        deg = np.diff(np.asarray(g.offsets))
        cand = np.flatnonzero(deg > 0)
        srcs = np.random.default_rng(SEED).choice(cand, size=256, replace=False).tolist()
        sp.run(corpus.BC, g, {"sourceSet": srcs[:8]})
        r = sp.run(corpus.BC, g, {"sourceSet": srcs})
        st = r.stats
        t = st["device_ms"] / 1e3
        b = 48 * st["edges_visited"] + 64 * st["vertices_visited"]
        out["bc_cfg4"] = {"graph": "rmat20 symmetrized", "n": g.n, "m": g.m, "sources": 256,
                          "gteps": st["edges_visited"] / t / 1e9, "ms": t * 1e3,
                          "roofline_frac": b / t / 1e9 / hbm_peak}
        g.close()
    if "tc" in a.algos:
        g = sp.generate("uniform", 1 << 24, 1 << 28, seed=SEED, undirected=True)
        sp.run(corpus.TC, g, {})
        ms = []
        for _ in range(reps):
            r = sp.run(corpus.TC, g, {})
            ms.append(r.stats["main_kernel_ms"])
        t = statistics.median(ms) / 1e3
        pairs = r.stats["edges_visited"]
        out["tc_cfg3"] = {"graph": "uniform 2^24 / 2^28 undirected", "n": g.n, "m": g.m,
                          "triangles": r.env.scalars["triangle_count"],
                          "gteps": (g.m // 2) / t / 1e9, "ms": t * 1e3, "pairs": pairs}
        g.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--algos", default="sssp,bc,tc",
                    help="secondary algorithms at N=1 ('' to skip)")
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    a.algos = [x for x in a.algos.split(",") if x and x != "none"]
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
