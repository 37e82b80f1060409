#!/usr/bin/env python
"""IFMM factorize+solve benchmark (BASELINE.json metric: unknowns/s).

A "step" = one pass of the hot path over the synthetic problem: sigma0
estimation + factorize (factor.py:176-230) + one solve (factor.py:99-157),
exactly what the reference's unknowns/s covers.  Setup --
points, octree, H2 operators, weights, and the per-step extended-graph
assembly (factorize consumes its graph) -- is outside the timed region.

  value  : N * K / (device time of K steps), rhs and solution resident on
           the GPU (CUDA events on the engine stream, max over ranks)
  e2e    : same, but every step's solve goes through the public API with a
           HOST numpy rhs (h2d of b and d2h of x inside the timed region)
  roofline : dominant device kernel category of one extra instrumented step
  cpu_baseline : the numpy oracle port on a bounded same-recipe sample, plus
           the unmodified reference timed on the FULL config once in the build
           container (full_size_reference, from tests/golden/mid/)
  parity : |x - x_reference| and the exact-matvec residuals of ours and of
           the reference's committed solution of the same config
--schedule: "wavefront" (default: the fastest; clusters at Chebyshev
distance >= 3 batched) or "reference" (Morton order + the reference's PCG64
sketch stream); see paper_1508_01835_b200.factor.factorize.

`--impl reference` times the CPU reference path (the oracle port of the
reference; the unmodified reference is Python and not installable on the
GPU box) on a bounded sample, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# SURVEY.md 8d pinned recipes: (N, dim, seed, kernel, leaf, n_cheb, eps)
CONFIGS = {
    "c1": (4096, 2, 0, "exp", 32, 4, 1e-8),
    "c2": (65536, 2, 1, "exp", 64, 6, 1e-10),
    "c3": (262144, 3, 2, "imq", 64, 4, 1e-6),
    "c4": (1048576, 3, 3, "imq", 64, 4, 1e-6),
}
DEFAULT_CONFIG = "c3"  # the headline recipe (3D IMQ, eps=1e-6) at the largest N whose 5+20-step driver run fits its time cap
METRIC = "IFMM factorize+solve unknowns/s"
# CPU sample sizes for the oracle leg (about 10-30 s of single-core work)
CPU_SAMPLE_N = {"c1": 4096, "c2": 8192, "c3": 4096, "c4": 4096}


def inputs(cfg, n=None):
    N, dim, seed, kern, leaf, nc, eps = CONFIGS[cfg]
    N = n or N
    g = np.random.Generator(np.random.PCG64(seed))
    if dim == 2:
        pts = np.column_stack([g.uniform(0.0, 1.0, size=(N, 2)), np.zeros(N)])
    else:
        pts = g.uniform(0.0, 1.0, size=(N, 3))
    gb = np.random.Generator(np.random.PCG64(seed + 1))
    b = gb.uniform(-1.0, 1.0, N) if dim == 2 else gb.standard_normal(N)
    h = N ** (-1.0 / 3.0)
    return dict(N=N, pts=pts, b=b, kern=kern, h=h, leaf=leaf, nc=nc, eps=eps, dim=dim)


def reference_golden(cfg):
    """The unmodified reference's solution of the full config, if committed."""
    name = {"c2": "c2_exp2d_n65536", "c3": "c3_imq3d_n262144"}.get(cfg)
    path = os.path.join(ROOT, "tests", "golden", "mid", f"{name}.npz") if name else None
    if not path or not os.path.exists(path):
        return None
    g = np.load(path)
    return {"x": g["x"], "sigma0": float(g["sigma0"]), "t": float(g["t_factorize"]) + float(g["t_solve"]),
            "levels": g["lv_compressed"].tolist()}


def workload_desc(cfg, inp):
    return {"workload": f"{cfg}: {inp['dim']}D N={inp['N']} {inp['kern']}"
                        f"{' h=N^-1/3' if inp['kern'] == 'imq' else ''}, leaf<= {inp['leaf']}, "
                        f"{inp['nc']}^3 Chebyshev, eps={inp['eps']:g}, fp64",
            "N": inp["N"], "epsilon": inp["eps"], "l2": "inputs >> L2 (graph blocks GBs)"}


# ---------------------------------------------------------------------------
# CPU legs (oracle = checker / reported baseline only)
# ---------------------------------------------------------------------------
def cpu_oracle_rate(cfg, threads):
    from threadpoolctl import threadpool_limits
    from oracle import ifmm_np as O
    n = CPU_SAMPLE_N[cfg]
    inp = inputs(cfg, n)
    block = O.exp_block if inp["kern"] == "exp" else O.imq_block(inp["h"])
    with threadpool_limits(limits=threads):
        tree, topo, ops = O.pipeline(inp["pts"], block, inp["leaf"], inp["nc"], inp["eps"])
        g = O.Graph(ops)
        t0 = time.perf_counter()
        f = O.factorize(g, inp["eps"], seed=0)
        x = f.solve(inp["b"])
        dt = time.perf_counter() - t0
    del x
    sample = (f"oracle numpy port of the reference path (pinned bitwise to the reference on "
              f"c2 / mid goldens), {cfg} recipe at a bounded N={n} (depth {tree.depth}; "
              f"sigma0+factorize+solve {dt:.2f} s on {threads} thread(s)); the per-unknown "
              f"rate falls with N (see full_size_reference)")
    return n / dt, dt, sample


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = args.config
    # single BLAS thread: faster than all cores for this small-block numpy
    # code (12-13 s with 1 thread vs ~19 s with 8)
    threads = 1
    times = []
    n = CPU_SAMPLE_N[cfg]
    for i in range(args.warmup + args.steps):
        rate, dt, sample = cpu_oracle_rate(cfg, threads)
        if i >= args.warmup:
            times.append(dt)
    tot = sum(times)
    val = n * len(times) / tot
    inp = inputs(cfg)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "unknowns/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot / max(len(times), 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_desc(cfg, inp),
            "cpu_baseline": {"value": val, "unit": "unknowns/s", "cores": threads,
                             "kind": "port", "sample": sample,
                             "full_size_reference": full_size_reference(cfg)},
            "e2e": {"value": val, "unit": "unknowns/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def full_size_reference(cfg):
    """The unmodified reference on the full config, measured once in the build
    container (1 thread): unknowns/s, or None when not measured."""
    g = reference_golden(cfg)
    if g is None:
        return None
    N = CONFIGS[cfg][0]
    return {"N": N, "seconds": round(g["t"], 1), "unknowns_per_s": N / g["t"], "cores": 1,
            "source": "tests/golden/mid (make_golden_mid.py), unmodified reference package"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, dev):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(dev), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = []
        for ln in open(self.f.name):
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) >= 7 and parts[0].isdigit():
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [int(r[0]) for r in rows]
        load = [s for s in sm if s > 500] or sm
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": int(rows[0][1]),
                "reasons": sorted(reasons), "samples": len(rows)}


def fp64_peak_tflops():
    """cuBLAS DGEMM 8192^3 best of 5 (MEASURED_PEAKS.json has no fp64 entry)."""
    import torch
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) * 1e-3)
    del a, b
    torch.cuda.empty_cache()
    return 2.0 * 8192 ** 3 / best / 1e12


def reduce_max(vals, device="cuda"):
    """Max over ranks of a list of timings (no-op without a process group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(vals)
    t = torch.tensor(list(vals), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def run_ours(args, rank, world):
    import torch
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    import paper_1508_01835_b200 as P
    from paper_1508_01835_b200 import _native as NN

    fp64_peak = fp64_peak_tflops() if rank == 0 else None
    if "IFMM_ARENA_GB" not in os.environ:  # the engine arena takes most of the device
        free, _ = torch.cuda.mem_get_info()
        # leave ~22 GB outside the arena for the dedicated >= 256 MB blocks
        os.environ["IFMM_ARENA_GB"] = f"{max(0.5 * free, free - 22 * 2**30) / 2**30:.1f}"
    cfg = args.config
    sched = args.schedule
    inp = inputs(cfg, args.n)
    N = inp["N"]
    K = P.exp_kernel() if inp["kern"] == "exp" else P.imq_kernel(inp["h"])
    t0 = time.perf_counter()
    tree, _ = P.build_octree(inp["pts"], inp["leaf"])
    topo = P.compute_topology(tree)

    def make_ops():
        o = P.chebyshev_operators(tree, topo, K, inp["nc"], epsilon=inp["eps"])
        P.initialize_weights(o, topo)
        return o
    ops = make_ops()
    t_setup = time.perf_counter() - t0
    b_host = np.ascontiguousarray(inp["b"])
    b_dev = torch.from_numpy(b_host).cuda()
    # large configs: the graph takes the operator blocks (no copy) and the
    # operators are rebuilt for the next step -- all outside the timed region
    consume = N >= args.consume_from
    state = {"ops": ops}

    def one_step(host_rhs: bool, timed: bool):
        if consume and state["ops"] is None:
            state["ops"] = make_ops()
        graph = P.assemble_extended_graph(state["ops"], consume=consume)
        if consume:
            state["ops"] = None
        NN.lib().ifmm_dev_sync(NN.ctx())
        NN.event(0)
        s0 = P.estimate_sigma0(graph, seed=0)
        fct = P.factorize(graph, inp["eps"], seed=0, sigma0=s0, schedule=sched)
        NN.event(1)
        x = fct.solve(b_host if host_rhs else b_dev)
        NN.event(2)
        t_f = NN.elapsed_ms(0, 1) * 1e-3
        t_s = NN.elapsed_ms(1, 2) * 1e-3
        return t_f, t_s, fct, x

    for _ in range(args.warmup):
        one_step(False, False)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(torch.cuda.current_device()) if rank == 0 else None
    l0 = NN.launches()
    tf, ts, tsh = [], [], []
    for _ in range(args.steps):
        a, b_, fct, x = one_step(False, True)
        # e2e: the same factorization's solve through the public API on host
        NN.event(3)
        xh = fct.solve(b_host)
        NN.event(4)
        tf.append(a)
        ts.append(b_)
        tsh.append(NN.elapsed_ms(3, 4) * 1e-3)
        del fct, x, xh
    launches = NN.launches() - l0
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks else None
    tot_dev = sum(tf) + sum(ts)
    tot_e2e = sum(tf) + sum(tsh)
    tot_dev, tot_e2e = reduce_max([tot_dev, tot_e2e])
    if rank != 0:
        return
    # ---- instrumented step for the kernel roofline ----
    NN.ktime(1)
    _, _, fct, x = one_step(False, False)
    kt = NN.ktime(0)
    if state["ops"] is None:
        state["ops"] = make_ops()
    xh = x.cpu().numpy()
    res = float(np.linalg.norm(P.h2_matvec(state["ops"], xh) - b_host) / np.linalg.norm(b_host))
    parity = {"schedule": sched, "factorize_levels_compressed": [s.compressed_pairs for s in fct.stats.levels]}
    gold = reference_golden(cfg) if args.n is None else None
    if gold is not None:
        Kx = P.exact_matvec(inp["pts"], K, xh)
        parity.update({
            "rel_diff_x_vs_reference": float(np.linalg.norm(xh - gold["x"]) / np.linalg.norm(gold["x"])),
            "exact_residual": float(np.linalg.norm(Kx - b_host) / np.linalg.norm(b_host)),
            "reference_exact_residual": float(np.linalg.norm(P.exact_matvec(inp["pts"], K, gold["x"]) - b_host)
                                              / np.linalg.norm(b_host)),
            "reference_levels_compressed": gold["levels"]})
    del fct, x
    # ---- HBM-bound stages: replay solve and H2 matvec (algorithmic bytes =
    # every stored factor / operator byte the stage reads) ----
    hbm_lines = {}
    if state["ops"] is not None:
        P.h2_matvec(state["ops"], b_dev)  # builds the cached block lists
        NN.ktime(1)
        for _ in range(5):
            P.h2_matvec(state["ops"], b_dev)
        km = NN.ktime(0)["spmv"]
        if km[2]:
            hbm_lines["h2_matvec"] = {"ms": 1e3 * km[0] / km[2], "algorithmic_GB": km[1] / km[2] / 1e9,
                                      "GB_per_s": km[1] / km[0] / 1e9}
    if kt.get("solve", (0, 0, 0))[2]:
        ks = kt["solve"]
        hbm_lines["solve"] = {"ms": 1e3 * ks[0] / ks[2], "algorithmic_GB": ks[1] / ks[2] / 1e9,
                              "GB_per_s": ks[1] / ks[0] / 1e9}
    # ---- the grouped DMMA GEMM (csrc/gemm.cu) alone on a large problem: what
    # the elimination's dense products reach when a launch is not latency-bound ----
    gemm_peak = None
    try:
        import ctypes as C
        ng = 4096
        ga = torch.randn(ng, ng, dtype=torch.float64, device="cuda")
        gb_ = torch.randn(ng, ng, dtype=torch.float64, device="cuda")
        gc = torch.zeros(ng, ng, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        call = lambda: NN.check(NN.lib().ifmm_dev_gemm(  # noqa: E731
            NN.ctx(), ng, ng, ng, C.c_void_p(ga.data_ptr()), ng, 0, C.c_void_p(gb_.data_ptr()), ng, 0,
            C.c_void_p(gc.data_ptr()), ng, 1.0, 0.0))
        call()
        NN.lib().ifmm_dev_sync(NN.ctx())
        NN.event(0)
        for _ in range(3):
            call()
        NN.event(1)
        tg = NN.elapsed_ms(0, 1) * 1e-3 / 3
        gemm_peak = {"problem": "4096^3 fp64, one problem through ifmm_dev_gemm", "ms": 1e3 * tg,
                     "TFLOP_per_s": 2.0 * ng ** 3 / tg / 1e12,
                     "frac_of_dgemm_peak": 2.0 * ng ** 3 / tg / 1e12 / fp64_peak}
        del ga, gb_, gc
    except Exception as e:  # diagnostics only
        gemm_peak = {"failed": str(e)[:120]}
    # ---- the relaxed (colour-wave) schedule on the same problem, one step,
    # outside the timed region: reported beside the headline, never as it ----
    relaxed = None
    if args.relaxed and sched != "colored":
        try:
            if consume and state["ops"] is None:
                state["ops"] = make_ops()
            graph = P.assemble_extended_graph(state["ops"], consume=consume)
            if consume:
                state["ops"] = None
            NN.lib().ifmm_dev_sync(NN.ctx())
            NN.event(0)
            s0c = P.estimate_sigma0(graph, seed=0)
            fc = P.factorize(graph, inp["eps"], seed=0, sigma0=s0c, schedule="colored")
            NN.event(1)
            xc = fc.solve(b_dev)
            NN.event(2)
            tcf, tcs = NN.elapsed_ms(0, 1) * 1e-3, NN.elapsed_ms(1, 2) * 1e-3
            relaxed = {"schedule": "colored", "t_factorize_s": tcf, "t_solve_s": tcs,
                       "unknowns_per_s": N / (tcf + tcs),
                       "levels_compressed": [s.compressed_pairs for s in fc.stats.levels],
                       "note": "relaxed elimination order (SURVEY.md 8e): not comparable with the "
                               "reference's statistics; validated by the residual criterion only"}
            if gold is not None:
                Kxc = P.exact_matvec(inp["pts"], K, xc.cpu().numpy())
                relaxed["exact_residual"] = float(np.linalg.norm(Kxc - b_host) / np.linalg.norm(b_host))
            del fc, xc
        except Exception as e:  # the relaxed order is experimental
            relaxed = {"schedule": "colored", "failed": f"{type(e).__name__}: {e}"[:200]}
    dom = max(kt.items(), key=lambda kv: kv[1][0])
    cat, (ksec, kwork, kcnt) = dom
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    if cat in ("solve", "copy", "spmv"):
        ach = kwork / ksec / 1e9 if ksec > 0 else 0.0
        roof = {"bound": "hbm", "kernel": cat, "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "traffic": None, "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    else:
        ach = kwork / ksec / 1e12 if ksec > 0 else 0.0
        roof = {"bound": "tensor", "kernel": cat, "achieved": ach, "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": ach / fp64_peak, "traffic": None,
                "peak_source": "fp64 cuBLAS DGEMM 8192^3 measured in this run"}
    prof = os.path.join(ROOT, "profiles", "r02_roofline_traffic.json")
    if os.path.exists(prof):  # dram bytes per launch of the dominant kernel, one ncu --set full capture
        tr = json.load(open(prof)).get(cat)
        if tr:
            roof["traffic"] = tr["dram_bytes_per_launch"]
            roof["traffic_source"] = tr["source"]
    roof["launches"] = kcnt
    roof["avg_launch_ms"] = 1e3 * ksec / max(kcnt, 1)
    roof["categories"] = {k: {"s": round(v[0], 4), "work": v[1], "n": v[2]}
                          for k, v in kt.items() if v[2]}
    # ---- CPU baseline (oracle port, bounded sample) ----
    cpu_rate, cpu_dt, sample = cpu_oracle_rate(cfg, 1)
    value = N * args.steps * world / tot_dev
    e2e = N * args.steps * world / tot_e2e
    line = {"metric": METRIC, "value": value, "unit": "unknowns/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_dev / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SURVEY.md 8d seeded recipe)",
            "config": dict(workload_desc(cfg, inp), parallelism=f"replicas{world}", schedule=sched),
            "e2e": {"value": e2e, "unit": "unknowns/s", "h2d_bytes_per_step": 8 * N,
                    "d2h_bytes_per_step": 8 * N},
            "gpu_launches": launches,
            "roofline": roof,
            "cpu_baseline": {"value": cpu_rate, "unit": "unknowns/s", "cores": 1,
                             "kind": "port", "sample": sample,
                             "full_size_reference": full_size_reference(cfg)},
            "parity": parity,
            "clocks": clk,
            "detail": {"t_factorize_s": statistics.mean(tf), "t_solve_dev_s": statistics.mean(ts),
                       "t_solve_host_s": statistics.mean(tsh), "t_setup_s": t_setup,
                       "rel_residual_h2": res, "hbm_stages": hbm_lines, "gemm_kernel": gemm_peak,
                       "relaxed_schedule": relaxed,
                       "hbm_peak_GB_per_s": hbm,
                       "fp64_dgemm_tflops": fp64_peak}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default: 2 for c1/c2, 1 otherwise)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--n", type=int, default=None, help="override N (diagnostics)")
    ap.add_argument("--schedule", default=os.environ.get("IFMM_SCHEDULE", "wavefront"),
                    choices=["wavefront", "reference", "colored"],
                    help="factorize schedule (paper_1508_01835_b200.factor.factorize)")
    ap.add_argument("--relaxed", type=int, default=1,
                    help="also run one step of the relaxed colour-wave schedule (reported in detail)")
    ap.add_argument("--consume-from", type=int, default=500000,
                    help="N at/above which graphs consume (move) the operator blocks")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 2 if args.config in ("c1", "c2") else 1
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
