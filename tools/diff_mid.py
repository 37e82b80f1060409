"""Run the CUDA path on a mid-size reference golden (tests/golden/mid/) and
diff its per-pair fill decisions against the reference's decision log.

    IFMM_TRACE=/tmp/t.txt python tools/diff_mid.py <case> [reference|wavefront] [exact]

Prints per-level statistics (ours vs reference), the first pair whose
(cj, ck, r1, r2) differs from the reference log (exact order only: the
default order permutes pairs across cluster waves, so there the multiset of
decisions per level is compared), and |x - x_ref|.
"""
import collections
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1508_01835_b200 as P  # noqa: E402
from golden_mid import load_mid, mid_inputs  # noqa: E402


def parse_trace(path):
    lev_of, out = {}, []
    cur_level = None
    for ln in open(path):
        t = ln.split()
        if t[0] == "E":
            cur_level = int(t[1])
        elif t[0] == "P":
            out.append((cur_level, int(t[1]), int(t[2]), int(t[3]), int(t[4])))
        elif t[0] == "D":
            out.append((cur_level, int(t[1]), int(t[2]), 0, 0))
    return out


def main():
    name = sys.argv[1]
    schedule = sys.argv[2] if len(sys.argv) > 2 else "reference"
    exact = len(sys.argv) > 3 and sys.argv[3] == "exact"
    g = load_mid(name)
    pts, b, K = mid_inputs(P, g)
    eps = float(g["eps"])
    tree, _ = P.build_octree(pts, int(g["leaf"]))
    topo = P.compute_topology(tree)
    ops = P.chebyshev_operators(tree, topo, K, int(g["n"]), epsilon=eps)
    ranks = np.array([ops.rank.get(c, -1) for c in range(tree.n_clusters)])
    print("ranks equal:", np.array_equal(ranks, g["ranks"]), flush=True)
    P.initialize_weights(ops, topo)
    graph = P.assemble_extended_graph(ops)
    t0 = time.perf_counter()
    fct = P.factorize(graph, eps, seed=0, sigma0=float(g["sigma0"]), exact_order=exact,
                      schedule=schedule)
    print("schedule", schedule, "strict pairs", exact, "factorize %.2f s" % (time.perf_counter() - t0),
          "rsvd", fct.rsvd, "timings", {k: round(v, 3) for k, v in fct.timings.items()})
    for s, l, c, d, a, rs in zip(fct.stats.levels, g["lv_level"], g["lv_compressed"],
                                 g["lv_dropped"], g["lv_added"], g["lv_ranksum"]):
        print(f"level {s.level}: ours comp {s.compressed_pairs} drop {s.dropped_pairs} "
              f"add {s.added} Σr {sum(s.ranks)} | ref {l}: comp {c} drop {d} add {a} Σr {rs}")
    print("peak edges ours", fct.stats.peak_edges, "ref", int(g["peak_edges"]))
    x = fct.solve(b)
    rel = np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"])
    print(f"|x - x_ref|/|x_ref| = {rel:.3e} (10 eps = {10 * eps:.1e})")
    nb = np.linalg.norm(b)
    r_ours = np.linalg.norm(P.exact_matvec(pts, K, x) - b) / nb
    r_ref = np.linalg.norm(P.exact_matvec(pts, K, g["x"]) - b) / nb
    r_h2 = np.linalg.norm(P.h2_matvec(ops, x) - b) / nb if not getattr(ops, "consumed", False) else float("nan")
    print(f"exact-matvec residual: ours {r_ours:.4e} reference {r_ref:.4e}")
    np.save(os.path.join(ROOT, "gpurun_out", f"x_{name}_{schedule}.npy"), x)
    tr = os.environ.get("IFMM_TRACE")
    if not tr:
        return
    ours = parse_trace(tr)
    ref = [(int(lv), int(cj), int(ck), max(int(r1), 0), max(int(r2), 0))
           for lv, cj, ck, r1, r2 in g["pairs"]]
    # level of our trace entries: map the eliminated cluster to its level
    lvl = np.asarray([c.level for c in tree.clusters])
    ours = [(int(lvl[cl]) if cl is not None and cl < len(lvl) else -1, cj, ck, r1, r2)
            for cl, cj, ck, r1, r2 in ours]
    print("pairs ours", len(ours), "ref", len(ref))
    if schedule == "reference":
        for i, (o, r) in enumerate(zip(ours, ref)):
            if o[1:] != r[1:]:
                print("first mismatch at", i, "ours", o, "ref", r)
                for j in range(max(0, i - 5), min(len(ref), i + 6)):
                    print("  ", j, ours[j] if j < len(ours) else None, ref[j])
                break
        else:
            print("pair sequences identical")
    for lv in sorted({r[0] for r in ref}):
        co = collections.Counter(o[1:] for o in ours if o[0] == lv)
        cr = collections.Counter(r[1:] for r in ref if r[0] == lv)
        only_o, only_r = co - cr, cr - co
        print(f"level {lv}: multiset diff ours-only {sum(only_o.values())} "
              f"ref-only {sum(only_r.values())}")
        ex = sorted(only_r.items())[:8]
        ey = sorted(only_o.items())[:8]
        print("   ref-only e.g.", ex)
        print("   ours-only e.g.", ey)


if __name__ == "__main__":
    main()
