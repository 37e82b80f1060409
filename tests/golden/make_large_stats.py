"""Reference-semantics statistics at BASELINE sizes, from the numpy oracle
(pinned to the reference by tests/test_oracle_golden.py).  Too slow for the
test suite; run once in the build container:
    python tests/golden/make_large_stats.py c3
Writes tests/golden/large/<cfg>_stats.json (tree/rank/fill statistics,
sigma0, solution checksum and the solution itself as .npy)."""
import json, os, sys, time
import numpy as np
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ifmm_np as O  # noqa: E402

cfg = sys.argv[1]
fseed = int(sys.argv[2]) if len(sys.argv) > 2 else 0   # factorize rng seed (rSVD sketches)
tag = cfg if fseed == 0 else f"{cfg}_seed{fseed}"
inp = O.config_inputs(cfg)
t0 = time.perf_counter()
tree, topo, ops = O.pipeline(inp["points"], inp["block"], inp["leaf"], inp["n"], inp["eps"])
t_setup = time.perf_counter() - t0
g = O.Graph(ops)
t0 = time.perf_counter()
s0 = O.sigma0_estimate(g, seed=0)
f = O.factorize(g, inp["eps"], seed=fseed, sigma0=s0)
t_fact = time.perf_counter() - t0
t0 = time.perf_counter()
x = f.solve(inp["b"])
t_solve = time.perf_counter() - t0
out = {"cfg": cfg, "factorize_seed": fseed, "N": inp["N"], "depth": tree.depth, "sigma0": s0,
       "levels": [[s.level, s.compressed_pairs, s.dropped_pairs, s.added, sum(s.ranks), s.max_rank]
                  for s in f.levels],
       "peak_edges": f.peak_edges, "max_basis_rank": f.max_basis_rank,
       "ranks_sum": int(sum(ops.rank.values())), "n_rebase": sum(1 for e in f.events if e[0] == "rebase"),
       "t_setup": t_setup, "t_factorize": t_fact, "t_solve": t_solve,
       "unknowns_per_s": inp["N"] / (t_fact + t_solve), "x_norm": float(np.linalg.norm(x))}
os.makedirs(os.path.join(HERE, "large"), exist_ok=True)
np.save(os.path.join(HERE, "large", f"{tag}_x.npy"), x)
json.dump(out, open(os.path.join(HERE, "large", f"{tag}_stats.json"), "w"), indent=1)
print(json.dumps(out))
