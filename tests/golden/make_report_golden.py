"""RunReports of the UNMODIFIED reference harness (experiments.py) for small
configs, as a JSON fixture: the non-timing fields (config echo, rank and
edge statistics, errors, GMRES iteration counts) are what the drop-in's
harness must reproduce.  Run in the build container:
    python tests/golden/make_report_golden.py
Writes tests/golden/reports.json."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref_shim  # noqa: E402

ifmm = ref_shim.import_reference()
from ifmm.experiments import RunConfig, run_direct, run_iterative  # noqa: E402

BASE = dict(kernel="benchmark", n_points=300, distribution="cube", cheb_nodes=2, epsilon=1e-3,
            leaf_target=30, d=1e-2, seed=0)
CASES = {
    "direct_small": dict(BASE),
    "direct_sphere_n4": dict(BASE, n_points=1000, distribution="sphere", cheb_nodes=4, d=1e-3,
                             d_scaling="sphere", leaf_target=100),
    "direct_tight": dict(BASE, n_points=600, epsilon=1e-6, cheb_nodes=3),
    "gmres_none": dict(BASE, mode="gmres", precond="none"),
    "gmres_ifmm": dict(BASE, mode="gmres", precond="ifmm"),
    "gmres_ifmm_left": dict(BASE, mode="gmres", precond="ifmm", precond_side="left"),
    "gmres_blockdiag": dict(BASE, mode="gmres", precond="blockdiag", blockdiag_size=50),
    "gmres_lattice": dict(BASE, mode="gmres", precond="ifmm", distribution="lattice",
                          lattice_shape=(2, 2, 2), subdivision=1, leaf_target=20),
}
out = {}
for name, kw in CASES.items():
    cfg = RunConfig(**kw)
    rep = run_direct(cfg) if cfg.mode == "direct" else run_iterative(cfg)
    d = rep.to_dict()
    out[name] = {"kwargs": {k: (list(v) if isinstance(v, tuple) else v) for k, v in kw.items()},
                 "report": d}
    print(name, d["errors"], d["rank_stats"]["max_basis_rank"], (d["iteration"] or {}).get("iterations"))
json.dump(out, open(os.path.join(HERE, "reports.json"), "w"), indent=1)
