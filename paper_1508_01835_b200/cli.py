"""``ifmm-bench`` command line (mirror of ``ifmm.cli``, cli.py:16-175).

One experiment per invocation -- a direct solve, GMRES, or a scaling sweep
over N -- printed as a JSON summary and optionally written as a JSON/CSV
report.  ``--config`` reads flag defaults from JSON (underscored keys;
command-line flags win), ``--scene-out`` exports the scene, ``--dump-pattern``
the extended graph's sparsity pattern.  Same flags and defaults as the
reference.

    python -m paper_1508_01835_b200.cli --n-points 20000 --epsilon 1e-6
"""

from __future__ import annotations

import argparse
import json
import sys

from .experiments import (RunConfig, build_pipeline, fit_loglog_slope, run_direct,
                          run_iterative, run_scaling)
from .graph import assemble_extended_graph
from .kernels import scene_to_text
from .reports import write_csv

# (flag, type, default, choices, help) -- cli.py:17-83
_FLAGS = (
    ("--config", str, None, None, "JSON file with flag defaults (underscored keys); "
                                  "command-line flags override it"),
    ("--kernel", str, "benchmark", ("benchmark", "rpy"), None),
    ("--n-points", int, 1000, None, "point count (sphere/cube distributions)"),
    ("--sweep", str, None, None, "comma-separated N list; runs a scaling sweep"),
    ("--distribution", str, "cube", ("sphere", "cube", "lattice", "shells"), None),
    ("--cheb-nodes", int, 3, None, None),
    ("--epsilon", float, 1e-3, None, None),
    ("--leaf-target", int, 100, None, None),
    ("--d", float, 1e-3, None, None),
    ("--d-scaling", str, "none", ("none", "sphere", "cube"), None),
    ("--mode", str, "direct", ("direct", "gmres"), None),
    ("--precond", str, "none", ("none", "blockdiag", "ifmm"), None),
    ("--precond-side", str, "right", ("left", "right"), None),
    ("--gmres-tol", float, 1e-10, None, None),
    ("--max-iters", int, 500, None, None),
    ("--seed", int, 0, None, None),
    ("--depth", int, None, None, "force the octree depth (default: automatic)"),
    ("--weights-mode", str, "rigorous", ("rigorous", "sampled"), None),
    ("--rpy-radius", float, 0.25, None, None),
    ("--viscosity", float, 1.0, None, None),
    ("--lattice", str, "4,4,4", None, "lattice shape nx,ny,nz"),
    ("--lattice-spacing", float, 4.0, None, None),
    ("--body-radius", float, 1.0, None, None),
    ("--subdivision", int, 1, None, "icosphere subdivision for lattice bodies"),
    ("--shell-subdivisions", str, "1,2,3", None, None),
    ("--shell-radii", str, None, None, "comma-separated radii (default: doubling from 1)"),
    ("--blockdiag-size", int, 126, None, None),
    ("--dense-cap", int, 25000, None, "largest dimension using exact matvecs"),
    ("--out", str, None, None, "report path"),
    ("--format", str, "json", ("json", "csv"), None),
    ("--scene-out", str, None, None, "export the generated scene as x y z text"),
    ("--dump-pattern", str, None, None, "dump the extended sparsity pattern as JSON"),
)


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="ifmm-bench",
                                description="IFMM direct solver / preconditioner benchmarks for "
                                            "dense kernel matrices (B200 engine).")
    for flag, typ, default, choices, hlp in _FLAGS:
        kw = {"type": typ, "default": default}
        if choices:
            kw["choices"] = list(choices)
        if hlp:
            kw["help"] = hlp
        p.add_argument(flag, **kw)
    return p


def _ints(s):
    return tuple(int(v) for v in s.split(","))


def config_from_args(a) -> RunConfig:
    """cli.py:86-117."""
    return RunConfig(kernel=a.kernel, n_points=a.n_points, distribution=a.distribution,
                     cheb_nodes=a.cheb_nodes, epsilon=a.epsilon, leaf_target=a.leaf_target,
                     d=a.d, d_scaling=a.d_scaling, mode=a.mode, precond=a.precond,
                     precond_side=a.precond_side, gmres_tol=a.gmres_tol,
                     max_iters=a.max_iters, seed=a.seed, depth=a.depth,
                     weights_mode=a.weights_mode, rpy_radius=a.rpy_radius,
                     viscosity=a.viscosity, lattice_shape=_ints(a.lattice),
                     lattice_spacing=a.lattice_spacing, body_radius=a.body_radius,
                     subdivision=a.subdivision, shell_subdivisions=_ints(a.shell_subdivisions),
                     shell_radii=(tuple(float(v) for v in a.shell_radii.split(","))
                                  if a.shell_radii else None),
                     blockdiag_size=a.blockdiag_size, dense_cap=a.dense_cap)


def _parse(argv):
    parser = build_parser()
    args = parser.parse_args(argv)
    if args.config:
        with open(args.config) as fh:
            defaults = json.load(fh)
        bad = sorted(set(defaults) - set(vars(args)))
        if bad:
            parser.error(f"unknown config keys: {bad}")
        parser.set_defaults(**defaults)
        args = parser.parse_args(argv)
    return args


def _sweep(config, args) -> int:
    ns = [int(v) for v in args.sweep.split(",")]
    reports = run_scaling(config, ns)
    totals = [r.timings["total"] for r in reports]
    slope = fit_loglog_slope(ns, totals)
    print(f"scaling sweep over N={ns}")
    for n, r in zip(ns, reports):
        print(f"  N={n:>8d}  total={r.timings['total']:.3f}s  "
              f"err={r.errors['relative_error']:.3e}  max_rank={r.rank_stats['max_basis_rank']}")
    print(f"fitted log-log slope: {slope:.3f}")
    if args.out:
        if args.format == "csv":
            write_csv(reports, args.out)
        else:
            with open(args.out, "w") as fh:
                json.dump({"slope": slope, "runs": [r.to_dict() for r in reports]}, fh, indent=2)
        print(f"report written to {args.out}")
    return 0


def main(argv=None) -> int:
    """cli.py:120-175."""
    args = _parse(argv)
    config = config_from_args(args)
    if args.scene_out:
        scene_to_text(config.scene(), args.scene_out)
        print(f"scene written to {args.scene_out}")
    if args.dump_pattern:
        graph = assemble_extended_graph(build_pipeline(config).ops)
        with open(args.dump_pattern, "w") as fh:
            json.dump(graph.sparsity_pattern(), fh)
        print(f"sparsity pattern written to {args.dump_pattern}")
    if args.sweep:
        return _sweep(config, args)
    report = run_direct(config) if args.mode == "direct" else run_iterative(config)
    summary = {"total_time": round(report.timings["total"], 4),
               "relative_error": report.errors.get("relative_error"),
               "relative_residual": report.errors.get("relative_residual")}
    if report.iteration:
        summary["iterations"] = report.iteration["iterations"]
        summary["converged"] = report.iteration["converged"]
    print(json.dumps(summary, indent=2))
    if args.out:
        if args.format == "csv":
            write_csv([report], args.out)
        else:
            report.to_json(args.out)
        print(f"report written to {args.out}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
