"""Run reports (mirror of ``ifmm.reports``, reports.py:1-112).

The report layout and the JSON schema (``run_report.schema.json``, version
1) are the reference's data format, so reports from the reference package
and from this engine diff field by field.  Serialises to JSON or flat CSV.
"""

from __future__ import annotations

import csv
import json
from dataclasses import asdict, dataclass

SCHEMA_VERSION = 1

# CSV columns: (column, section, key) -- reports.py:41-63
_CSV = (("n_points", "config", "n_points"), ("cheb_nodes", "config", "cheb_nodes"),
        ("epsilon", "config", "epsilon"), ("distribution", "config", "distribution"),
        ("seed", "config", "seed"), ("t_initialization", "timings", "initialization"),
        ("t_sigma0", "timings", "sigma0_estimation"), ("t_elimination", "timings", "elimination"),
        ("t_substitution", "timings", "substitution"), ("t_total", "timings", "total"),
        ("relative_error", "errors", "relative_error"),
        ("relative_residual", "errors", "relative_residual"),
        ("max_basis_rank", "rank_stats", "max_basis_rank"),
        ("max_fill_rank", "rank_stats", "max_fill_rank"),
        ("peak_edges", "edge_stats", "peak_edges"),
        ("edge_bound_constant", "edge_stats", "edge_bound_constant"),
        ("iterations", "iteration", "iterations"), ("converged", "iteration", "converged"))


@dataclass
class RunReport:
    schema_version: int
    config: dict
    timings: dict
    elimination_breakdown: dict
    rank_stats: dict
    edge_stats: dict
    errors: dict
    iteration: dict | None = None

    def to_dict(self) -> dict:
        return asdict(self)

    def to_json(self, path=None, indent=2):
        text = json.dumps(self.to_dict(), indent=indent)
        if path is None:
            return text
        with open(path, "w") as fh:
            fh.write(text + "\n")

    def csv_row(self) -> dict:
        d = self.to_dict()
        return {col: (d.get(sec) or {}).get(key) for col, sec, key in _CSV}


def write_csv(reports, path) -> None:
    rows = [r.csv_row() for r in reports]
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=[c for c, _, _ in _CSV])
        w.writeheader()
        w.writerows(rows)


def _obj(required, **props):
    return {"type": "object", "required": list(required), "properties": props}


_NUM, _INT, _STR, _BOOL = ({"type": "number"}, {"type": "integer"}, {"type": "string"},
                           {"type": "boolean"})


def _opt(t):
    return {"type": [t, "null"]}


def load_schema() -> dict:
    """The report schema, version 1 (the reference's run_report.schema.json,
    draft-07): the keys and JSON types every report carries."""
    timing_keys = ("initialization", "sigma0_estimation", "elimination", "substitution", "total")
    breakdown_keys = ("lu_and_triangular_solves", "matmul_updates", "lowrank_approximations",
                      "operator_transfer")
    schema = _obj(
        ("schema_version", "config", "timings", "elimination_breakdown", "rank_stats",
         "edge_stats", "errors"),
        schema_version={"type": "integer", "const": SCHEMA_VERSION},
        config=_obj(("kernel", "n_points", "distribution", "cheb_nodes", "epsilon",
                     "leaf_target", "seed", "mode"),
                    kernel=_STR, n_points=_INT, distribution=_STR, cheb_nodes=_INT,
                    epsilon=_NUM, leaf_target=_INT, seed=_INT, mode=_STR, d=_opt("number"),
                    precond=_opt("string"), precond_side=_opt("string"),
                    gmres_tol=_opt("number"), max_iters=_opt("integer")),
        timings=_obj(timing_keys, **{k: _NUM for k in timing_keys}),
        elimination_breakdown=_obj(breakdown_keys, **{k: _NUM for k in breakdown_keys}),
        rank_stats=_obj(("max_basis_rank", "max_fill_rank"), max_basis_rank=_INT,
                        max_fill_rank=_INT,
                        per_level={"type": "array", "items": {"type": "object"}}),
        edge_stats=_obj(("peak_edges", "n_clusters", "edge_bound_constant"), peak_edges=_INT,
                        n_clusters=_INT, edge_bound_constant=_NUM),
        errors=_obj((), relative_error=_opt("number"), relative_residual=_opt("number")),
        iteration={"type": ["object", "null"],
                   "properties": {"iterations": _INT, "converged": _BOOL, "side": _STR,
                                  "residual_history": {"type": "array", "items": _NUM}}},
    )
    schema["$schema"] = "http://json-schema.org/draft-07/schema#"
    schema["title"] = "ifmm run report"
    return schema


_JSON_TYPES = {"object": (dict,), "number": (int, float), "integer": (int,), "string": (str,),
               "boolean": (bool,), "array": (list,), "null": (type(None),)}


def _is(value, t):
    if t in ("integer", "number") and isinstance(value, bool):
        return False
    return isinstance(value, _JSON_TYPES[t])


def _check(value, schema, path):
    t = schema.get("type")
    if t is not None:
        ts = t if isinstance(t, list) else [t]
        if not any(_is(value, x) for x in ts):
            raise ValueError(f"{path}: expected {t}, got {type(value).__name__}")
    if "const" in schema and value != schema["const"]:
        raise ValueError(f"{path}: expected constant {schema['const']}")
    if isinstance(value, dict):
        missing = [k for k in schema.get("required", []) if k not in value]
        if missing:
            raise ValueError(f"{path}: missing required key '{missing[0]}'")
        for k, sub in schema.get("properties", {}).items():
            if k in value:
                _check(value[k], sub, f"{path}.{k}")
    if isinstance(value, list) and "items" in schema:
        for i, v in enumerate(value):
            _check(v, schema["items"], f"{path}[{i}]")


def validate_report(d: dict) -> None:
    """reports.py:76-84: required keys and primitive types against the
    shipped schema; ValueError on the first violation."""
    _check(d, load_schema(), "$")
