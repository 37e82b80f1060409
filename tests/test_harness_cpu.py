"""Harness host logic (experiments/reports/cli mirrors)
and scene generators (CPU): report schema, CSV layout, CLI flags and config
files, scenes and the RPY block against the reference fixtures."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN


def test_scenes_match_reference_fixture():
    import paper_1508_01835_b200 as P
    g = np.load(os.path.join(GOLDEN, "scenes.npz"))
    for s in range(4):
        np.testing.assert_array_equal(P.icosphere(s), g[f"ico{s}"])
    np.testing.assert_array_equal(P.sphere_lattice(2, 3, 2, 1, 4.0, 1.5).points, g["lattice"])
    np.testing.assert_array_equal(P.concentric_shells([0, 1, 2], [1.0, 2.0, 3.5]).points,
                                  g["shells"])
    np.testing.assert_array_equal(P.sphere_surface(50, 4).points, g["sphere"])
    np.testing.assert_array_equal(P.cube_uniform(50, 4).points, g["cube"])
    np.testing.assert_allclose(P.rpy_kernel(0.3, 0.7).block(g["rpy_P"], g["rpy_Q"]), g["rpy"],
                               rtol=1e-14, atol=1e-15)
    with pytest.raises(ValueError):
        P.icosphere(-1)
    with pytest.raises(ValueError):
        P.concentric_shells([1], [1.0, 2.0])
    with pytest.raises(ValueError):
        P.rpy_kernel(0.0)
    # a block_dim the engine does not implement is refused up front, no fallback
    with pytest.raises(ValueError):
        P.Kernel("rpy", 2, {"radius": 0.3, "viscosity": 1.0}, lambda A, B: None).device_spec()


def test_scene_text_roundtrip(tmp_path):
    import paper_1508_01835_b200 as P
    sc = P.sphere_lattice(1, 2, 1, 0, 3.0)
    f = tmp_path / "s.txt"
    P.scene_to_text(sc, f)
    np.testing.assert_array_equal(P.scene_from_text(f).points, sc.points)
    (tmp_path / "bad.txt").write_text("1 2\n3 4\n")
    with pytest.raises(ValueError):
        P.scene_from_text(tmp_path / "bad.txt")


def test_reference_reports_validate_against_our_schema():
    from paper_1508_01835_b200.reports import validate_report
    gold = json.load(open(os.path.join(GOLDEN, "reports.json")))
    for case in gold.values():
        validate_report(case["report"])
    d = json.loads(json.dumps(next(iter(gold.values()))["report"]))
    del d["timings"]["total"]
    with pytest.raises(ValueError, match="total"):
        validate_report(d)
    d = json.loads(json.dumps(next(iter(gold.values()))["report"]))
    d["schema_version"] = 2
    with pytest.raises(ValueError):
        validate_report(d)
    d = json.loads(json.dumps(next(iter(gold.values()))["report"]))
    d["edge_stats"]["peak_edges"] = True  # bool is not an integer
    with pytest.raises(ValueError):
        validate_report(d)


def test_report_csv_and_json(tmp_path):
    from paper_1508_01835_b200.reports import RunReport, write_csv
    gold = json.load(open(os.path.join(GOLDEN, "reports.json")))["gmres_ifmm"]["report"]
    rep = RunReport(**gold)
    row = rep.csv_row()
    assert row["n_points"] == 300 and row["iterations"] == 5 and row["converged"] is True
    assert row["t_total"] == gold["timings"]["total"]
    write_csv([rep, rep], tmp_path / "r.csv")
    lines = (tmp_path / "r.csv").read_text().strip().splitlines()
    assert len(lines) == 3 and lines[0].startswith("n_points,cheb_nodes,epsilon")
    rep.to_json(tmp_path / "r.json")
    assert json.load(open(tmp_path / "r.json")) == gold


def test_cli_flags_and_config_file(tmp_path):
    from paper_1508_01835_b200.cli import _parse, build_parser, config_from_args
    a = build_parser().parse_args([])
    cfg = config_from_args(a)
    from paper_1508_01835_b200.experiments import RunConfig
    assert cfg == RunConfig()  # flag defaults are the RunConfig defaults (cli.py:17-83)
    f = tmp_path / "c.json"
    f.write_text(json.dumps({"n_points": 777, "epsilon": 1e-5, "lattice": "2,2,3"}))
    a = _parse(["--config", str(f), "--epsilon", "1e-4"])
    cfg = config_from_args(a)
    assert cfg.n_points == 777 and cfg.epsilon == 1e-4 and cfg.lattice_shape == (2, 2, 3)
    f.write_text(json.dumps({"bogus": 1}))
    with pytest.raises(SystemExit):
        _parse(["--config", str(f)])


def test_runconfig_scene_kernel_dispatch():
    from paper_1508_01835_b200.experiments import RunConfig
    assert RunConfig(distribution="shells").scene().points.shape == (42 + 162 + 642, 3)
    assert RunConfig(d_scaling="cube", n_points=8000).effective_d() == pytest.approx(5e-4)
    with pytest.raises(ValueError):
        RunConfig(distribution="torus").scene()
    with pytest.raises(ValueError):
        RunConfig(kernel="laplace").make_kernel()
    with pytest.raises(ValueError):
        RunConfig(d_scaling="x").effective_d()
