"""CLI routing: the reference's config documents, artifacts
and exit codes, running on the B200 engine."""

import csv
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2005_11976_b200 as P
from paper_2005_11976_b200 import cli
from paper_2005_11976_b200 import io as pio

REF = Path(__file__).resolve().parent / "golden" / "io_ref"


def _cfg(tmp_path, name, payload):
    p = tmp_path / name
    p.write_text(json.dumps(payload))
    return str(p)


def test_config_errors_map_to_exit_codes(tmp_path, capsys):
    bad_json = tmp_path / "bad.json"
    bad_json.write_text("{not json")
    assert cli.main(["reconstruct", "--config", str(bad_json), "--out", str(tmp_path)]) == 2
    # schema violation: grid.shape must have 3 entries
    c = _cfg(tmp_path, "c1.json", {"projections": "x", "grid": {"shape": [1, 2],
                                                                 "radius_mm": 1.0,
                                                                 "height_mm": 1.0}})
    assert cli.main(["reconstruct", "--config", c, "--out", str(tmp_path)]) == 2
    # pose estimation is not on the B200 path -> config error, before any I/O
    c = _cfg(tmp_path, "c2.json", {"projections": "x", "grid": {"shape": [2, 4, 2],
                                                                 "radius_mm": 1.0,
                                                                 "height_mm": 1.0}})
    assert cli.main(["reconstruct", "--config", c, "--out", str(tmp_path)]) == 2
    # missing projections file -> io error
    c = _cfg(tmp_path, "c3.json", {"projections": str(tmp_path / "nope"), "pose": {
        "alpha_rad": 0, "beta_rad": 0, "gamma_rad": 0, "t_mm": [0, 0, 0]},
        "grid": {"shape": [2, 4, 2], "radius_mm": 1.0, "height_mm": 1.0}})
    assert cli.main(["reconstruct", "--config", c, "--out", str(tmp_path)]) == 3
    assert "io error" in capsys.readouterr().err


def test_geometry_from_config_matches_reference_defaults():
    g = cli.geometry_from_config({})
    assert (g.sdd, g.sod, g.det_cols, g.det_rows, g.pixel_pitch) == (791.0, 679.0, 96, 192, 0.66)
    assert g.principal_point == (47.5, 95.5) and g.n_proj == 21
    assert np.isclose(g.stage_angles[-1], np.radians(200.0))
    g = cli.geometry_from_config({"n_views": 4, "full_turn": True})
    assert np.allclose(g.stage_angles, [0, np.pi / 2, np.pi, 3 * np.pi / 2])


@pytest.mark.gpu
def test_simulate_then_reconstruct(tmp_path):
    grid = P.CylGrid(8, 16, 8, 4.0, 8.0, P.Pose.tilt(0.3, 0.05, [0.2, 0.0, 0.1]))
    vol = P.CylVolume(grid, np.random.default_rng(1).random(grid.shape) * 0.05)
    pio.write_volume(vol, tmp_path / "truth")
    sim = _cfg(tmp_path, "sim.json", {"volume": str(tmp_path / "truth.json"), "geometry": {
        "sdd_mm": 400.0, "sod_mm": 200.0, "det_cols": 48, "det_rows": 40,
        "pixel_pitch_mm": 0.25, "n_views": 12, "full_turn": True}})
    assert cli.main(["simulate", "--config", sim, "--out", str(tmp_path / "s")]) == 0
    rec = _cfg(tmp_path, "rec.json", {
        "projections": str(tmp_path / "s" / "projections.json"), "pose": grid.pose.to_dict(),
        "grid": {"shape": [8, 16, 8], "radius_mm": 4.0, "height_mm": 8.0},
        "sart": {"relaxation": 0.5, "passes": 3, "subsets": 4}})
    assert cli.main(["reconstruct", "--config", rec, "--out", str(tmp_path / "r")]) == 0
    out = pio.read_volume(tmp_path / "r" / "volume")
    report = json.loads((tmp_path / "r" / "report.json").read_text())
    ps = pio.read_projections(tmp_path / "s" / "projections")
    direct, rep = P.sart_run(ps, grid, P.SartConfig(relaxation=0.5, n_iterations=3,
                                                    n_subsets=4))
    assert np.array_equal(out.mu, direct.mu)
    assert report["residuals"] == rep.residuals
    rows = list(csv.reader(open(tmp_path / "r" / "residuals.csv")))
    assert rows[0] == ["pass", "residual_l2"] and len(rows) == 4


@pytest.mark.gpu
def test_batch_study_small(tmp_path):
    c = _cfg(tmp_path, "b.json", {"n_samples": 4, "recon_shape": [24, 8, 12],
                                  "sim_shape": [24, 8, 12], "strategies": ["a", "c"],
                                  "geometry": {"det_cols": 48, "det_rows": 96}})
    assert cli.main(["batch", "--config", c, "--out", str(tmp_path)]) == 0
    rows = list(csv.reader(open(tmp_path / "batch_results.csv")))
    assert rows[0] == ["sample", "present", "presence_a", "presence_c"] and len(rows) == 5
    assert (tmp_path / "batch_summary.csv").exists()
