"""CLI routing: the reference's config documents, artifacts
and exit codes, running on the B200 engine."""

import csv
import json
import warnings
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
    # default pose = "estimate": projections are read first (reference order) -> io error
    c = _cfg(tmp_path, "c2.json", {"projections": str(tmp_path / "x"),
                                   "grid": {"shape": [2, 4, 2], "radius_mm": 1.0,
                                            "height_mm": 1.0}})
    assert cli.main(["reconstruct", "--config", c, "--out", str(tmp_path)]) == 3
    # pose needs projections (the reference's precision study is out of scope)
    c = _cfg(tmp_path, "p.json", {"study": {"noise_sigma": 0.1}})
    assert cli.main(["pose", "--config", c, "--out", str(tmp_path)]) == 2
    # missing projections file -> io error
    c = _cfg(tmp_path, "c3.json", {"projections": str(tmp_path / "nope"), "pose": {
        "alpha_rad": 0, "beta_rad": 0, "gamma_rad": 0, "t_mm": [0, 0, 0]},
        "grid": {"shape": [2, 4, 2], "radius_mm": 1.0, "height_mm": 1.0}})
    assert cli.main(["reconstruct", "--config", c, "--out", str(tmp_path)]) == 3
    assert "io error" in capsys.readouterr().err


def test_pose_params_from_config():
    p = cli.pose_params_from_config({"threshold_level": 1.8, "threshold_levels": 9,
                                     "threshold_span": 1.0, "exclude_rects": [[0, 5, 0, 9]],
                                     "lm": {"max_iterations": 7}})
    assert p.levels()[0] == pytest.approx(0.8) and p.exclude_rects == ((0, 5, 0, 9),)
    assert p.lm.max_iterations == 7 and p.band == 1 and p.nuisance_level is None
    assert cli.pose_params_from_config({}).threshold_level == "auto"


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
                                  "pose_source": "true",
                                  "geometry": {"det_cols": 48, "det_rows": 96}})
    assert cli.main(["batch", "--config", c, "--out", str(tmp_path)]) == 0
    rows = list(csv.reader(open(tmp_path / "batch_results.csv")))
    assert rows[0] == ["sample", "present", "presence_a", "presence_c"] and len(rows) == 5
    assert (tmp_path / "batch_summary.csv").exists()


@pytest.mark.gpu
def test_pose_then_reconstruct_with_estimated_pose(tmp_path):
    """cyltomo pose -> pose.json; reconstruct with pose = "estimate" uses the
    same fit (cyltomo/cli.py:286-313, 351-355)."""
    import math
    true = P.Pose(alpha=0.6, beta=math.radians(3.0), t=[1.0, -1.5, 0.5])
    geom = cli.geometry_from_config({})
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        vol = P.make_assembly_phantom(cli._device_components(True),
                                      P.CylGrid(60, 16, 32, 8.0, 60.0, true))
    ps = P.simulate_scan(vol, geom, P.RaySamplingConfig())
    pio.write_projections(ps, tmp_path / "proj")
    params = cli.DEVICE_POSE_PARAMS
    c = _cfg(tmp_path, "pose.json", {"projections": str(tmp_path / "proj.json"),
                                     "params": params})
    assert cli.main(["pose", "--config", c, "--out", str(tmp_path / "p")]) == 0
    doc = json.loads((tmp_path / "p" / "pose.json").read_text())
    assert abs(doc["beta_rad"] - true.beta) < math.radians(0.2)
    assert np.abs(np.array(doc["t_mm"]) - true.t).max() < 0.2
    direct = P.fit_pose(pio.read_projections(tmp_path / "proj"), P.PoseFitParams(**params))
    assert doc["alpha_rad"] == direct.pose.alpha and doc["t_mm"] == list(direct.pose.t)
    rec = _cfg(tmp_path, "rec.json", {
        "projections": str(tmp_path / "proj.json"), "pose": "estimate", "pose_params": params,
        "grid": {"shape": [24, 8, 12], "radius_mm": 8.0, "height_mm": 60.0},
        "sart": {"passes": 1}})
    assert cli.main(["reconstruct", "--config", rec, "--out", str(tmp_path / "r")]) == 0
    report = json.loads((tmp_path / "r" / "report.json").read_text())
    assert report["pose"]["alpha_rad"] == direct.pose.alpha


@pytest.mark.gpu
def test_reconstruct_matches_reference_cli_artifacts(tmp_path, monkeypatch):
    """`reconstruct` on the reference-written projections and config document
    (tests/golden/make_golden_cli.py ran the unmodified reference CLI,
    cyltomo/cli.py:341-397): same artifacts, same report schema and pose
    echo, volume and residuals within the north_star reconstruction
    tolerance."""
    import shutil
    src = Path(__file__).resolve().parent / "golden" / "cli_ref"
    work = tmp_path / "cli_ref"
    shutil.copytree(src, work)
    monkeypatch.chdir(work)
    assert cli.main(["reconstruct", "--config", "reconstruct.json", "--out", "ours"]) == 0
    ref_vol = pio.read_volume(work / "volume.json")
    our_vol = pio.read_volume(work / "ours" / "volume.json")
    a, b = np.asarray(our_vol.mu, np.float64), np.asarray(ref_vol.mu, np.float64)
    assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-3
    ref_rep = json.loads((work / "report.json").read_text())
    our_rep = json.loads((work / "ours" / "report.json").read_text())
    assert set(ref_rep) == set(our_rep)
    assert our_rep["pose"] == ref_rep["pose"]
    for k, v in ref_rep["config"].items():
        assert our_rep["config"][k] == v, k
    assert np.allclose(our_rep["residuals"], ref_rep["residuals"], rtol=1e-3)
    ref_rows = list(csv.reader(open(work / "residuals.csv")))
    our_rows = list(csv.reader(open(work / "ours" / "residuals.csv")))
    assert our_rows[0] == ref_rows[0] and [r[0] for r in our_rows] == [r[0] for r in ref_rows]
    assert np.allclose([float(r[1]) for r in our_rows[1:]],
                       [float(r[1]) for r in ref_rows[1:]], rtol=1e-3)
    # the volume header the reference reader expects
    assert json.loads((work / "ours" / "volume.json").read_text()).keys() == \
        json.loads((work / "volume.json").read_text()).keys()


def test_reference_flags_preset_and_threads(tmp_path, monkeypatch):
    """The reference's common flags parse (cyltomo/cli.py:551-555), --preset
    paper selects the paper-scale simulation geometry (:250-252) and --threads
    caps the host worker pool."""
    seen = {}

    class Stop(Exception):
        pass

    def fake_sim(vol, geom, *a, **k):
        seen["geom"] = geom
        raise Stop

    monkeypatch.setattr(cli.io, "read_volume", lambda *a, **k: None)
    monkeypatch.setattr(cli, "simulate_scan", fake_sim)
    monkeypatch.delenv("CT_HOST_THREADS", raising=False)
    c = _cfg(tmp_path, "s.json", {"volume": "v.json"})
    with pytest.raises(Stop):
        cli.main(["simulate", "--preset", "paper", "--threads", "3", "--config", c])
    g = seen["geom"]
    assert (g.n_proj, g.det_cols, g.det_rows, g.pixel_pitch) == (4096, 2048, 128, 0.0096)
    assert np.isclose(g.stage_angles[1] - g.stage_angles[0], 2 * np.pi / 4096)
    import os
    assert os.environ["CT_HOST_THREADS"] == "3"
    with pytest.raises(Stop):
        cli.main(["simulate", "--preset", "desk", "--config", c])
    assert seen["geom"].n_proj == 21
    args = cli.build_parser().parse_args(["reconstruct", "--threads", "2", "--preset", "desk",
                                          "--init", "none"])
    assert args.threads == 2 and args.preset == "desk" and args.init == "none"


def test_config_merge_semantics():
    base = {"a": 1, "g": {"x": 1, "y": {"p": 1, "q": 2}}, "l": [1, 2]}
    got = cli.merged(base, {"g": {"y": {"q": 3}, "z": 4}, "l": [9], "b": None})
    assert got == {"a": 1, "g": {"x": 1, "y": {"p": 1, "q": 3}, "z": 4}, "l": [9], "b": None}
    assert base["g"]["y"]["q"] == 2                       # defaults untouched


@pytest.mark.gpu
def test_batch_with_estimated_poses(tmp_path):
    c = _cfg(tmp_path, "b.json", {"n_samples": 4, "recon_shape": [48, 8, 12],
                                  "sim_shape": [60, 16, 32], "strategies": ["a"],
                                  "pose_source": "estimated"})
    assert cli.main(["batch", "--config", c, "--out", str(tmp_path)]) == 0
    rows = list(csv.reader(open(tmp_path / "batch_results.csv")))
    assert len(rows) == 5
