"""Artifact files: byte-compatible with the reference's
cyltomo/io.py in both directions (tests/golden/io_ref/ was written by the
unmodified reference), bit-exact round trips, and the reference's errors."""

import json
import math
import shutil
from pathlib import Path

import numpy as np
import pytest

import paper_2005_11976_b200 as P
from paper_2005_11976_b200 import io as pio
from paper_2005_11976_b200.errors import SchemaMismatch, SizeMismatch

REF = Path(__file__).resolve().parent / "golden" / "io_ref"


def test_reads_reference_artifacts(golden_small):
    vol = pio.read_volume(REF / "cylvol.json")
    assert isinstance(vol, P.CylVolume)
    assert vol.grid.shape == (3, 5, 4)
    assert np.array_equal(vol.mu.ravel(), np.fromfile(REF / "cylvol.raw", dtype="<f4"))
    assert np.array_equal(vol.grid.rotation, golden_small["geo_rotation"])
    cart = pio.read_volume(REF / "cartvol")
    assert isinstance(cart, P.CartVolume) and cart.grid.shape == (2, 3, 4)
    ps = pio.read_projections(REF / "proj.json")
    assert ps.images.shape == (8, 33, 65) and ps.kind == "line_integral"
    assert np.array_equal(ps.images.ravel(), np.fromfile(REF / "proj.raw", dtype="<f4"))
    geom = pio.read_geometry(REF / "geom.json")
    assert np.array_equal(geom.stage_angles, ps.geom.stage_angles)
    pose = pio.read_pose(REF / "pose.json")
    assert np.array_equal(pose.rotation(), golden_small["geo_rotation"])


def test_writes_reference_identical_files(tmp_path):
    """Re-writing the reference's artifacts reproduces them byte for byte."""
    for name in ("cylvol", "cartvol", "proj"):
        obj = (pio.read_projections if name == "proj" else pio.read_volume)(REF / name)
        (pio.write_projections if name == "proj" else pio.write_volume)(obj, tmp_path / name)
        assert (tmp_path / f"{name}.raw").read_bytes() == (REF / f"{name}.raw").read_bytes()
        assert json.loads((tmp_path / f"{name}.json").read_text()) == \
            json.loads((REF / f"{name}.json").read_text())


def test_round_trip_bit_exact(tmp_path, rng):
    grid = P.CylGrid(4, 6, 5, 2.0, 3.0, P.Pose(0.1, 0.2, 0.3, t=[1, 2, 3]))
    vol = P.CylVolume(grid, rng.random(grid.shape))
    pio.write_volume(vol, tmp_path / "v.json")
    back = pio.read_volume(tmp_path / "v")
    assert np.array_equal(back.mu, vol.mu)
    assert back.grid.to_dict() == grid.to_dict()


def test_errors(tmp_path):
    m = json.loads((REF / "cylvol.json").read_text())
    m["raw"] = "a.raw"
    (tmp_path / "a.json").write_text(json.dumps(m))
    (tmp_path / "a.raw").write_bytes(b"\0" * 8)
    with pytest.raises(SizeMismatch):
        pio.read_volume(tmp_path / "a")
    m = json.loads((REF / "cylvol.json").read_text())
    m["schema_version"] = 2
    (tmp_path / "b.json").write_text(json.dumps(m))
    with pytest.raises(SchemaMismatch):
        pio.read_volume(tmp_path / "b")
    m["schema_version"] = 1
    m["kind"] = "projections"
    (tmp_path / "c.json").write_text(json.dumps(m))
    with pytest.raises(SchemaMismatch):
        pio.read_volume(tmp_path / "c")


def test_pgm_round_trip(tmp_path):
    img = (np.arange(12).reshape(3, 4) * 5000).astype(np.uint16)
    pio.write_pgm(img, tmp_path / "x.pgm", maxval=65535)
    assert np.array_equal(pio.read_pgm(tmp_path / "x.pgm"), img)


@pytest.mark.gpu
def test_device_read_and_beer_lambert(tmp_path):
    import torch
    ps = pio.read_projections(REF / "proj", device=True)
    assert ps.on_device
    host = pio.read_projections(REF / "proj")
    assert np.array_equal(ps.images.cpu().numpy(), host.images)
    vol = pio.read_volume(REF / "cylvol", device=True)
    assert vol.on_device
    # Beer-Lambert kernel with an (H, W) flat field broadcast over views
    geom = host.geom
    flat = np.linspace(900.0, 1100.0, geom.det_rows * geom.det_cols).reshape(
        geom.det_rows, geom.det_cols)
    p = host.images.astype(np.float64) * 3.0
    inten = P.ProjectionSet(geom, (np.exp(-p) * flat).astype(np.float32), kind="intensity")
    out = P.intensities_to_line_integrals(inten, flat)
    expect = -np.log(inten.images.astype(np.float64) / flat.astype(np.float32))
    assert np.abs(out.images - expect).max() < 1e-5
