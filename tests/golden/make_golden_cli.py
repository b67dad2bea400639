"""Reference-written CLI artifacts for the `reconstruct` parity test
(tests/test_cli.py::test_reconstruct_matches_reference_cli_artifacts).

Runs the UNMODIFIED reference CLI (cyltomo/cli.py:248-265 simulate,
:341-397 reconstruct) in the build container and keeps its outputs under
tests/golden/cli_ref/:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_golden_cli.py
"""

from __future__ import annotations

import json
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent / "cli_ref"

import cyltomo as ref  # noqa: E402  (the reference, from PYTHONPATH)
from cyltomo import io as rio  # noqa: E402

POSE = {"alpha_rad": 0.3, "beta_rad": 0.05, "gamma_rad": 0.0, "t_mm": [0.2, 0.0, 0.1]}
GRID = {"shape": [8, 16, 8], "radius_mm": 4.0, "height_mm": 8.0}
GEOMETRY = {"sdd_mm": 400.0, "sod_mm": 200.0, "det_cols": 48, "det_rows": 40,
            "pixel_pitch_mm": 0.25, "n_views": 12, "full_turn": True}
SART = {"relaxation": 0.5, "passes": 3}


def run(*argv, cwd):
    subprocess.run([sys.executable, "-m", "cyltomo.cli", *argv], check=True, cwd=cwd)


def main():
    if OUT.exists():
        shutil.rmtree(OUT)
    OUT.mkdir(parents=True)
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        grid = ref.CylGrid(8, 16, 8, 4.0, 8.0, pose=ref.Pose.from_dict(POSE))
        mu = np.random.default_rng(1).random(grid.shape).astype(np.float32).astype(float) * 0.05
        rio.write_volume(ref.CylVolume(grid, mu), OUT / "truth")
        (OUT / "simulate.json").write_text(json.dumps(
            {"volume": "truth.json", "geometry": GEOMETRY}, indent=1))
        run("simulate", "--config", str(OUT / "simulate.json"), "--out", str(tmp / "s"),
            cwd=OUT)
        for f in ("projections.json", "projections.raw"):
            shutil.copy(tmp / "s" / f, OUT / f)
        (OUT / "reconstruct.json").write_text(json.dumps(
            {"projections": "projections.json", "pose": POSE, "grid": GRID, "sart": SART},
            indent=1))
        run("reconstruct", "--config", str(OUT / "reconstruct.json"), "--out",
            str(tmp / "r"), cwd=OUT)
        for f in ("volume.json", "volume.raw", "report.json", "residuals.csv"):
            shutil.copy(tmp / "r" / f, OUT / f)
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
