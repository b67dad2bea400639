"""Measured parity margins of the FP against the fp64 oracle (the tests only
assert the tolerance): rel-L2 on seeded pixel samples of C1 / C2 / C5 views."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np
import torch

import oracle as orc
import paper_2005_11976_b200 as P
from paper_2005_11976_b200 import workloads as W


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    orc.build()
    for name, wl, views, npx in (("c1", W.c1_small(), (0, 17, 45), 4000),
                                 ("c2", W.c2_medium(), (3, 211), 3000),
                                 ("c5", W.c5_object(0), (7,), 1500)):
        vol = P.CylVolume(wl.grid, torch.as_tensor(wl.mu, device="cuda"))
        errs = []
        for i in views:
            rng = np.random.default_rng(i)
            idx = rng.choice(wl.geom.det_rows * wl.geom.det_cols, npx, replace=False)
            rows, cols = np.divmod(idx, wl.geom.det_cols)
            p_o, _ = orc.forward_pixels(wl.mu, wl.grid, wl.geom, i, rows, cols)
            p = P.forward_project(vol, wl.geom, i).cpu().numpy()[rows, cols]
            errs.append(rel_l2(p, p_o))
        print(name, "FP rel-L2 vs fp64 oracle per view:", ["%.2e" % e for e in errs],
              "(tolerance 1e-4)", flush=True)


if __name__ == "__main__":
    main()
