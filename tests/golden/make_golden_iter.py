"""Golden fixtures for WHOLE reconstruction iterations at full config size,
produced by the pinned CPU oracle (oracle/, itself pinned to the unmodified
reference by tests/test_oracle_golden.py).  TEST INFRASTRUCTURE ONLY.

The fp64 oracle needs ~35 min (8 cores) for one C2 OS-SART iteration and
~6 min for two C3 SART passes, far too slow for the GPU test run, so the
results are committed (tests/test_gpu_iterations.py reads them):

* golden_c2_iter.npz -- BASELINE configs[1] (C2): (256,512,256) grid, 360
  views on 512^2, ONE full OS-SART iteration (8 interleaved subsets, lambda
  0.3, nonnegativity) from a zero volume, measured data = the oracle's own
  noise-free projections of the seeded C2 phantom; stores the pass residual,
  20,000 seeded voxel samples, two whole h layers (fp32) and the sha256 of
  the fp64 volume.
* golden_c3_iter.npz -- BASELINE configs[2] (C3): 30 views, per-view SART,
  weight map (1.0 ROI / 0.2), template initial volume, lambda 0.5, TWO
  passes (SURVEY.md §8c's plan); the same kinds of samples.
* golden_c5_iter.npz -- BASELINE configs[4] (C5), object 0: (512,1024,384)
  grid, 120 views on 1024^2, ONE full OS-SART iteration (6 subsets, lambda
  0.3) from the shared template (~40 min on 8 cores); 20,000 voxel samples
  (half seeded, half where the update from the template is largest), the
  h layer with the largest update, the pass residual.

The phantoms, poses and weight maps are pure functions of committed seeded
code (paper_2005_11976_b200.workloads); their sha256 is stored so a drift in
the generator is detected.

    python tests/golden/make_golden_iter.py [c2] [c3]
"""

from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
ROOT = OUT.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import oracle as orc  # noqa: E402
from paper_2005_11976_b200 import workloads as W  # noqa: E402

N_SAMPLES = 20000
LAYERS = (64, 192)


def sha(a, dtype=np.float32) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dtype).tobytes()).hexdigest()


def oracle_projections(wl):
    t = time.time()
    imgs = np.empty((wl.geom.n_proj, wl.geom.det_rows, wl.geom.det_cols), np.float32)
    for i in range(wl.geom.n_proj):
        imgs[i] = orc.forward(wl.mu, wl.grid, wl.geom, i)[0]
    print(f"  projections {time.time() - t:.0f} s", flush=True)
    return imgs


def samples(mu, seed):
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(mu.size, N_SAMPLES, replace=False))
    return idx, mu.reshape(-1)[idx]


def c2():
    wl = W.c2_medium()
    imgs = oracle_projections(wl)
    t = time.time()
    mu, res = orc.sart(imgs, wl.grid, wl.geom, relaxation=wl.relaxation, n_iterations=1,
                       n_subsets=wl.n_subsets)
    print(f"  C2 OS-SART iteration {time.time() - t:.0f} s, residual {res}", flush=True)
    idx, val = samples(mu, 2)
    np.savez_compressed(OUT / "golden_c2_iter.npz", residuals=np.array(res), idx=idx, val=val,
                        layers=np.array(LAYERS),
                        layer_mu=mu[list(LAYERS)].astype(np.float32),
                        mu_sha=sha(mu, np.float64), phantom_sha=sha(wl.mu),
                        images_sha=sha(imgs), norm=np.linalg.norm(mu))


def c3():
    wl = W.c3_sparse()
    imgs = oracle_projections(wl)
    t = time.time()
    mu, res = orc.sart(imgs, wl.grid, wl.geom, relaxation=wl.relaxation, n_iterations=2,
                       weights=wl.weights, initial=wl.template)
    print(f"  C3 2 SART passes {time.time() - t:.0f} s, residuals {res}", flush=True)
    idx, val = samples(mu, 3)
    np.savez_compressed(OUT / "golden_c3_iter.npz", residuals=np.array(res), idx=idx, val=val,
                        layers=np.array(LAYERS),
                        layer_mu=mu[list(LAYERS)].astype(np.float32),
                        mu_sha=sha(mu, np.float64), phantom_sha=sha(wl.mu),
                        weights_sha=sha(wl.weights), template_sha=sha(wl.template),
                        images_sha=sha(imgs), norm=np.linalg.norm(mu))


def c5():
    wl = W.c5_object(0)
    template = W.c5_template()
    imgs = oracle_projections(wl)
    t = time.time()
    mu, res = orc.sart(imgs, wl.grid, wl.geom, relaxation=wl.relaxation, n_iterations=1,
                       n_subsets=wl.n_subsets, initial=template)
    print(f"  C5 OS-SART iteration {time.time() - t:.0f} s, residual {res}", flush=True)
    upd = np.abs(mu - template).reshape(-1)
    rng = np.random.default_rng(5)
    top = np.argpartition(upd, -N_SAMPLES // 2)[-N_SAMPLES // 2:]
    rest = np.setdiff1d(np.arange(mu.size), top)
    idx = np.sort(np.concatenate([top, rng.choice(rest, N_SAMPLES // 2, replace=False)]))
    # the h layer the update from the template is largest in (the changed inclusion)
    layer = int(np.argmax(np.abs(mu - template).sum(axis=(1, 2))))
    np.savez_compressed(OUT / "golden_c5_iter.npz", residuals=np.array(res), idx=idx,
                        val=mu.reshape(-1)[idx], layers=np.array([layer]),
                        layer_mu=mu[[layer]].astype(np.float32),
                        mu_sha=sha(mu, np.float64), phantom_sha=sha(wl.mu),
                        template_sha=sha(template), images_sha=sha(imgs),
                        norm=np.linalg.norm(mu))


if __name__ == "__main__":
    which = sys.argv[1:] or ["c3", "c2"]
    for name in which:
        print(name, flush=True)
        globals()[name]()
