"""Whole reconstruction iterations at full config size against committed
oracle goldens (tests/golden/make_golden_iter.py: the pinned fp64 oracle,
~35 min of host time for C2, too slow to run with the GPU suite).

* C2 (BASELINE configs[1]): ONE complete OS-SART iteration -- 8 interleaved
  subsets of 45 views, lambda 0.3, from zero, residual FP -- vs the oracle's
  volume (20,000 seeded voxels + two whole h layers) and pass residual.
* C3 (configs[2]): TWO per-view SART passes over 30 views with the weight map
  and the template initial volume, vs the oracle's volumes' update from the
  template and residuals.

The golden's measured data are the oracle's own projections of the seeded
phantom; here the projections come from our batched FP of the same phantom
(<= 2e-6 rel-L2 apart, tools/parity_margins.py), so the comparison also
carries the FP's error through the iteration -- far inside the 1e-3
reconstruction tolerance of north_star.
"""

import hashlib

import numpy as np
import pytest
import torch

import paper_2005_11976_b200 as P
from paper_2005_11976_b200 import workloads as W

pytestmark = pytest.mark.gpu

RECON_TOL = 1e-3


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def load(name):
    from conftest import load_golden
    return load_golden(name)


def _samples(mu, g):
    flat = mu.reshape(-1)
    idx = torch.as_tensor(g["idx"], device=mu.device)
    return flat[idx].cpu().numpy().astype(np.float64)


def test_c2_full_os_sart_iteration_vs_oracle_golden():
    g = load("golden_c2_iter.npz")
    wl = W.c2_medium()
    assert sha(wl.mu) == str(g["phantom_sha"])          # the generator did not drift
    vol = P.CylVolume(wl.grid, dev(wl.mu))
    ps = P.forward_project_all(vol, wl.geom)
    del vol
    out, rep = P.sart_run(ps, wl.grid, P.SartConfig(relaxation=wl.relaxation, n_iterations=1,
                                                     n_subsets=wl.n_subsets))
    mu = out.mu
    assert rel_l2(_samples(mu, g), g["val"]) < RECON_TOL
    layers = mu[torch.as_tensor(g["layers"], device="cuda")].cpu().numpy()
    assert rel_l2(layers, g["layer_mu"]) < RECON_TOL
    assert float(torch.linalg.vector_norm(mu.double())) == pytest.approx(float(g["norm"]),
                                                                          rel=RECON_TOL)
    assert rep.residuals[0] == pytest.approx(float(g["residuals"][0]), rel=RECON_TOL)


def test_c3_two_weighted_template_passes_vs_oracle_golden():
    g = load("golden_c3_iter.npz")
    wl = W.c3_sparse()
    assert sha(wl.mu) == str(g["phantom_sha"])
    assert sha(wl.weights) == str(g["weights_sha"])
    assert sha(wl.template) == str(g["template_sha"])
    vol = P.CylVolume(wl.grid, dev(wl.mu))
    ps = P.forward_project_all(vol, wl.geom)
    cfg = P.SartConfig(relaxation=wl.relaxation, n_iterations=2, weights=wl.weights,
                       initial=P.CylVolume(wl.grid, dev(wl.template)))
    out, rep = P.sart_run(ps, wl.grid, cfg)
    mu = out.mu
    # the update from the template (the template itself would dominate mu)
    t = dev(wl.template)
    start = _samples(t, g)
    assert rel_l2(_samples(mu, g) - start, g["val"] - start) < RECON_TOL
    li = torch.as_tensor(g["layers"], device="cuda")
    d_layers = (mu[li] - t[li]).cpu().numpy()
    assert rel_l2(d_layers, g["layer_mu"].astype(np.float64) - wl.template[g["layers"]]) \
        < RECON_TOL
    assert np.allclose(rep.residuals, g["residuals"], rtol=RECON_TOL)


def test_c5_full_os_sart_iteration_vs_oracle_golden():
    """BASELINE configs[4] (the headline workload), object 0: ONE complete
    OS-SART iteration (6 subsets of 20 views on 1024^2, lambda 0.3, from the
    shared template, residual FP) through the production path (bricked
    GL_QUAD layout, quad BP) vs the oracle: the update from the template at
    20,000 voxels (half of them where it is largest), over the whole h layer
    where it is largest, and the pass residual."""
    g = load("golden_c5_iter.npz")
    wl = W.c5_object(0)
    template = W.c5_template()
    assert sha(wl.mu) == str(g["phantom_sha"])
    assert sha(template) == str(g["template_sha"])
    vol = P.CylVolume(wl.grid, dev(wl.mu))
    ps = P.forward_project_all(vol, wl.geom)
    del vol
    t = dev(template)
    cfg = P.SartConfig(relaxation=wl.relaxation, n_iterations=1, n_subsets=wl.n_subsets,
                       initial=P.CylVolume(wl.grid, t))
    out, rep = P.sart_run(ps, wl.grid, cfg)
    mu = out.mu
    start = _samples(t, g)
    assert rel_l2(_samples(mu, g) - start, g["val"] - start) < RECON_TOL
    li = torch.as_tensor(g["layers"], device="cuda")
    d_layer = (mu[li] - t[li]).cpu().numpy()
    assert rel_l2(d_layer, g["layer_mu"].astype(np.float64) - template[g["layers"]]) < RECON_TOL
    assert rep.residuals[0] == pytest.approx(float(g["residuals"][0]), rel=RECON_TOL)
