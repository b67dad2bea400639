"""Parity of the PRODUCTION kernel paths behind the C4 / C5 timings, at full size.

The batched launches that the benchmarks time use the large-volume gather
layouts -- bricked 16-byte GL_QUAD cells for the (512,1024,384) cylinder of
C4 / C5 and 2x2-bricked 32-byte GL_OCTB cells for the 512^3 Cartesian grid of
C4 (``ct_gather_layout_*`` proves which one a case ran) -- and the BP reads
packed footprint quads.  Every case here goes through those exact launches
(``forward_project_all`` with >= GATHER_MIN_VIEWS views, ``SartRun``'s
correction / quad / update launchers) and is compared with the fp64 oracle
(oracle/, pinned to the reference by tests/test_oracle_golden.py):

* FP: sampled pixels of 4 batched views, row sums bit-exact, projections
  <= 1e-4 rel-L2 (north_star);
* BP: 20,000 sampled voxels of one view's num / den against the oracle's
  per-voxel restatement (``oracle.back_voxels``, the same function as the
  whole-volume BP);
* C5 OS-SART subset (20 views, template initial volume, lambda 0.3) through
  SartRun: the corrections' implied simulations at sampled pixels <= 1e-4,
  and the update delta at 20,000 sampled voxels <= 1e-3 against oracle BP
  sums of the same correction images + the reference update rule
  (``recon.py:105-119``).

A whole-volume fp64 BP at these sizes costs ~2 s per view on the host and a
full FP ~4-8 s per view, hence the sampling.
"""

import ctypes as C

import numpy as np
import pytest
import torch

import paper_2005_11976_b200 as P
from paper_2005_11976_b200 import _device as D
from paper_2005_11976_b200 import _native as N
from paper_2005_11976_b200 import workloads as W
from paper_2005_11976_b200.recon import SartRun

pytestmark = pytest.mark.gpu

PROJ_TOL = 1e-4
RECON_TOL = 1e-3
BP_TOL = 1e-4
GL_QUAD, GL_OCTB = 2, 3


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def f32(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def layout(grid):
    lib = N.load_library()
    g = D.grid_c(grid)
    fn = lib.ct_gather_layout_cyl if isinstance(grid, P.CylGrid) else lib.ct_gather_layout_cart
    return fn(C.byref(g))


def sample_pixels(geom, n, seed):
    rng = np.random.default_rng(seed)
    idx = rng.choice(geom.det_rows * geom.det_cols, n, replace=False)
    return np.divmod(idx, geom.det_cols)


def sample_voxels(grid, n, seed):
    return np.sort(np.random.default_rng(seed).choice(grid.n_voxels, n, replace=False))


@pytest.fixture(scope="module")
def c4():
    cyl, cart, geom, ph = W.c4_grids()
    return cyl, cart, geom, W.rasterize_cyl(ph, cyl), W.rasterize_cart(ph, cart)


@pytest.mark.parametrize("kind", ["cyl", "cart"])
def test_c4_batched_fp_production_layout_vs_oracle(oracle, c4, kind):
    """C4 at full size, 4 views in ONE batched launch through the gather
    layout the C4 sweep uses (GL_QUAD bricks for the cylinder, GL_OCTB for
    the Cartesian grid)."""
    cyl, cart, geom, mu_c, mu_x = c4
    grid, mu = (cyl, mu_c) if kind == "cyl" else (cart, mu_x)
    assert layout(grid) == (GL_QUAD if kind == "cyl" else GL_OCTB)
    views = [5, 188, 401, 719]
    sub = geom.subset(views)
    vol = (P.CylVolume if kind == "cyl" else P.CartVolume)(grid, dev(mu))
    assert len(views) >= P.projector.GATHER_MIN_VIEWS
    imgs = P.forward_project_all(vol, sub).images.cpu().numpy()
    # w of the same rays (the plain path: row sums do not depend on the layout)
    for b, i in enumerate(views):
        rows, cols = sample_pixels(geom, 1200, i)
        p_o, w_o = oracle.forward_pixels(mu, grid, geom, i, rows, cols)
        _, w = P.forward_project(vol, geom, i, return_weights=True)
        assert np.array_equal(w.cpu().numpy()[rows, cols], f32(w_o))
        assert rel_l2(imgs[b][rows, cols], p_o) < PROJ_TOL, (kind, i)


def test_c4_cyl_bp_vs_oracle_sampled_voxels(oracle, c4):
    """C4 cylindrical BP (201M voxels, 768^2 detector) of one view: the plain
    BP and the quad-footprint BP that SART uses, at 20k sampled voxels."""
    cyl, _, geom, _, _ = c4
    i = 311
    corr = np.random.default_rng(41).normal(0, 0.01, (geom.det_rows, geom.det_cols))
    corr = corr.astype(np.float32)
    idx = sample_voxels(cyl, 20000, 41)
    n_o, d_o = oracle.back_voxels(corr, geom, i, cyl, idx)
    assert (d_o > 0).mean() > 0.9
    num, den = P.back_project(dev(corr), geom, i, cyl)
    t_idx = torch.as_tensor(idx, device="cuda")
    assert rel_l2(num.view(-1)[t_idx].cpu().numpy(), n_o) < BP_TOL
    assert rel_l2(den.view(-1)[t_idx].cpu().numpy(), d_o) < BP_TOL
    # the production BP: packed quads, batch slot table
    from paper_2005_11976_b200.recon import SartEngine
    eng = SartEngine(cyl, geom, P.RaySamplingConfig(), views=[i])
    quads = eng.alloc_quads(1)
    c = dev(corr).view(1, geom.det_rows, geom.det_cols)
    eng.pack_quads(c, 1, quads)
    num2 = torch.empty(cyl.shape, device="cuda")
    den2 = torch.empty(cyl.shape, device="cuda")
    eng.bp_partial(c, D.upload_i32([0]), 1, num2, den2, quads)
    assert rel_l2(num2.view(-1)[t_idx].cpu().numpy(), n_o) < BP_TOL
    assert rel_l2(den2.view(-1)[t_idx].cpu().numpy(), d_o) < BP_TOL


def test_c4_cart_bp_vs_oracle_sampled_voxels(oracle, c4):
    _, cart, geom, _, _ = c4
    i = 77
    corr = np.random.default_rng(42).normal(0, 0.01, (geom.det_rows, geom.det_cols))
    corr = corr.astype(np.float32)
    idx = sample_voxels(cart, 20000, 42)
    n_o, d_o = oracle.back_voxels(corr, geom, i, cart, idx)
    num, den = P.back_project(dev(corr), geom, i, cart)
    t_idx = torch.as_tensor(idx, device="cuda")
    assert rel_l2(num.view(-1)[t_idx].cpu().numpy(), n_o) < BP_TOL
    assert rel_l2(den.view(-1)[t_idx].cpu().numpy(), d_o) < BP_TOL


@pytest.fixture(scope="module")
def c5_run():
    """One C5 object and its SartRun (template init, 6 subsets, lambda 0.3),
    measured data = our batched FP of the object (noise-free)."""
    wl = W.c5_object(7)
    vol = P.CylVolume(wl.grid, dev(wl.mu))
    ps = P.forward_project_all(vol, wl.geom)
    template = W.c5_template()
    cfg = P.SartConfig(relaxation=wl.relaxation, n_iterations=1, n_subsets=wl.n_subsets,
                       initial=P.CylVolume(wl.grid, dev(template)), compute_residuals=False)
    run = SartRun(ps, wl.grid, cfg)
    del vol
    return wl, ps, template, run


def test_c5_os_subset_update_production_path_vs_oracle(oracle, c5_run):
    """The C5 bench's subset step at full size: bricked GL_QUAD correction FP
    over the subset's 20 views, quad packing, fused BP update."""
    wl, ps, template, run = c5_run
    assert layout(wl.grid) == GL_QUAD
    e = run.eng
    s, slots = run.subsets[0], run.subset_slots[0]
    n = len(s)
    assert n == 20
    mu0 = run.mu.clone()
    e.pack(run.mu, run.gather)
    e.correction(run.mu, run.p_meas, slots, n, run.corr, run.gather)
    corr = run.corr[:n].cpu().numpy()
    e.pack_quads(run.corr, n, run.quads)
    e.bp_update(run.corr, slots, n, run.upd, run.quads)
    torch.cuda.synchronize()
    images = ps.images
    # (a) corrections: c = (p - sim) / w on valid rays (recon.py:96-102); the
    # implied simulation sim = p - c w is a projection -> 1e-4 rel-L2
    max_row = e.row_max()
    sims_o, sims = [], []
    for b, i in enumerate(s):
        i = int(i)
        rows, cols = sample_pixels(wl.geom, 600, 100 + i)
        sim_o, w_o = oracle.forward_pixels(template, wl.grid, wl.geom, i, rows, cols)
        valid = w_o > 1e-6 * max_row[i]
        p = images[i].cpu().numpy()[rows, cols].astype(np.float64)
        c = corr[b][rows, cols].astype(np.float64)
        c_o = np.where(valid, (p - sim_o) / np.where(valid, w_o, 1.0), 0.0)
        assert np.array_equal(c[~valid], c_o[~valid])
        sims.append((p - c * w_o)[valid])
        sims_o.append(sim_o[valid])
    assert rel_l2(np.concatenate(sims), np.concatenate(sims_o)) < PROJ_TOL
    # (b) the fused update at sampled voxels: oracle BP sums of the same
    # correction images + the reference update rule.  The update from the
    # template is sparse (rays through the added / missing inclusions), so
    # half the samples are drawn among the voxels the subset changed.
    changed = torch.nonzero((run.mu != mu0).view(-1)).view(-1).cpu().numpy()
    assert changed.size > 10000
    rng = np.random.default_rng(5)
    idx = np.unique(np.concatenate([sample_voxels(wl.grid, 10000, 5),
                                    rng.choice(changed, 10000, replace=False)]))
    num = np.zeros(idx.size)
    den = np.zeros(idx.size)
    for b, i in enumerate(s):
        oracle.back_voxels(corr[b], wl.geom, int(i), wl.grid, idx, out=(num, den))
    mu_o = template.reshape(-1)[idx].astype(np.float64)
    mu_start = mu_o.copy()
    oracle._apply_update(mu_o, num, den, None, wl.relaxation, True)
    t_idx = torch.as_tensor(idx, device="cuda")
    got = run.mu.view(-1)[t_idx].cpu().numpy().astype(np.float64)
    start = mu0.view(-1)[t_idx].cpu().numpy().astype(np.float64)
    assert np.array_equal(start, f32(mu_start))
    assert (den > 0).mean() > 0.99
    delta_o = mu_o - mu_start
    assert np.count_nonzero(delta_o) > 0.4 * idx.size                  # a real update
    assert rel_l2(got - start, delta_o) < RECON_TOL


def test_c5_full_pass_residual_consistency(c5_run):
    """The rest of the C5 pass (subsets 2-6) and the residual FP on the
    production path: a second run from the same start reproduces the first
    bit for bit, and the residual equals the norm of the stacked residual
    images of an independent batched FP of the result."""
    wl, ps, template, _ = c5_run
    cfg = P.SartConfig(relaxation=wl.relaxation, n_iterations=1, n_subsets=wl.n_subsets,
                       initial=P.CylVolume(wl.grid, dev(template)))
    out1, rep1 = SartRun(ps, wl.grid, cfg).run()
    out2, rep2 = SartRun(ps, wl.grid, cfg).run()
    assert torch.equal(out1.mu, out2.mu)
    assert rep1.residuals == rep2.residuals
    sim = P.forward_project_all(out1, wl.geom).images
    r = float(torch.linalg.vector_norm((ps.images.double() - sim.double())))
    assert rep1.residuals[0] == pytest.approx(r, rel=1e-9)
