"""Pose step on the GPU: the segmentation kernels
(ct_image_minmax / ct_image_histogram / ct_threshold_dilate / ct_row_extents /
ct_row_extents_levels / ct_strip_profiles) against the oracle, and fit_pose
end to end against the reference's outputs (tests/golden/golden_pose.npz).

Integer/index work (histograms, masks, extents, axis observations) must be
bit-exact; the strip means are fp64 sums in a different order than numpy's
pairwise mean (1e-12 relative)."""

import math
import sys
import warnings
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))

import pose_oracle as O  # noqa: E402
import paper_2005_11976_b200 as P  # noqa: E402
from paper_2005_11976_b200 import imgproc as IP  # noqa: E402
from paper_2005_11976_b200.errors import (DegenerateHistogram, DegenerateMask,  # noqa: E402
                                          EmptyResult, FlatSignal, NoConvergenceWarning,
                                          OutOfFrame)

pytestmark = pytest.mark.gpu

G = np.load(ROOT / "tests" / "golden" / "golden_pose.npz")
from test_pose import CASES, extents, oracle_kwargs, pose_geometry  # noqa: E402


def ps_a():
    return P.ProjectionSet(pose_geometry(), G["pose_img_a"])


def test_minmax_and_histograms_match_numpy(rng):
    imgs = np.concatenate([G["pose_img_a"], G["pose_img_b"]])
    imgs[3, :5, :5] = -7.25                    # negative values through the key transform
    vs = IP.ViewStack(imgs)
    lo, hi = vs.minmax()
    assert np.array_equal(lo, imgs.reshape(len(imgs), -1).min(1).astype(np.float64))
    assert np.array_equal(hi, imgs.reshape(len(imgs), -1).max(1).astype(np.float64))
    for bins in (256, 7, 1000):
        counts = vs.histograms(lo, hi, bins)
        for v in range(len(imgs)):
            want, _ = np.histogram(imgs[v].astype(np.float64), bins=bins, range=(lo[v], hi[v]))
            assert np.array_equal(counts[v], want), (bins, v)
    # values exactly on bin edges and the right edge
    x = np.linspace(0.0, 1.0, 257, dtype=np.float32)[None, None, :]
    vs = IP.ViewStack(x)
    want, _ = np.histogram(x[0, 0].astype(np.float64), bins=256, range=(0.0, 1.0))
    assert np.array_equal(vs.histograms([0.0], [1.0], 256)[0], want)


def test_otsu_levels_match_reference():
    imgs = np.concatenate([G["pose_img_a"], G["pose_img_b"]])
    assert np.array_equal(IP.ViewStack(imgs).otsu_levels(), G["pose_otsu"])
    assert P.otsu_level(G["pose_img_a"][4]) == G["pose_otsu"][4]
    with pytest.raises(DegenerateHistogram):
        P.otsu_level(np.full((5, 5), 1.0, dtype=np.float32))


@pytest.mark.parametrize("radius", [0, 1, 3])
def test_masks_and_extents_match_oracle(radius, rng):
    imgs = G["pose_img_a"][::4]
    vs = IP.ViewStack(imgs)
    lv = np.array([0.05, 0.6, 1.8, 3.0, 0.9, 2.2])[:vs.n]
    m = vs.masks(lv, radius).cpu().numpy().astype(bool)
    for v in range(vs.n):
        want = O.dilate(O.threshold(imgs[v].astype(np.float64), lv[v]), radius)
        assert np.array_equal(m[v], want)
    nuis = vs.masks(np.full(vs.n, 2.5), 2)
    rects = ((180, 256, 0, 64), (0, 5, 0, 128), (-40, -20, 100, 200))
    left, right = vs.extents(mask=vs.masks(lv, radius), remove=nuis, exclude_rects=rects)
    nm = nuis.cpu().numpy().astype(bool)
    for v in range(vs.n):
        want = m[v] & ~nm[v]
        for r0, r1, c0, c1 in rects:
            want[r0:r1, c0:c1] = False
        wl, wr = extents(want)
        assert np.array_equal(left[0, v], wl) and np.array_equal(right[0, v], wr)


def test_fused_ladder_extents_equal_mask_extents():
    imgs = G["pose_img_a"]
    vs = IP.ViewStack(imgs)
    ladder = np.stack([1.8 + np.linspace(-1.0, 1.0, 18)] * vs.n)       # > 16 -> two passes
    ladder[5] += 0.01
    left, right = vs.extents(levels=ladder, exclude_rects=((100, 120, 0, 70),))
    for k in (0, 7, 16, 17):
        lm, rm = vs.extents(mask=vs.masks(ladder[:, k], 0), exclude_rects=((100, 120, 0, 70),))
        assert np.array_equal(left[k], lm[0]) and np.array_equal(right[k], rm[0])


def test_axis_endpoint_kernel_equals_full_mask_rule(rng):
    """ct_axis_endpoints on row extents == the reference's np.nonzero band rule
    (oracle) on random blobs of every band width, incl. the degenerate masks."""
    masks, bands = [], []
    for _ in range(300):
        m = np.zeros((32, 24), dtype=bool)
        h, w = rng.integers(1, 32), rng.integers(1, 24)
        m[:h, :w] = rng.random((h, w)) > rng.uniform(0.3, 0.995)
        masks.append(m)
        bands.append(int(rng.integers(0, 5)))
    vs = IP.ViewStack(np.stack(masks).astype(np.float32))
    left, right = vs._extents_dev(mask=vs.images.to(__import__("torch").uint8))
    for band in range(5):
        tu, tv, bu, bv, st = vs.axis_table(left, right, band)
        for i, m in enumerate(masks):
            if bands[i] != band:
                continue
            try:
                want = O.axis_endpoints(m, band)
            except O.OracleError:
                assert st[0, i] != IP.OK
                continue
            assert st[0, i] == IP.OK
            assert (tu[0, i], tv[0, i], bu[0, i], bv[0, i]) == want


@pytest.mark.parametrize("case", ["core", "auto", "nuis", "dil"])
def test_fit_pose_matches_reference(case):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", NoConvergenceWarning)
        res = P.fit_pose(ps_a(), P.PoseFitParams(**CASES[case]))
    ax = np.array([[a.top.u, a.top.v, a.bottom.u, a.bottom.v] for a in res.axes])
    assert np.array_equal(ax, G[f"pose_{case}_axes"])          # bit-exact observations
    ref = G[f"pose_{case}_pose"]
    assert abs(res.pose.alpha - ref[0]) < 1e-8 and abs(res.pose.beta - ref[1]) < 1e-8
    assert np.abs(res.pose.t - ref[3:]).max() < 1e-8
    assert [res.top.residual_rms, res.bottom.residual_rms] == pytest.approx(
        list(G[f"pose_{case}_rms"][:2]), rel=1e-9)
    doc = res.to_dict()
    for key in ("alpha_rad", "beta_deg", "t_mm", "residual_rms_px", "converged"):
        assert key in doc


def test_fit_pose_recovers_tilt():
    true_beta = math.radians(5.0)
    res = P.fit_pose(ps_a(), P.PoseFitParams(**CASES["core"]))
    assert math.degrees(abs(res.pose.beta - true_beta)) < 0.1
    assert res.top.converged and res.bottom.converged


def test_gamma_from_strip_signal_matches_reference():
    ps = P.ProjectionSet(pose_geometry(), G["pose_img_b"])
    kw = dict(CASES["core"], estimate_gamma=True, strip_offset=10.0, strip_width=8.0)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", NoConvergenceWarning)
        res = P.fit_pose(ps, P.PoseFitParams(**kw))
    sig = IP.ViewStack(G["pose_img_b"]).strip_profiles(res.axes, 10.0, 8.0)
    assert np.abs(sig - G["pose_gamma_signal"]).max() <= 1e-12 * np.abs(sig).max()
    assert res.gamma == pytest.approx(G["pose_gamma_pose"][2], abs=1e-9)
    assert res.to_dict()["gamma_estimated"]
    if G["pose_gamma_flat14"][0]:
        with pytest.raises(FlatSignal):
            P.fit_pose(ps, P.PoseFitParams(**dict(kw, strip_offset=14.0)))


def test_strip_profiles_match_reference_and_oracle():
    b = G["pose_img_b"]
    ax = IP.AxisObservation(P.DetectorPoint(60.25, 70.5), P.DetectorPoint(66.0, 190.0))
    k = 0
    for off, wd in ((-6.0, 1.0), (0.0, 3.0), (14.0, 8.0), (-40.5, 2.4), (70.0, 1.0)):
        for i in (0, 5, 13):
            want = G["pose_strips"][k]
            k += 1
            if math.isnan(want):
                with pytest.raises(OutOfFrame):
                    P.strip_profile(b[i], ax, off, wd)
                continue
            got = P.strip_profile(b[i], ax, off, wd)
            assert got == pytest.approx(want, rel=1e-12, abs=1e-300)


def test_per_image_api_and_errors(rng):
    img = np.zeros((10, 10), dtype=np.float32)
    img[3:7, 3:7] = 10.0
    assert np.array_equal(P.threshold(img, "auto"), img == 10.0)
    assert not P.threshold(np.full((8, 8), 3.0, np.float32), 5.0).any()
    with pytest.raises(ValueError):
        P.threshold(img, "median")
    m = rng.random((20, 20)) > 0.8
    assert np.array_equal(P.dilate(m, 2), O.dilate(m, 2))
    one = np.zeros((7, 7), dtype=bool)
    one[3, 3] = True
    assert P.dilate(one, 1).sum() == 9
    with pytest.raises(ValueError):
        P.dilate(m, -1)
    with pytest.raises(EmptyResult):
        P.remove_features(m, [np.ones((20, 20), dtype=bool)])
    for seed in range(12):
        mm = np.random.default_rng(seed).random((40, 30)) > 0.7
        mm[:seed % 4] = False
        ob = P.axis_endpoints(mm, band=1 + seed % 3)
        assert [ob.top.u, ob.top.v, ob.bottom.u, ob.bottom.v] == list(G["pose_ends"][seed])
    with pytest.raises(DegenerateMask):
        P.axis_endpoints(np.zeros((5, 5), dtype=bool))
    axis = IP.AxisObservation(P.DetectorPoint(10.0, 2.0), P.DetectorPoint(10.0, 17.0))
    assert P.strip_profile(np.full((20, 20), 4.2, np.float32), axis, -3.0) == pytest.approx(
        float(np.float32(4.2)))
    with pytest.raises(OutOfFrame):
        P.strip_profile(np.zeros((20, 20), np.float32), axis, 100.0)


def test_segmentation_errors_follow_view_order():
    imgs = G["pose_img_a"].copy()
    imgs[2] = 0.0                                    # view 2: constant image
    ps = P.ProjectionSet(pose_geometry(), imgs)
    with pytest.raises(DegenerateHistogram):
        P.fit_pose(ps, P.PoseFitParams())            # "auto" on a constant view
    with pytest.raises(DegenerateMask):
        P.fit_pose(ps, P.PoseFitParams(threshold_level=0.5))
    with pytest.raises(EmptyResult):
        P.fit_pose(ps, P.PoseFitParams(threshold_level=0.5, exclude_rects=((0, 256, 0, 128),)))


def test_table1_size_extents_property():
    """At the BASELINE Table-1 detector size (1944 x 1536, 21 views) the fused
    ladder pass equals torch-computed extents of the thresholded images."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(5)
    imgs = torch.rand((21, 1536, 1944), device="cuda", generator=g) * 0.5
    imgs[:, 300:1200, 800:1100] += 2.0
    vs = IP.ViewStack(imgs)
    lv = np.tile(np.array([1.0, 2.2, 2.45]), (21, 1))
    left, right = vs.extents(levels=lv)
    cols = torch.arange(1944, device="cuda")
    for k in range(3):
        m = imgs.double() > lv[0, k]
        has = m.any(dim=2)
        lo = torch.where(m, cols, 1 << 30).amin(dim=2)
        hi = torch.where(m, cols, -1).amax(dim=2)
        assert np.array_equal(left[k], torch.where(has, lo, -1).cpu().numpy())
        assert np.array_equal(right[k], hi.cpu().numpy())
