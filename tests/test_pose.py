"""Pose step, host side: the oracle pinned to the
reference's outputs (tests/golden/golden_pose.npz, written by the unmodified
reference), and the host logic of paper_2005_11976_b200.imgproc / posefit
(Otsu from counts, LM triangulation, axis_to_pose, phase fit) against both;
the kernels are in tests/test_gpu_pose.py.  Behavioural cases follow the reference's
tests/test_posefit.py and tests/test_imgproc.py."""

import math
import sys
import warnings
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))

import pose_oracle as O  # noqa: E402
from paper_2005_11976_b200 import (DetectorPoint, LmConfig, Pose, PoseFitParams,  # noqa: E402
                                   ScanGeometry, axis_to_pose, euler_to_matrix,
                                   make_circular_trajectory, project_point, track_point)
from paper_2005_11976_b200.errors import (DegenerateAxis, FlatSignal,  # noqa: E402
                                          IllPosed, NoConvergenceWarning)
from paper_2005_11976_b200.geometry import (detector_point_world, project_point_jacobian,  # noqa: E402
                                            view_basis, wrap_angle)
from paper_2005_11976_b200.imgproc import AxisObservation, otsu_from_histogram  # noqa: E402
from paper_2005_11976_b200.posefit import (_midpoint_init, _residuals_jacobian,  # noqa: E402
                                           phase_from_signal)

G = np.load(ROOT / "tests" / "golden" / "golden_pose.npz")

CASES = {   # the reference PoseFitParams of each golden case (make_golden.pose_cases)
    "core": dict(threshold_level=1.8, threshold_levels=9, threshold_span=1.0, band=1),
    "auto": dict(threshold_level="auto", dilation_radius=1, band=2),
    "nuis": dict(threshold_level=0.3, threshold_levels=3, threshold_span=0.1,
                 nuisance_level=2.5, nuisance_dilation=2,
                 exclude_rects=((180, 256, 0, 64), (0, 5, 0, 128))),
    "dil": dict(threshold_level=1.0, threshold_levels=4, threshold_span=0.5,
                dilation_radius=2, band=3),
}


def pose_geometry():
    return ScanGeometry(791.0, 679.0, 128, 256, 0.52, (63.5, 127.5),
                        make_circular_trajectory(21, math.radians(200.0)))


@pytest.fixture
def desk():
    return ScanGeometry(791.0, 679.0, 256, 128, 0.748, (127.5, 63.5),
                        make_circular_trajectory(21, math.radians(200.0)))


def oracle_kwargs(kw):
    p = PoseFitParams(**kw)
    return dict(levels=p.levels(), dilation_radius=p.dilation_radius, band=p.band,
                nuisance_level=p.nuisance_level, nuisance_dilation=p.nuisance_dilation,
                exclude_rects=p.exclude_rects)


def extents(mask):
    m = np.asarray(mask, dtype=bool)
    has = m.any(axis=1)
    left = np.where(has, m.argmax(axis=1), -1)
    right = np.where(has, m.shape[1] - 1 - m[:, ::-1].argmax(axis=1), -1)
    return left, right


# ---- the oracle, pinned to the reference ------------------------------------
@pytest.mark.parametrize("case", ["core", "auto", "nuis", "dil"])
def test_oracle_axes_match_reference(case):
    ax = O.fit_axes(G["pose_img_a"].astype(np.float64), **oracle_kwargs(CASES[case]))
    assert np.array_equal(ax, G[f"pose_{case}_axes"])


def test_oracle_image_functions_match_reference():
    imgs = np.concatenate([G["pose_img_a"], G["pose_img_b"]]).astype(np.float64)
    assert np.array_equal([O.otsu_level(x) for x in imgs], G["pose_otsu"])
    sig = [O.strip_profile(G["pose_img_b"][i].astype(np.float64), G["pose_gamma_axes"][i],
                           10.0, 8.0) for i in range(21)]
    assert np.array_equal(sig, G["pose_gamma_signal"])
    for seed in range(12):
        m = np.random.default_rng(seed).random((40, 30)) > 0.7
        m[:seed % 4] = False
        assert np.array_equal(O.axis_endpoints(m, 1 + seed % 3), G["pose_ends"][seed])


# ---- host logic of the product ----------------------------------------------
def test_otsu_from_counts_matches_reference():
    imgs = np.concatenate([G["pose_img_a"], G["pose_img_b"]]).astype(np.float64)
    got = []
    for x in imgs:
        lo, hi = float(x.min()), float(x.max())
        counts, _ = np.histogram(x, bins=256, range=(lo, hi))
        got.append(otsu_from_histogram(counts, lo, hi))
    assert np.array_equal(got, G["pose_otsu"])


def test_axis_observation_swap():
    ob = AxisObservation(top=DetectorPoint(1.0, 9.0), bottom=DetectorPoint(2.0, 3.0))
    assert ob.top.v < ob.bottom.v


def test_levels_ladder():
    assert PoseFitParams().levels() == ["auto"]
    lv = PoseFitParams(threshold_level=1.8, threshold_levels=9, threshold_span=1.0).levels()
    assert np.array_equal(lv, 1.8 + np.linspace(-1.0, 1.0, 9))
    with pytest.raises(ValueError):
        PoseFitParams(threshold_levels=3, threshold_span=0.5).levels()   # "auto" + ladder


# ---- geometry helpers --------------------------------------------------------
def test_projection_jacobian_matches_finite_differences(desk, rng):
    for _ in range(10):
        x = rng.uniform(-20, 20, 3)
        i = int(rng.integers(0, 21))
        jac = project_point_jacobian(desk, i, x)
        num = np.zeros((2, 3))
        for k in range(3):
            e = np.zeros(3)
            e[k] = 1e-5
            a, b = project_point(desk, i, x + e), project_point(desk, i, x - e)
            num[:, k] = [(a.u - b.u) / 2e-5, (a.v - b.v) / 2e-5]
        assert np.abs(jac - num).max() < 1e-5 * max(1.0, np.abs(jac).max())
        pt = project_point(desk, i, x)
        w = detector_point_world(desk, i, pt)
        src = view_basis(desk, i)[0]
        # the world detector point lies on the ray through x
        d1, d2 = w - src, x - src
        assert np.linalg.norm(np.cross(d1, d2)) / (np.linalg.norm(d1) * np.linalg.norm(d2)) < 1e-12


# ---- triangulation (cyltomo tests/test_posefit.py:29-91 behaviours) ----------
def observe(geom, x, views):
    return [(i, project_point(geom, i, x)) for i in views]


def test_track_point_noiseless_round_trip(desk, rng):
    for _ in range(20):
        x = rng.uniform(-20, 20, size=3)
        tp = track_point(observe(desk, x, range(0, 21, 4)), desk)
        assert np.abs(tp.solution - x).max() < 1e-6
        assert tp.residual_rms < 1e-9 and tp.converged


def test_track_point_principal_point_gives_origin(desk):
    u0, v0 = desk.principal_point
    tp = track_point([(i, DetectorPoint(u0, v0)) for i in range(21)], desk)
    assert np.abs(tp.solution).max() < 1e-9


def test_track_point_not_worse_than_init(desk, rng):
    x = rng.uniform(-15, 15, size=3)
    noisy = [(i, DetectorPoint(p.u + rng.normal(0, 0.3), p.v + rng.normal(0, 0.3)))
             for i, p in observe(desk, x, range(0, 21, 2))]
    res0, _ = _residuals_jacobian(_midpoint_init(noisy, desk), noisy, desk)
    tp = track_point(noisy, desk)
    assert tp.residual_rms <= math.sqrt(res0 @ res0 / len(noisy)) + 1e-12


def test_track_point_ill_posed(desk):
    pt = DetectorPoint(100.0, 60.0)
    with pytest.raises(IllPosed):
        track_point([(0, pt)], desk)
    same = ScanGeometry(791.0, 679.0, 256, 128, 0.748, (127.5, 63.5), np.zeros(4))
    with pytest.raises(IllPosed):
        track_point([(i, pt) for i in range(4)], same)


def test_track_point_iteration_cap(desk, rng):
    x = rng.uniform(-15, 15, size=3)
    noisy = [(i, DetectorPoint(p.u + rng.normal(0, 1.0), p.v + rng.normal(0, 1.0)))
             for i, p in observe(desk, x, range(0, 21, 3))]
    cfg = LmConfig(max_iterations=1, step_tolerance=1e-15, residual_tolerance=1e-30)
    with pytest.warns(NoConvergenceWarning):
        tp = track_point(noisy, desk, cfg)
    assert not tp.converged and np.isfinite(tp.solution).all()


def test_lm_config_validation():
    with pytest.raises(ValueError):
        LmConfig(damping_init=0.0)
    with pytest.raises(ValueError):
        LmConfig(damping_up=0.5)


def test_track_point_matches_reference_solutions(desk):
    """Noisy triangulations solved by the reference (vectorised residuals here;
    same minimiser to 1e-8 mm)."""
    for obs, sol in zip(G["pose_lm_obs"], G["pose_lm_sol"]):
        pts = [(int(i), DetectorPoint(u, v)) for i, u, v in obs]
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", NoConvergenceWarning)
            tp = track_point(pts, desk)
        assert np.abs(tp.solution - sol[:3]).max() < 1e-8
        assert tp.residual_rms == pytest.approx(sol[3], rel=1e-9)


# ---- axis -> pose (tests/test_posefit.py:94-127) -----------------------------
def test_axis_to_pose_up_down_and_degenerate():
    p = axis_to_pose([0.0, 0.0, 1.0], [0.0, 0.0, -1.0])
    assert (p.alpha, p.beta, p.gamma) == (0.0, 0.0, 0.0) and np.allclose(p.t, 0.0)
    assert axis_to_pose([0.0, 0.0, -1.0], [0.0, 0.0, 1.0]).beta == pytest.approx(math.pi)
    with pytest.raises(DegenerateAxis):
        axis_to_pose([1.0, 2.0, 3.0], [1.0, 2.0, 3.0])


def test_axis_to_pose_round_trip(rng):
    for _ in range(200):
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        pose = axis_to_pose(5.0 * d, -5.0 * d)
        assert np.abs(euler_to_matrix(pose) @ [0, 0, 1] - d).max() < 1e-12
    for _ in range(100):
        alpha, beta = rng.uniform(-math.pi, math.pi), rng.uniform(0.05, math.pi - 0.05)
        t = rng.uniform(-10, 10, size=3)
        r = euler_to_matrix(Pose(alpha, beta, rng.uniform(-3, 3), t=t))
        back = axis_to_pose(r @ [0, 0, 7.0] + t, r @ [0, 0, -7.0] + t)
        assert back.alpha == pytest.approx(alpha, abs=1e-9)
        assert back.beta == pytest.approx(beta, abs=1e-9)
        assert np.abs(back.t - t).max() < 1e-9


@pytest.mark.parametrize("case", ["core", "auto", "nuis", "dil"])
def test_pose_from_reference_axes(case):
    """Host half of fit_pose on the reference's own axis observations."""
    geom = pose_geometry()
    ax = G[f"pose_{case}_axes"]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", NoConvergenceWarning)
        top = track_point([(i, DetectorPoint(a[0], a[1])) for i, a in enumerate(ax)], geom)
        bot = track_point([(i, DetectorPoint(a[2], a[3])) for i, a in enumerate(ax)], geom)
    pa, pb = top.solution, bot.solution
    if pa[2] < pb[2]:
        pa, pb = pb, pa
    pose = axis_to_pose(pa, pb)
    ref = G[f"pose_{case}_pose"]
    assert np.abs(np.array([pose.alpha, pose.beta]) - ref[:2]).max() < 1e-8
    assert np.abs(pose.t - ref[3:]).max() < 1e-8
    assert np.abs(np.concatenate([top.solution, bot.solution]) - G[f"pose_{case}_pts"]).max() < 1e-8


# ---- phase (tests/test_posefit.py:130-173) -----------------------------------
def synthetic_signal(phi_p, n=24, mean=5.0, amp=1.0):
    phis = make_circular_trajectory(n, 2 * math.pi * (n - 1) / n)
    zeta = phis[0] - phis
    return phis, mean + amp * np.cos(zeta - phi_p)


def test_phase_from_signal():
    for phi_p in (0.3, -2.0, 3.0):
        phis, s = synthetic_signal(phi_p)
        assert phase_from_signal(phis, s, Pose()) == pytest.approx(
            wrap_angle(phi_p - phis[0]), abs=1e-9)
    phis, s = synthetic_signal(0.8)
    want = wrap_angle(0.8 - math.atan(math.tan(0.3) / math.cos(0.4)))
    assert phase_from_signal(phis, s, Pose(alpha=0.3, beta=0.4)) == pytest.approx(want, abs=1e-9)
    with pytest.raises(FlatSignal):
        phase_from_signal(*synthetic_signal(0.0, amp=0.0), Pose())


def test_phase_from_reference_signal():
    ref = G["pose_gamma_pose"]
    pose = Pose(ref[0], ref[1], 0.0, t=ref[3:])
    gamma = phase_from_signal(pose_geometry().stage_angles, G["pose_gamma_signal"], pose)
    assert gamma == pytest.approx(ref[2], abs=1e-12)
