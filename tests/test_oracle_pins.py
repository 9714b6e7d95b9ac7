"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Nothing here compares the oracle with itself: every expectation is a value
printed in PAPER.md / SPEC.md (tests/golden/, each cited), a closed form, an
invariant, an independent library routine (scipy Rotation, numpy eigvalsh,
math.exp), a finite-difference derivative, or brute force on tiny inputs.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle
from helpers import make_scene, make_view, quat_mul
from paper_2503_08217_b200 import scenegen as sg

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_examples.json")))
WORK = json.load(open(os.path.join(GOLD, "worked_examples.json")))


# --------------------------------------------------------------------------
# time, filter, life, commit, reset  (Eq.5, Eq.6)
# --------------------------------------------------------------------------

def test_normalize_time_golden():
    for i, n, t in SPEC["normalize_time"]["cases"]:
        assert oracle.normalize_time(i, n) == t
    ts = [oracle.normalize_time(i, 37) for i in range(37)]
    assert all(a < b for a, b in zip(ts, ts[1:]))          # strictly monotone


def test_temporal_filter_golden():
    for (vs, ve), t, inc in SPEC["temporal_filter"]["cases"]:
        s = make_scene([[0, 0, 5]], 0.1, vis=[[vs, ve]])
        assert (len(oracle.temporal_filter(s, t)) == 1) == inc, (vs, ve, t)


def test_temporal_filter_random_1e5():
    rng = np.random.default_rng(0)
    n = 100_000
    a = rng.uniform(-1.2, 1.2, n)
    b = a + rng.uniform(-0.3, 1.0, n)
    vis = np.stack([a, b], 1).astype(np.float32)
    vis[::997, 0] = np.nan                                  # NaN bound -> excluded
    s = make_scene(np.zeros((n, 3)), 0.1, vis=vis)
    for t in (-1.0, -0.37, 0.0, 0.5, 1.0):
        idx = oracle.temporal_filter(s, t)
        t32 = np.float32(t)
        want = np.nonzero((vis[:, 0] <= t32) & (t32 <= vis[:, 1]))[0]
        assert np.array_equal(idx, want)
        assert np.all(np.diff(idx) > 0)                     # ascending list


def test_update_life_golden():
    for life, m, t, want in SPEC["update_life"]["cases"]:
        s = make_scene([[0, 0, 5]], 0.1)
        s.life[:] = life
        oracle.update_life(s, np.array([m], np.uint8), t)
        assert np.array_equal(s.life[0], np.float32(want))


def test_commit_and_reset_golden():
    for life, want in SPEC["commit"]["cases"]:
        s = make_scene([[0, 0, 5]], 0.1)
        s.life[:] = life
        oracle.commit_visibility(s, 0.1)
        assert np.array_equal(s.visibility[0], np.float32(want)), (life, s.visibility[0])
        assert np.array_equal(s.life[0], np.float32([1, -1]))    # life reset (R18)
    s = make_scene(np.zeros((5, 3)), 0.1, vis=np.random.default_rng(1).uniform(-1, 1, (5, 2)))
    oracle.reset_visibility(s)
    v1 = s.visibility.copy()
    oracle.reset_visibility(s)
    assert np.array_equal(v1, s.visibility)
    assert np.all(v1 == np.float32([-1, 1]))
    for t in (-1.0, 0.0, 1.0):
        assert len(oracle.temporal_filter(s, t)) == 5


def test_life_monotone_and_margin():
    """l_s never increases / l_e never decreases; commit keeps every observation
    time inside the interval with margin >= 0.1 up to clamping."""
    rng = np.random.default_rng(5)
    s = make_scene(np.zeros((200, 3)), 0.1)
    seen = [[] for _ in range(200)]
    prev = s.life.copy()
    for _ in range(30):
        t = float(np.float32(rng.uniform(-1, 1)))
        m = (rng.random(200) < 0.3).astype(np.uint8)
        oracle.update_life(s, m, t)
        assert np.all(s.life[:, 0] <= prev[:, 0]) and np.all(s.life[:, 1] >= prev[:, 1])
        prev = s.life.copy()
        for g in np.nonzero(m)[0]:
            seen[g].append(np.float32(t))
    oracle.commit_visibility(s, 0.1)
    for g in range(200):
        if seen[g]:
            lo, hi = min(seen[g]), max(seen[g])
            assert s.visibility[g, 0] <= max(np.float32(-1), lo - np.float32(0.1)) + 1e-7
            assert s.visibility[g, 1] >= min(np.float32(1), hi + np.float32(0.1)) - 1e-7
        else:
            assert np.array_equal(s.visibility[g], np.float32([-1, 1]))


# --------------------------------------------------------------------------
# LOD (Eq.7 rows 1-3)
# --------------------------------------------------------------------------

def test_drop_probability_golden():
    g = SPEC["drop_probability"]
    for d, p in g["cases"]:
        p64 = oracle.drop_probability(d, g["pmax"], g["D"], "f64")
        p32 = oracle.drop_probability(d, g["pmax"], g["D"], "f32")
        assert abs(p64 - p) < 1e-12
        assert abs(p32 - p) < 2e-7
    # exact at d = D and d >= D (S:683 acceptance 5)
    assert oracle.drop_probability(50.0, 0.5, 50.0) == 0.5
    assert oracle.drop_probability(500.0, 0.5, 50.0) == 0.5
    # monotone non-decreasing in d, clamped to [0,1]
    ds = np.linspace(0, 200, 401)
    ps = [oracle.drop_probability(float(d), 0.7, 60.0, "f64") for d in ds]
    assert all(a <= b + 1e-15 for a, b in zip(ps, ps[1:]))
    # p runs from 0.01 at d = 0 to p_max at d >= D, whatever p_max in [0,1] is
    for pmax in (0.0, 0.005, 0.3, 1.0):
        assert abs(oracle.drop_probability(0.0, pmax, 50.0, "f64") - 0.01) < 1e-15
        assert oracle.drop_probability(80.0, pmax, 50.0, "f64") == pmax


def _lod_scene(n, depth, sigma=0.001, seed=0):
    rng = np.random.default_rng(seed)
    pts = np.stack([rng.uniform(-0.3, 0.3, n) * depth, rng.uniform(-0.3, 0.3, n) * depth,
                    np.full(n, depth)], 1)
    return make_scene(pts, sigma, opacity=0.5)


@pytest.mark.parametrize("depth", [10.0, 30.0, 60.0])
def test_lod_keep_rate_binomial(depth):
    """Empirical drop rate within 3 binomial sigma of p(d) for N = 1e4."""
    n = 10_000
    s = _lod_scene(n, depth)
    v = make_view(100.0, 64.0, 128, 128, lod=(4.0, 0.5, 50.0), seed=987654321)
    o = oracle.render_view(s, v, pairs=False, image=False)
    small = (o["flags"] & oracle.F_SMALL) != 0
    assert small.sum() == n
    dropped = ((o["flags"] & oracle.F_DROPPED) != 0).sum()
    p = 0.5 + 0.49 * min(0.0, (depth - 50.0) / 50.0)
    sd = math.sqrt(n * p * (1 - p))
    assert abs(dropped - n * p) <= 3 * sd, (dropped, n * p, sd)
    assert o["stats"]["n_lod_dropped"] == dropped
    assert o["stats"]["n_rendered"] == n - dropped


def test_lod_disabled_and_deterministic():
    s = _lod_scene(2000, 40.0)
    v0 = make_view(100.0, 64.0, 128, 128, lod=(0.0, 0.9, 50.0), seed=1)
    o = oracle.render_view(s, v0, pairs=False, image=False)
    assert o["stats"]["n_lod_small"] == 0 and o["stats"]["n_lod_dropped"] == 0   # r = 0 disables
    v1 = make_view(100.0, 64.0, 128, 128, lod=(4.0, 0.9, 50.0), seed=1)
    a = oracle.render_view(s, v1, pairs=False, image=False)["flags"]
    b = oracle.render_view(s, v1, pairs=False, image=False)["flags"]
    assert np.array_equal(a, b)
    v2 = make_view(100.0, 64.0, 128, 128, lod=(4.0, 0.9, 50.0), seed=2)
    c = oracle.render_view(s, v2, pairs=False, image=False)["flags"]
    assert not np.array_equal(a, c)


def test_lod_uniform_distribution():
    u = np.array([oracle.lod_uniform(77, g) for g in range(20000)])
    assert np.all((u >= 0) & (u < 1))
    assert np.all(u * 2**24 == np.round(u * 2**24))           # 24-bit grid
    hist = np.histogram(u, bins=10, range=(0, 1))[0]
    assert np.all(np.abs(hist - 2000) < 5 * math.sqrt(2000 * 0.9))


def test_splitmix64_reference_outputs():
    outs = [int(h, 16) for h in WORK["splitmix64"]["outputs_from_state0"]]
    state = 0
    for want in outs:
        assert oracle.splitmix64(state) == want
        state = (state + 0x9E3779B97F4A7C15) & ((1 << 64) - 1)


@pytest.mark.parametrize("sig,scale", [((1.0, 1.0, 1.0), 3.0), ((2.0, 1.0, 1.0), 6.0)])
def test_scale2d_golden(sig, scale):
    """scale2d(I) = 3, scale2d(diag(4,1)) = 6, realised with J = I:
    a Gaussian on the optical axis at z = f.  The small set is inclusive (<= r)."""
    s = make_scene([[0, 0, 100.0]], [sig], opacity=0.5)
    for r, small in ((scale, True), (scale * 1.001, True), (scale * 0.999, False)):
        v = make_view(100.0, 64.0, 128, 128, lod=(r, 1.0, 50.0))
        o = oracle.render_view(s, v, pairs=False, image=False)
        assert bool(o["flags"][0] & oracle.F_SMALL) == small, (r, o["keys"][0])
        # p_max = 1 at d >= D: every small Gaussian is dropped, large ones never
        assert bool(o["flags"][0] & oracle.F_DROPPED) == small
        assert bool(o["flags"][0] & oracle.F_RENDERED) == (not small)


# --------------------------------------------------------------------------
# projection (Eq.1) and instance-specific projection
# --------------------------------------------------------------------------

@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_projection_golden(prec):
    g = SPEC["projection"]
    cam = g["camera"]
    for p, (mx, my, z) in g["cases"]:
        s = make_scene([p], 0.01)
        v = make_view(cam["f"], cam["c"], cam["w"], cam["h"])
        st, k = oracle.project(s, v, 0, prec)
        assert st == 0
        tol = 1e-5 if prec == "f32" else 1e-6      # inputs are fp32 (0.1 is not exact)
        assert abs(k[0] - mx) < tol and abs(k[1] - my) < tol and abs(k[2] - z) < tol


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_closed_form_projection(prec):
    g = WORK["closed_form_projection"]
    s = make_scene([g["point"]], g["sigma"])
    v = make_view(g["f"], g["c"], g["w"], g["h"])
    st, k = oracle.project(s, v, 0, prec)
    tol = 2e-6 if prec == "f32" else 1e-9
    assert st == 0
    assert np.allclose(k[:2], g["mean"], atol=tol * 100) and abs(k[2] - g["depth"]) < tol
    assert np.allclose(k[3:], g["cov2d"], atol=tol * 10), k


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_tangent_clamp_far_off_screen(prec):
    """Reading R5 (3DGS practice): the Jacobian takes x/z and y/z clamped to the
    1.3x-extended image, u in [(-0.15 W - cx)/fx, (1.15 W - cx)/fx] (v alike),
    while the mean keeps the unclamped u.  An isotropic Gaussian (identity
    camera) far to the right and below the view then has, in closed form,
    Sigma' = s^2 J J^T = s^2 [[fx^2 (1 + uc^2), fx fy uc vc], [., fy^2 (1 + vc^2)]] / z^2
    with (uc, vc) the bounds; inside the bounds the same formula holds with (u, v)."""
    W, H, fx, fy, cx, cy = 160, 120, 100.0, 90.0, 80.0, 60.0
    sig, z = 0.2, 10.0
    v = make_view(fx, cx, W, H, fy=fy, cy=cy)
    hix = (1.15 * W - cx) / fx
    hiy = (1.15 * H - cy) / fy
    for (x, y) in [(3.0 * hix * z, 2.5 * hiy * z), (0.5 * hix * z, 0.4 * hiy * z)]:
        s = make_scene([[x, y, z]], sig)
        st, k = oracle.project(s, v, 0, prec)
        assert st == 0
        x, y = float(np.float32(x)), float(np.float32(y))      # the scene is fp32
        u, vv = x / z, y / z
        uc, vc = min(u, hix), min(vv, hiy)
        s2 = np.float64(np.float32(sig)) ** 2
        want = s2 / z ** 2 * np.array([fx * fx * (1 + uc * uc), fx * fy * uc * vc,
                                         fy * fy * (1 + vc * vc)])
        tol = 1e-5 if prec == "f32" else 1e-11
        assert np.allclose(k[3:], want, rtol=tol, atol=0), (k[3:], want)
        assert np.isclose(k[0], fx * u + cx, rtol=1e-6)        # the mean is not clamped


def test_commit_single_observation():
    """Eq.6 for a Gaussian observed at exactly one time t: l_s = l_e = t,
    so the committed interval is [t - 0.1, t + 0.1] — not the never-observed
    case (l_s > l_e, reading R18), which becomes visible at all times."""
    s = make_scene([[0, 0, 5], [0, 0, 6]], 0.1)
    t = float(np.float32(0.3))
    oracle.update_life(s, np.array([1, 0], np.uint8), t)
    assert s.life[0, 0] == s.life[0, 1] == np.float32(t)
    oracle.commit_visibility(s, 0.1)
    want = [np.float32(np.float32(t) - np.float32(0.1)), np.float32(np.float32(t) + np.float32(0.1))]
    assert np.array_equal(s.visibility[0], np.float32(want)), s.visibility[0]
    assert np.array_equal(s.visibility[1], np.float32([-1, 1]))     # never observed


def test_covariance_yaw_golden():
    g = SPEC["covariance_yaw"]
    s = make_scene([[0, 0, 100.0]], [g["sigma"]], quats=[g["quat"]])
    v = make_view(100.0, 64.0, 128, 128)
    st, k = oracle.project(s, v, 0, "f64")
    e = g["expect_2x2"]
    assert np.allclose([k[3], k[4], k[5]], [e[0][0], e[0][1], e[1][1]], atol=1e-12)


def _pinhole(p, fx, fy, cx, cy):
    return np.array([fx * p[0] / p[2] + cx, fy * p[1] / p[2] + cy])


def test_cov2d_matches_finite_difference_jacobian():
    """Sigma' = J W Sigma W^T J^T with J from central differences of the pinhole map
    and R(q) from scipy (independent quaternion convention) — S:113."""
    rng = np.random.default_rng(3)
    n = 300
    pts = np.stack([rng.uniform(-2, 2, n), rng.uniform(-1.5, 1.5, n), rng.uniform(4, 12, n)], 1)
    sig = np.exp(rng.uniform(-3, 0, (n, 3)))
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    s = make_scene(pts, sig, quats=q)
    Rw = Rotation.from_euler("xyz", [0.05, -0.08, 0.1]).as_matrix()
    tw = np.array([0.2, -0.1, 0.3])
    w2c = np.concatenate([Rw, tw[:, None]], 1)
    fx, fy, cx, cy = 500.0, 520.0, 320.5, 240.25
    v = make_view(fx, cx, 640, 480, w2c=w2c, fy=fy, cy=cy)
    Rw32 = np.asarray(v.w2c[:, :3], np.float64)
    tw32 = np.asarray(v.w2c[:, 3], np.float64)
    checked = 0
    for g in range(n):
        st, k = oracle.project(s, v, g, "f64")
        assert st == 0
        mu = s.means_opacity[g, :3].astype(np.float64)
        pc = Rw32 @ mu + tw32
        u, vv = pc[0] / pc[2], pc[1] / pc[2]
        if not (-0.15 * 640 - cx) / fx < u < (1.15 * 640 - cx) / fx or \
           not (-0.15 * 480 - cy) / fy < vv < (1.15 * 480 - cy) / fy:
            continue                                      # tangent clamp active
        h = 1e-6 * np.linalg.norm(pc)
        J = np.zeros((2, 3))
        for a in range(3):
            e = np.zeros(3)
            e[a] = h
            J[:, a] = (_pinhole(pc + e, fx, fy, cx, cy) - _pinhole(pc - e, fx, fy, cx, cy)) / (2 * h)
        qq = s.rotations[g].astype(np.float64)
        Rq = Rotation.from_quat([qq[1], qq[2], qq[3], qq[0]]).as_matrix()
        S = np.diag(s.scales[g, :3].astype(np.float64) ** 2)
        Sig = Rw32 @ Rq @ S @ Rq.T @ Rw32.T
        C2 = J @ Sig @ J.T
        got = np.array([[k[3], k[4]], [k[4], k[5]]])
        assert np.allclose(got, C2, rtol=1e-5, atol=1e-7 * np.abs(C2).max()), (g, got, C2)
        assert np.allclose(k[:2], _pinhole(pc, fx, fy, cx, cy), atol=1e-9)
        checked += 1
    assert checked > 200


def _dyadic_pose(rng):
    """A rotation by a multiple of 90 deg about a random axis and a dyadic
    translation: representable exactly, so fp64 products are exact."""
    axis = rng.integers(0, 3)
    k = rng.integers(1, 4)
    R = np.round(Rotation.from_rotvec(np.eye(3)[axis] * k * np.pi / 2).as_matrix())
    t = rng.integers(-64, 64, 3) / 8.0
    return R, t


def test_compose_instance_cameras():
    """W_{t,i} = W_t W_{t,i2g} vs a 4x4 homogeneous product."""
    rng = np.random.default_rng(11)
    w2c = np.concatenate([Rotation.random(random_state=1).as_matrix(), rng.normal(size=(3, 1))], 1)
    i2g = np.stack([np.concatenate([Rotation.random(random_state=i + 2).as_matrix(),
                                    rng.normal(size=(3, 1)) * 10], 1) for i in range(5)])
    v = make_view(100, 50, 100, 100, w2c=w2c, i2g=i2g)
    tab = oracle.compose(v)
    assert np.array_equal(tab[0], v.w2c.reshape(12))                  # slot 0 = W_t
    h = lambda m: np.concatenate([np.asarray(m, np.float64), [[0, 0, 0, 1]]], 0)
    for i in range(5):
        want = (h(v.w2c) @ h(v.i2g[i]))[:3].reshape(12)
        assert np.allclose(tab[i + 1], want, rtol=0, atol=2e-6 * (1 + np.abs(want)))
    # identity and commuting translations are exact
    I = np.concatenate([np.eye(3), [[1.0], [0.0], [0.0]]], 1)
    J = np.concatenate([np.eye(3), [[0.0], [2.0], [0.0]]], 1)
    tab = oracle.compose(make_view(100, 50, 100, 100, w2c=I, i2g=J[None]))
    assert np.array_equal(tab[1].reshape(3, 4)[:, 3], np.float32([1, 2, 0]))


def test_instance_projection_equivalence_exact():
    """Local Gaussians through W_t W_{t,i2g} == world Gaussians through W_t,
    component-wise within 1e-9 in fp64 over 1e4 (Gaussian, pose, camera)
    triples (S:121, S:680 acceptance 2; the theorem of).  Poses are
    exactly representable so the only difference is the order of operations."""
    rng = np.random.default_rng(12)
    n_per, K = 1000, 10
    Rw, tw = _dyadic_pose(rng)
    w2c = np.concatenate([Rw, tw[:, None]], 1)
    poses = [_dyadic_pose(rng) for _ in range(K)]
    pts_local = rng.integers(-256, 256, (n_per * K, 3)) / 64.0
    ids = np.repeat(np.arange(1, K + 1), n_per).astype(np.int32)
    q = rng.standard_normal((n_per * K, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q = q.astype(np.float32).astype(np.float64)
    sig = np.exp(rng.uniform(-3, -1, (n_per * K, 3)))
    i2g = np.stack([np.concatenate([R, t[:, None]], 1) for R, t in poses])
    # place the camera so that the objects are in front of it
    w2c[:, 3] += np.array([0.0, 0.0, 40.0]) - 0.0
    loc = make_scene(pts_local, sig, quats=q, ids=ids, num_instances=K + 1)
    view_loc = make_view(300.0, 160.0, 320, 320, w2c=w2c, i2g=i2g)
    # conventional: transform to world, all ids 0, table = [W_t]
    pw = np.zeros_like(pts_local)
    qw = np.zeros_like(q)
    for k, (R, t) in enumerate(poses):
        sl = ids == k + 1
        pw[sl] = pts_local[sl] @ R.T + t
        qk = Rotation.from_matrix(R).as_quat()          # (x,y,z,w)
        qk = np.array([qk[3], qk[0], qk[1], qk[2]])
        qw[sl] = [quat_mul(qk, qq) for qq in q[sl]]
    wor = make_scene(pw, sig, quats=qw, ids=np.zeros(n_per * K, np.int32), num_instances=1)
    view_w = make_view(300.0, 160.0, 320, 320, w2c=w2c)
    n_ok = 0
    for g in range(0, n_per * K):
        a_st, a = oracle.project(loc, view_loc, g, "f64")
        b_st, b = oracle.project(wor, view_w, g, "f64")
        assert a_st == b_st
        if a_st:
            continue
        scale = np.maximum(1.0, np.abs(b))
        # mean and depth: exact inputs, so agreement to fp64 rounding
        assert np.all(np.abs(a[:3] - b[:3]) <= 1e-9 * scale[:3]), (g, a, b)
        # covariance: the world quaternion q_i2g * q is stored in fp32 (the scene
        # format), which perturbs it by ~6e-8 relative before projection
        cs = abs(b[3]) + abs(b[5])
        assert np.all(np.abs(a[3:] - b[3:]) <= 5e-7 * cs), (g, a, b)
        n_ok += 1
    assert n_ok > 5000


# --------------------------------------------------------------------------
# blending (Eq.2)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_W1_worked_example(prec):
    g = WORK["W1"]
    s = make_scene([g["point"]], g["sigma"], opacity=g["opacity"], rgb=[g["rgb"]])
    v = make_view(g["f"], g["c"], g["w"], g["h"])
    o = oracle.render_view(s, v, prec)
    # f64: sigma = 0.05 is stored in fp32 (relative error 1.5e-8), hence 1e-7
    tol = 3e-6 if prec == "f32" else 1e-7
    assert np.allclose(o["keys"][0, 3:], g["cov2d"], atol=tol)
    assert list(o["rect"][0]) == g["tiles"]
    assert o["stats"]["n_pairs"] == g["n_pairs"]
    assert sorted(o["pair_tile"].tolist()) == [1 * 4 + 1, 1 * 4 + 2, 2 * 4 + 1, 2 * 4 + 2]
    # the whole image in closed form
    ys, xs = np.mgrid[0:64, 0:64]
    in_rect = (xs // 16 >= 1) & (xs // 16 <= 2) & (ys // 16 >= 1) & (ys // 16 <= 2)
    alpha = np.where(in_rect, g["opacity"] * np.exp(-((xs - 32.0) ** 2 + (ys - 32.0) ** 2) / 5.72), 0)
    assert np.allclose(o["final_T"], 1 - alpha, atol=tol, rtol=0)
    assert np.allclose(o["depth"], 2 * alpha, atol=2 * tol, rtol=0)
    assert np.allclose(o["rgb"], alpha[..., None] * np.array(g["rgb"]), atol=tol, rtol=0)
    for p in g["pixels"]:
        x, y = p["px"]
        assert abs((1 - o["final_T"][y, x]) - p["alpha"]) < tol
        if "depth" in p:
            assert abs(o["depth"][y, x] - p["depth"]) < 2 * tol
        if "rgb" in p:
            assert np.allclose(o["rgb"][y, x], p["rgb"], atol=tol)
    assert np.all(o["rgb"][:, :16] == 0) and np.all(o["final_T"][:, :16] == 1)
    # 2D scale = 4.8 px: small iff r >= 4.8 (inclusive)
    for r, small in ((4.81, True), (4.79, False)):
        v2 = make_view(g["f"], g["c"], g["w"], g["h"], lod=(r, 0.5, 10.0))
        f = oracle.render_view(s, v2, prec, pairs=False, image=False)["flags"][0]
        assert bool(f & oracle.F_SMALL) == small


def test_two_gaussian_occlusion():
    g = WORK["occlusion"]
    f, b = g["front"], g["back"]
    # same footprint in pixels: scale sigma with depth
    s = make_scene([[0, 0, b["z"]], [0, 0, f["z"]]], [[0.1 * b["z"]] * 3, [0.1 * f["z"]] * 3],
                   opacity=[b["o"], f["o"]], rgb=[b["rgb"], f["rgb"]])
    v = make_view(64.0, 32.0, 64, 64)
    o = oracle.render_view(s, v, "f64")
    c = o["rgb"][32, 32]
    assert c[1] <= g["max_back_weight"] + 1e-12 and c[1] > 0   # back (green) behind front
    assert abs(c[0] - 0.99) < 1e-12                              # front (red)
    # depth order is by z, not by index: the front Gaussian has the larger index
    assert list(o["pair_gauss"][:2]) == [1, 0]


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_equal_depth_ties_by_index(prec):
    """Reading R11: equal depths are ordered by ascending Gaussian index (a car
    face seen along a camera axis puts thousands of Gaussians at one depth).
    Three Gaussians at the same point and depth: the pair list of the centre
    tile lists them as 0, 1, 2, and the centre pixel blends them in that order
    (alpha = o there: power = 0), so its colour is the closed form
    c0 a0 + c1 a1 (1 - a0) + c2 a2 (1 - a0)(1 - a1)."""
    o_ = [0.6, 0.5, 0.4]
    rgb = [[1.0, 0, 0], [0, 1.0, 0], [0, 0, 1.0]]
    s = make_scene([[0, 0, 5.0]] * 3, 0.3, opacity=o_, rgb=rgb)
    v = make_view(64.0, 32.0, 64, 64)
    o = oracle.render_view(s, v, prec)
    tile = (32 // 16) * 4 + 32 // 16
    pt, pg = o["pair_tile"], o["pair_gauss"]
    assert list(pg[pt == tile]) == [0, 1, 2]
    a = [np.float32(x) if prec == "f32" else np.float64(np.float32(x)) for x in o_]
    want = [a[0], a[1] * (1 - a[0]), a[2] * (1 - a[0]) * (1 - a[1])]
    tol = 1e-6 if prec == "f32" else 1e-12
    assert np.allclose(o["rgb"][32, 32], want, atol=tol), (o["rgb"][32, 32], want)


def test_empty_scene_is_black():
    s = make_scene([[0, 0, -5.0]], 0.1)                 # behind the camera
    v = make_view(64.0, 32.0, 64, 64)
    o = oracle.render_view(s, v)
    assert np.all(o["rgb"] == 0) and np.all(o["depth"] == 0) and np.all(o["final_T"] == 1)
    assert o["stats"]["n_visible"] == 0 and o["stats"]["n_pairs"] == 0
    s0 = make_scene(np.zeros((0, 3)), 0.1)
    o = oracle.render_view(s0, v)
    assert np.all(o["rgb"] == 0) and o["stats"]["n_temporal"] == 0


def _random_small(seed, n=60, w=70, h=45, fresh=False, lod=(0.0, 0.5, 10.0)):
    scene, views = sg.make_random_dynamic(seed, n, 2, 10, w, h, 2, lod=lod, fresh=fresh)
    return scene, views


def test_out_of_frustum_gaussian_changes_nothing():
    scene, views = _random_small(4)
    v = views[0]
    a = oracle.render_view(scene, v)
    n = scene.n
    extra = make_scene([[0, 0, -3.0], [1e4, 0, 5.0]], 0.5)
    big = sg.Scene("x", *[np.concatenate([getattr(scene, k), getattr(extra, k)]) for k in
                          ("means_opacity", "scales", "rotations", "colors", "instance_ids",
                           "visibility", "life")], scene.num_instances)
    b = oracle.render_view(big, v)
    assert np.array_equal(a["rgb"], b["rgb"]) and np.array_equal(a["depth"], b["depth"])
    assert b["visible"][n:].sum() == 0


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_transmittance_invariant(prec):
    """sum_i w_i + T_final = 1 per pixel (telescoping of Eq.2), and T in [0,1]."""
    scene, views = _random_small(7, n=300, w=96, h=80, fresh=True)
    scene.colors[:, :3] = 1.0
    for v in views:
        o = oracle.render_view(scene, v, prec)
        tol = 2e-6 if prec == "f32" else 1e-13
        assert np.allclose(o["rgb"][..., 0] + o["final_T"], 1.0, atol=tol, rtol=0)
        assert np.all(o["final_T"] >= 0) and np.all(o["final_T"] <= 1)
        assert o["final_T"].min() < 0.5        # the invariant is exercised


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_tiled_blend_equals_bruteforce(seed, prec):
    """O5+O6 (pair list, tile ranges) == per-pixel gather + sort (bit-identical)."""
    scene, views = _random_small(seed, n=150, w=83, h=61, lod=(3.0, 0.5, 15.0))
    for v in views:
        o = oracle.render_view(scene, v, prec)
        rgb, depth, T = oracle.blend_bruteforce(scene, v, o["flags"], o["keys"], o["rect"], prec)
        assert np.array_equal(o["rgb"], rgb) and np.array_equal(o["depth"], depth)
        assert np.array_equal(o["final_T"], T)
        # pair list sorted by (tile, depth, index); ranges partition it
        pt, pg = o["pair_tile"], o["pair_gauss"]
        z = o["keys"][pg, 2]
        key = list(zip(pt.tolist(), z.tolist(), pg.tolist()))
        assert key == sorted(key)
        r = o["ranges"]
        assert r[0, 0] == 0 and r[-1, 1] == len(pt) and np.all(r[1:, 0] == r[:-1, 1])


@pytest.mark.parametrize("seed", [5, 6])
def test_rect_matches_pixel_enumeration(seed):
    """Tile rectangle == the tiles touched by the integer pixel box of
    mean +- ceil(3 sqrt(lambda_max(dilated Sigma'))) clipped to the image,
    with lambda from numpy eigvalsh (reading R12)."""
    scene, views = _random_small(seed, n=400, w=150, h=100)
    for v in views:
        o = oracle.render_view(scene, v, "f32", pairs=False, image=False)
        W, H = v.width, v.height
        for g in np.nonzero(o["flags"] & oracle.F_TEMPORAL)[0]:
            k = o["keys"][g].astype(np.float64)
            if np.isnan(k).any():
                continue
            lam = np.linalg.eigvalsh([[k[3] + 0.3, k[4]], [k[4], k[5] + 0.3]]).max()
            rf = 3 * math.sqrt(lam)
            if abs(rf - round(rf)) < 1e-4:
                continue                               # fp32 rounding may decide
            r = math.ceil(rf)
            xlo, xhi = math.ceil(k[0] - r), math.floor(k[0] + r)
            ylo, yhi = math.ceil(k[1] - r), math.floor(k[1] + r)
            if min(abs(k[0] - r - round(k[0] - r)), abs(k[1] - r - round(k[1] - r))) < 1e-4:
                continue
            vis = xlo <= W - 1 and xhi >= 0 and ylo <= H - 1 and yhi >= 0
            assert bool(o["flags"][g] & oracle.F_VISIBLE) == vis, g
            if vis:
                want = [max(xlo, 0) // 16, min(xhi, W - 1) // 16, max(ylo, 0) // 16,
                        min(yhi, H - 1) // 16]
                assert list(o["rect"][g]) == want


def test_single_anisotropic_gaussian_density():
    """alpha at each pixel == o exp(-1/2 d^T (Sigma'+0.3I)^-1 d) with the inverse
    from numpy (checks conic signs and the cross term)."""
    q = Rotation.from_euler("xyz", [0.3, -0.4, 0.7]).as_quat()
    s = make_scene([[0.3, -0.2, 4.0]], [[0.4, 0.1, 0.05]], quats=[[q[3], q[0], q[1], q[2]]],
                   opacity=0.6, rgb=[[1, 1, 1]])
    v = make_view(80.0, 40.0, 80, 80)
    o = oracle.render_view(s, v, "f64")
    k = o["keys"][0]
    Sinv = np.linalg.inv([[k[3] + 0.3, k[4]], [k[4], k[5] + 0.3]])
    ys, xs = np.mgrid[0:80, 0:80]
    d = np.stack([k[0] - xs, k[1] - ys], -1)
    a = 0.6 * np.exp(-0.5 * np.einsum("...i,ij,...j->...", d, Sinv, d))
    tx0, tx1, ty0, ty1 = o["rect"][0]
    m = (xs // 16 >= tx0) & (xs // 16 <= tx1) & (ys // 16 >= ty0) & (ys // 16 <= ty1)
    assert np.allclose(o["rgb"][..., 0], np.where(m, a, 0), atol=1e-12)
    assert abs(k[4]) > 0.1                            # the cross term matters


# --------------------------------------------------------------------------
# pipeline properties (acceptance 1 and 3)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("seed", [21, 22, 23, 24, 25])
def test_streamlined_equals_conventional(seed):
    """Streamlined (r = 0, fresh v, instance cameras) == conventional (objects
    transformed to world, projected through W_t) — acceptance 1.
    Exact poses and fp32-exact positions; the world quaternion q_i2g * q is
    stored in fp32 (~6e-8 relative), so fp64 images agree to the spec's 1e-5."""
    rng = np.random.default_rng(seed)
    K, per, nst = 3, 40, 150
    poses = [_dyadic_pose(rng) for _ in range(K)]
    for k in range(K):
        poses[k] = (poses[k][0], poses[k][1] + np.array([0, 0, 12.0]))
    pts_s = np.stack([rng.uniform(-6, 6, nst), rng.uniform(-4, 4, nst), rng.uniform(3, 25, nst)], 1)
    pts_d = rng.uniform(-2, 2, (K * per, 3)).astype(np.float32).astype(np.float64)
    pts_s = pts_s.astype(np.float32).astype(np.float64)
    ids = np.concatenate([np.zeros(nst), np.repeat(np.arange(1, K + 1), per)]).astype(np.int32)
    n = nst + K * per
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q = q.astype(np.float32).astype(np.float64)
    sig = np.exp(rng.uniform(-3.5, -0.5, (n, 3)))
    col = rng.random((n, 3))
    op = rng.uniform(0.05, 0.99, n)
    loc = make_scene(np.concatenate([pts_s, pts_d]), sig, quats=q, opacity=op, rgb=col, ids=ids,
                     num_instances=K + 1)
    pw, qw = np.concatenate([pts_s, pts_d]), q.copy()
    for k, (R, t) in enumerate(poses):
        sl = ids == k + 1
        pw[sl] = pw[sl] @ R.T + t
        qk = Rotation.from_matrix(R).as_quat()
        qk = np.array([qk[3], qk[0], qk[1], qk[2]])
        qw[sl] = [quat_mul(qk, qq) for qq in q[sl]]
    wor = make_scene(pw, sig, quats=qw, opacity=op, rgb=col, num_instances=1)
    i2g = np.stack([np.concatenate([R, t[:, None]], 1) for R, t in poses])
    a = oracle.render_view(loc, make_view(100.0, 64.0, 128, 128, i2g=i2g), "f64")
    b = oracle.render_view(wor, make_view(100.0, 64.0, 128, 128), "f64")
    assert np.array_equal(a["flags"], b["flags"])
    assert np.abs(a["rgb"] - b["rgb"]).max() < 1e-5
    assert a["stats"]["n_rendered"] > 50


def test_conservativeness_after_sweep():
    """After one sweep over the training views with fresh intervals and a commit,
    the streamlined visible set at every training view equals the frustum set of
    the unfiltered render (S:203, S:681 acceptance 3)."""
    scene, views = sg.make_random_dynamic(31, 400, 3, 30, 96, 64, 6, fresh=True)
    times = [-1.0, -0.5, 0.0, 0.25, 0.5, 1.0]
    for v, t in zip(views, times):
        v.t = t
    ref = []
    for v in views:
        o = oracle.render_view(scene, v, pairs=False, image=False)
        ref.append(o["visible"].copy())
        oracle.update_life(scene, o["visible"], v.t)
    oracle.commit_visibility(scene, 0.1)
    n_filtered = 0
    for v, m in zip(views, ref):
        o = oracle.render_view(scene, v, pairs=False, image=False)
        assert np.array_equal(o["visible"], m)
        n_filtered += scene.n - o["stats"]["n_temporal"]
    assert n_filtered > 0                      # the filter did remove Gaussians


def test_bad_instance_and_near_plane():
    s = make_scene([[0, 0, 3.0], [0, 0, 3.0], [0, 0, 0.005], [0, 0, 0.02]],
                   [[0.1] * 3, [0.1] * 3, [0.1] * 3, [0.1] * 3], ids=[0, 5, 0, 0], num_instances=1)
    v = make_view(64.0, 32.0, 64, 64)
    o = oracle.render_view(s, v)
    assert o["rc"] == -2 and o["stats"]["n_bad_instance"] == 1
    assert o["flags"][1] & oracle.F_BADID and not o["flags"][1] & oracle.F_VISIBLE
    assert o["flags"][0] & oracle.F_VISIBLE
    assert not o["flags"][2] & oracle.F_VISIBLE                 # z <= near (0.01)
    # z just past the near plane: a huge splat covering every tile (stress)
    assert o["flags"][3] & oracle.F_VISIBLE and list(o["rect"][3]) == [0, 3, 0, 3]


def test_f32_contract_tracks_f64_shadow():
    """The fp32 contract stays within rounding of the fp64 shadow: keys to 1e-5
    relative, decisions identical except near thresholds, images within 1e-4 on
    all but a handful of pixels (decision flips)."""
    scene, views = sg.make_config("street", scale=0.05, n_views=2, width=320, height=224)
    for v in views:
        a = oracle.render_view(scene, v, "f32")
        b = oracle.render_view(scene, v, "f64")
        m = ~np.isnan(a["keys"][:, 0])
        ka, kb = a["keys"][m].astype(np.float64), b["keys"][m]
        scale = np.maximum(np.abs(kb), np.abs(kb[:, 3:4]) + np.abs(kb[:, 5:6]))
        assert np.all(np.abs(ka - kb) <= 1e-5 * np.maximum(scale, 1.0))
        same = (a["flags"] == b["flags"]).mean()
        assert same > 0.999
        d = np.abs(a["rgb"] - b["rgb"]).max(-1)
        assert (d > 1e-4).mean() < 2e-3


def test_exp2_contract():
    """s3r_exp2 vs the exact 2^x: <= 2.02 ulp on [-24, 0]; 2^0 = 1 and 2^-n exact;
    flush below -24."""
    xs = np.float32(-np.linspace(0, 24, 240001))
    worst = 0.0
    for x in xs:
        got = np.float32(oracle.exp2_32(float(x)))
        want = 2.0 ** float(x)
        ulp = float(np.spacing(np.float32(want)))
        worst = max(worst, abs(float(got) - want) / ulp)
    assert worst < WORK["exp"]["max_ulp"]
    for k in range(25):
        assert oracle.exp2_32(-float(k)) == 2.0 ** -k
    assert oracle.exp2_32(-24.01) == 0.0 and oracle.exp2_32(-1e30) == 0.0


# --------------------------------------------------------------------------
# Eq.2 edge rules of reading R14: the 0.99
# clamp on alpha and include-then-stop at T < 1e-4.  Each expectation is a
# closed form of the concentric-Gaussian stack at its common centre pixel,
# where power = 0 and exp(power) = 1 exactly.
# --------------------------------------------------------------------------

def _concentric(zs, opac, rgb):
    """Gaussians on the optical axis with the same 3.2-px footprint (sigma
    proportional to z), so every one of them covers the centre pixel (32, 32)
    of a 64x64 view (f = 64, c = 32) with power = 0 there."""
    return make_scene([[0, 0, z] for z in zs], [[0.05 * z] * 3 for z in zs],
                      opacity=opac, rgb=rgb)


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_early_termination_include_then_stop(prec):
    """Five concentric o = 0.95 Gaussians: T = (1 - o)^k after k of them.
    0.05^3 = 1.25e-4 >= 1e-4, so the 4th is blended; 0.05^4 = 6.25e-6 < 1e-4,
    so blending stops and the 5th is not.  Discriminates: a threshold of 1e-3
    (would stop after the 3rd: no blue), stop-before-include (would refuse the
    4th because T would fall below: no blue), no termination at all (green >
    0).  Expectations use the fp32-stored opacity (the scene is fp32)."""
    zs = [2.0, 3.0, 4.0, 5.0, 6.0]
    rgb = np.zeros((5, 3))
    rgb[3] = [0, 0, 1]          # only the 4th carries blue
    rgb[4] = [0, 1, 0]          # only the 5th carries green
    o = oracle.render_view(_concentric(zs, 0.95, rgb), make_view(64.0, 32.0, 64, 64), prec)
    a = float(np.float32(0.95))
    q = 1.0 - a
    tol = 1e-4 if prec == "f32" else 1e-12          # relative; fp32: the T - w chain
    T = float(o["final_T"][32, 32])
    assert abs(T - q ** 4) <= tol * q ** 4
    blue = float(o["rgb"][32, 32, 2])
    assert abs(blue - a * q ** 3) <= tol * a * q ** 3
    assert o["rgb"][32, 32, 1] == 0.0 and o["rgb"][32, 32, 0] == 0.0
    want_d = sum(a * q ** k * z for k, z in enumerate(zs[:4]))
    assert abs(o["depth"][32, 32] - want_d) <= tol * want_d
    # the neighbouring pixel (power < 0) is not terminated after 4: T stays larger
    assert o["final_T"][32, 34] > 1e-4


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_termination_threshold_is_strict_1e4(prec):
    """o chosen so that T after two Gaussians is 1.2e-4 (>= 1e-4, continue) and
    after three is 2.4e-6 (< 1e-4, stop): alpha_1 = 0.99 (clamped from 0.995),
    alpha_2 = 0.988, alpha_3 = 0.98.  A 4th Gaussian must not contribute and a
    threshold of 2e-4 or 1e-3 would drop the 3rd's red."""
    zs = [2.0, 3.0, 4.0, 5.0]
    rgb = np.array([[0, 0, 0], [0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    o = oracle.render_view(_concentric(zs, [0.995, 0.988, 0.98, 0.9], rgb),
                           make_view(64.0, 32.0, 64, 64), prec)
    a2, a3 = float(np.float32(0.988)), float(np.float32(0.98))
    T2 = (1 - 0.99) * (1 - a2)
    tol = 1e-4 if prec == "f32" else 1e-12
    assert T2 > 1e-4 and T2 * (1 - a3) < 1e-4
    assert abs(o["rgb"][32, 32, 0] - a3 * T2) <= tol * a3 * T2
    assert o["rgb"][32, 32, 1] == 0.0
    assert abs(o["final_T"][32, 32] - (1 - a3) * T2) <= tol * (1 - a3) * T2


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_alpha_clamp_at_099(prec):
    """alpha = min(0.99, o exp(power)) (reading R14): a front Gaussian of
    opacity 0.999 blends with weight 0.99 at its centre (not 0.999) and leaves
    T = 0.01 for the one behind it (o = 0.5 -> weight 0.005); away from the
    centre, where o exp(power) < 0.99, the clamp is inactive and alpha is the
    closed form o exp(-r^2 / (2 s^2)) of the isotropic splat."""
    zs = [2.0, 4.0]
    rgb = np.array([[1, 0, 0], [0, 1, 0]], float)
    s = _concentric(zs, [0.999, 0.5], rgb)
    o = oracle.render_view(s, make_view(64.0, 32.0, 64, 64), prec)
    tol = 2e-6 if prec == "f32" else 1e-12
    assert abs(o["rgb"][32, 32, 0] - 0.99) <= tol
    assert abs(o["final_T"][32, 32] - 0.01 * 0.5) <= tol * 0.01
    assert abs(o["rgb"][32, 32, 1] - 0.005) <= tol * 0.01
    # off centre: the front splat's Sigma' = (64 sigma / z)^2 I (+0.3 dilation),
    # sigma = fp32(0.1) as stored
    op = float(np.float32(0.999))
    s2 = (64.0 * float(np.float32(0.1)) / 2.0) ** 2 + 0.3
    for dx in (3, 5):
        a = op * math.exp(-0.5 * dx * dx / s2)
        assert a < 0.99
        assert abs(o["rgb"][32, 32 + dx, 0] - a) <= (4e-6 if prec == "f32" else 1e-12)
