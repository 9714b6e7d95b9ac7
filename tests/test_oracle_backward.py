"""Pins for the oracle's fp64 adjoint (config 5): central finite differences of
the fp64 forward, on tiny scenes built so that no piecewise boundary is crossed
by the perturbation (every Gaussian's 3-sigma box stays inside one 16x16 tile,
opacities <= 0.6 so neither the 0.99 clamp nor termination is reached).
Gate (north_star): per attribute, max|g_adjoint - g_fd| <= 1e-3 max|g_fd|."""
import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle
from helpers import make_scene, make_view

ATTR = {"mean": [0, 1, 2], "opacity": [3], "scale": [4, 5, 6], "rot": [8, 9, 10, 11],
        "color": [12, 13, 14]}


def _scene(seed, n_static=8, n_dyn=4):
    """Gaussians centred on tile centres of a 64x48 image (f = 80, z in [3, 6])."""
    rng = np.random.default_rng(seed)
    centres = [(8 + 16 * i, 8 + 16 * j) for i in range(4) for j in range(3)]
    pick = rng.permutation(len(centres))
    n = n_static + n_dyn
    f, cx, cy = 80.0, 32.0, 24.0
    pts, ids = [], []
    Rk = Rotation.from_euler("z", 0.4).as_matrix()
    tk = np.array([0.1, -0.05, 0.3])
    for k in range(n):
        px, py = centres[pick[k % len(centres)]]
        px += rng.uniform(-1.5, 1.5)
        py += rng.uniform(-1.5, 1.5)
        z = rng.uniform(3.0, 6.0)
        pw = np.array([(px - cx) * z / f, (py - cy) * z / f, z])
        if k >= n_static:           # dynamic: store in the object's local frame
            ids.append(1)
            pts.append(Rk.T @ (pw - tk))
        else:
            ids.append(0)
            pts.append(pw)
    sig = np.exp(rng.uniform(np.log(0.01), np.log(0.03), (n, 3)))
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    s = make_scene(np.array(pts), sig, quats=q, opacity=rng.uniform(0.2, 0.6, n),
                   rgb=rng.random((n, 3)), ids=np.array(ids, np.int32), num_instances=2)
    i2g = np.concatenate([Rk, tk[:, None]], 1)[None]
    v = make_view(f, cx, 64, 48, cy=cy, i2g=i2g)
    return s, v, rng


def _loss(scene, view, wr, wd, wt):
    o = oracle.render_view(scene, view, "f64", pairs=False)
    return float((o["rgb"] * wr).sum() + (o["depth"] * wd).sum() + (o["final_T"] * wt).sum())


def _field(scene, col):
    arr = [scene.means_opacity, scene.scales, scene.rotations, scene.colors][col // 4]
    return arr, col % 4


@pytest.mark.parametrize("seed", [0, 1])
def test_adjoint_matches_central_differences(seed):
    s, v, rng = _scene(seed)
    H, W = v.height, v.width
    wr = rng.standard_normal((H, W, 3))
    wd = rng.standard_normal((H, W)) * 0.1
    wt = rng.standard_normal((H, W))
    o = oracle.render_view(s, v, "f64", pairs=False)
    assert o["stats"]["n_rendered"] == s.n and o["final_T"].min() > 1e-3   # no termination
    g = oracle.backward(s, v, wr, wd, wt)
    fd = np.zeros_like(g)
    for gi in range(s.n):
        for cols in ATTR.values():
            for col in cols:
                arr, c = _field(s, col)
                x0 = arr[gi, c]
                h = np.float32(max(abs(float(x0)) * 2e-4, 2e-5))
                arr[gi, c] = x0 + h
                xp = float(arr[gi, c])
                lp = _loss(s, v, wr, wd, wt)
                arr[gi, c] = x0 - h
                xm = float(arr[gi, c])
                lm = _loss(s, v, wr, wd, wt)
                arr[gi, c] = x0
                fd[gi, col] = (lp - lm) / (xp - xm)
    for name, cols in ATTR.items():
        d = np.abs(g[:, cols] - fd[:, cols]).max()
        ref = np.abs(fd[:, cols]).max()
        assert ref > 0
        assert d <= 1e-3 * ref, (name, d, ref)


def test_adjoint_is_linear_and_zero_for_zero_cotangent():
    s, v, rng = _scene(3)
    H, W = v.height, v.width
    z = np.zeros((H, W, 3))
    assert np.all(oracle.backward(s, v, z) == 0)
    a, b = rng.standard_normal((H, W, 3)), rng.standard_normal((H, W, 3))
    ga, gb = oracle.backward(s, v, a), oracle.backward(s, v, b)
    gab = oracle.backward(s, v, 2.0 * a - b)
    assert np.allclose(gab, 2.0 * ga - gb, rtol=1e-9, atol=1e-12)


def test_color_gradient_is_blend_weight_sum():
    """dL/dc_i for L = sum(rgb) is sum over pixels of w_i (closed form)."""
    s, v, _ = _scene(4)
    H, W = v.height, v.width
    g = oracle.backward(s, v, np.ones((H, W, 3)))
    # with all colours set to 1, rgb = sum_i w_i per pixel, so sum of dL/dc_r = sum rgb
    s.colors[:, :3] = 1.0
    o = oracle.render_view(s, v, "f64", pairs=False)
    assert abs(g[:, 12].sum() - o["rgb"][..., 0].sum()) < 1e-9 * o["rgb"][..., 0].sum()


@pytest.mark.parametrize("seed", [5, 6])
def test_pose_gradient_matches_central_differences(seed):
    """NEXT-1 pose gradient: dL/d(instance camera table) [K+1][12] (slot 0 =
    W_t, slot 1 = the dynamic object's W_t W_{t,i2g}) vs central differences
    of the fp64 forward with the perturbed table; gate 1e-3 of the largest."""
    s, v, rng = _scene(seed)
    H, W = v.height, v.width
    wr = rng.standard_normal((H, W, 3))
    wd = rng.standard_normal((H, W)) * 0.1
    wt = rng.standard_normal((H, W))
    tab = oracle.compose(v).copy()
    gt = np.zeros((s.num_instances, 12))
    oracle.backward(s, v, wr, wd, wt, table=tab, g_table=gt)

    def loss(t):
        o = oracle.render_view(s, v, "f64", table=t, pairs=False)
        return float((o["rgb"] * wr).sum() + (o["depth"] * wd).sum() + (o["final_T"] * wt).sum())

    fd = np.zeros_like(gt)
    for i in range(s.num_instances):
        for k in range(12):
            x0 = tab[i, k]
            h = np.float32(max(abs(float(x0)) * 1e-3, 1e-4))
            tab[i, k] = x0 + h
            xp, lp = float(tab[i, k]), loss(tab)
            tab[i, k] = x0 - h
            xm, lm = float(tab[i, k]), loss(tab)
            tab[i, k] = x0
            fd[i, k] = (lp - lm) / (xp - xm)
    for i in range(s.num_instances):
        ref = np.abs(fd[i]).max()
        assert ref > 0
        assert np.abs(gt[i] - fd[i]).max() <= 1e-3 * ref, (i, gt[i], fd[i])


def test_adjoint_with_noisy_offset_matches_central_differences():
    """Backward through the LOD noisy offset (NEXT-3; reading R23: the offset is
    a constant of the backward).  Every Gaussian is LOD-small (r = 4 px), kept
    (p_max = 0) and beyond D (normalize(d) = 1), so its offset does not depend
    on the parameters and central differences of the fp64 forward measure the
    same derivative."""
    import dataclasses
    s, v, rng = _scene(8)
    v = dataclasses.replace(v, lod_r=4.0, lod_pmax=0.0, lod_D=2.0, lod_seed=77,
                            lod_jitter=(0.01, 0.01, 0.02))
    H, W = v.height, v.width
    wr = rng.standard_normal((H, W, 3))
    o = oracle.render_view(s, v, "f64", pairs=False)
    assert np.all(o["flags"] & oracle.F_JITTERED) and o["stats"]["n_rendered"] == s.n
    assert o["final_T"].min() > 1e-3
    g = oracle.backward(s, v, wr)
    fd = np.zeros_like(g)
    for gi in range(s.n):
        for cols in ATTR.values():
            for col in cols:
                arr, c = _field(s, col)
                x0 = arr[gi, c]
                h = np.float32(max(abs(float(x0)) * 2e-4, 2e-5))
                arr[gi, c] = x0 + h
                xp = float(arr[gi, c])
                lp = _loss(s, v, wr, 0, 0)
                arr[gi, c] = x0 - h
                xm = float(arr[gi, c])
                lm = _loss(s, v, wr, 0, 0)
                arr[gi, c] = x0
                fd[gi, col] = (lp - lm) / (xp - xm)
    for name, cols in ATTR.items():
        d = np.abs(g[:, cols] - fd[:, cols]).max()
        ref = np.abs(fd[:, cols]).max()
        assert ref > 0
        assert d <= 1e-3 * ref, (name, d, ref)
    # and the offset matters: the gradient differs from the unmoved render's
    g0 = oracle.backward(s, dataclasses.replace(v, lod_jitter=(0.0, 0.0, 0.0)), wr)
    assert not np.allclose(g0, g)


# --------------------------------------------------------------------------
# The adjoint's piecewise branches (reading R14): pixels where the front splat's
# alpha is clamped at 0.99 and pixels whose list terminates at T < 1e-4.
# Central differences of the fp64 forward are valid there as long as the
# perturbation crosses no branch boundary; the cotangent is restricted to
# pixels whose margins to every boundary (clamp, termination) exceed the
# perturbation's effect by orders of magnitude.  The margins are evaluated
# from the oracle's exported keys with a plain numpy loop (pixel selection
# only; the pin itself is the finite difference).
# --------------------------------------------------------------------------

def _stack_scene(seed):
    """Six near-concentric, mildly anisotropic Gaussians around the non-integer
    pixel (24.4, 23.7) of a 64x48 view (f = 80): the front one has o = 0.999
    (alpha clamped near the centre), the others o in [0.90, 0.96] so the centre
    pixels terminate after 4-5 of them; two low-opacity ones elsewhere."""
    rng = np.random.default_rng(seed)
    f, cx, cy = 80.0, 32.0, 24.0
    zs = [2.0, 2.6, 3.1, 3.7, 4.4, 5.2]
    ops = [0.999, 0.95, 0.93, 0.96, 0.90, 0.94]
    pts, sig = [], []
    for i, z in enumerate(zs):
        if i == 0:      # the clamped front splat: within 0.1 px of pixel (24, 24)
            px, py = 24.05 + rng.uniform(-0.04, 0.04), 23.95 + rng.uniform(-0.04, 0.04)
        else:
            px, py = 24.4 + rng.uniform(-0.3, 0.3), 23.7 + rng.uniform(-0.3, 0.3)
        pts.append([(px - cx) * z / f, (py - cy) * z / f, z])
        sig.append(0.045 * z * rng.uniform(0.85, 1.15, 3))
    for (px, py, z) in [(50.5, 10.2, 3.0), (44.1, 38.6, 4.0)]:
        pts.append([(px - cx) * z / f, (py - cy) * z / f, z])
        sig.append(0.02 * z * np.ones(3))
        ops.append(0.4)
    n = len(pts)
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    s = make_scene(np.array(pts), np.array(sig), quats=q, opacity=np.array(ops),
                   rgb=rng.random((n, 3)))
    return s, make_view(f, cx, 64, 48, cy=cy), rng


def _pixel_margins(s, v):
    """Per pixel: (clamped anywhere, terminated, min relative margin to the 0.99
    clamp, min relative margin of T_k to 1e-4) from the f64 keys, in the oracle's
    depth order (the stack's z are distinct)."""
    o = oracle.render_view(s, v, "f64")
    k = o["keys"]
    rend = np.nonzero(o["flags"] & oracle.F_RENDERED)[0]
    rend = rend[np.argsort(k[rend, 2])]
    H, W = v.height, v.width
    clamp = np.zeros((H, W), bool)
    term = np.zeros((H, W), bool)
    mc = np.full((H, W), np.inf)
    mt = np.full((H, W), np.inf)
    rect = o["rect"]
    for py in range(H):
        for px in range(W):
            T = 1.0
            for g in rend:
                x0, x1, y0, y1 = rect[g]
                if not (x0 <= px // 16 <= x1 and y0 <= py // 16 <= y1):
                    continue
                mx, my, z, a, b, c = k[g]
                ad, cd = a + 0.3, c + 0.3
                det = ad * cd - b * b
                A, B, C = cd / det, -b / det, ad / det
                dx, dy = mx - px, my - py
                pw = min(0.0, -0.5 * (A * dx * dx + C * dy * dy) - B * dx * dy)
                og = float(s.means_opacity[g, 3]) * np.exp(pw)
                mc[py, px] = min(mc[py, px], abs(og / 0.99 - 1.0))
                clamp[py, px] |= og >= 0.99
                T = T * (1.0 - min(0.99, og))
                mt[py, px] = min(mt[py, px], abs(T / 1e-4 - 1.0))
                if T < 1e-4:
                    term[py, px] = True
                    break
    return clamp, term, mc, mt


@pytest.mark.parametrize("seed", [11, 12])
def test_adjoint_at_clamped_and_terminated_pixels(seed):
    s, v, rng = _stack_scene(seed)
    H, W = v.height, v.width
    clamp, term, mc, mt = _pixel_margins(s, v)
    safe = (mc > 2e-3) & (mt > 2e-2)
    assert (safe & clamp).sum() >= 1 and (safe & term).sum() >= 4
    mask = safe & (clamp | term)
    wr = rng.standard_normal((H, W, 3)) * mask[..., None]
    wd = rng.standard_normal((H, W)) * 0.1 * mask
    wt = rng.standard_normal((H, W)) * mask * 100.0      # final T ~ 1e-5 there
    g = oracle.backward(s, v, wr, wd, wt)
    fd = np.zeros_like(g)
    for gi in range(s.n):
        for cols in ATTR.values():
            for col in cols:
                arr, c = _field(s, col)
                x0 = arr[gi, c]
                h = np.float32(max(abs(float(x0)) * 2e-5, 2e-6))
                arr[gi, c] = x0 + h
                xp = float(arr[gi, c])
                lp = _loss(s, v, wr, wd, wt)
                arr[gi, c] = x0 - h
                xm = float(arr[gi, c])
                lm = _loss(s, v, wr, wd, wt)
                arr[gi, c] = x0
                fd[gi, col] = (lp - lm) / (xp - xm)
    for name, cols in ATTR.items():
        d = np.abs(g[:, cols] - fd[:, cols]).max()
        ref = np.abs(fd[:, cols]).max()
        assert ref > 0
        assert d <= 1e-3 * ref, (name, d, ref)
    # the clamped front splat passes no opacity gradient through its clamped
    # pixels: with the cotangent on those pixels only, dL/do_0 == 0 (FD agrees)
    only = safe & clamp
    wr0 = rng.standard_normal((H, W, 3)) * only[..., None]
    g0 = oracle.backward(s, v, wr0)
    arr = s.means_opacity
    x0 = arr[0, 3]
    h = np.float32(1e-4)
    arr[0, 3] = x0 + h
    lp = _loss(s, v, wr0, 0, 0)
    arr[0, 3] = x0 - h
    lm = _loss(s, v, wr0, 0, 0)
    arr[0, 3] = x0
    assert g0[0, 3] == 0.0 and abs(lp - lm) < 1e-12
