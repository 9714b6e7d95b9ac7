"""Config-level parity at the configured sizes (BASELINE.json configs C2, C4, C5)
in the launch configuration bench.py times, CUDA path vs the CPU oracle.

north_star: "bit-exact indexing and sub-1e-4 images against the oracle on all
five configs"; gradients within 1e-3.  C1 and C3 are covered in
test_gpu_parity.py (test_c1_toy, test_full_size_av2_sampled).  The oracle runs
in forked worker processes on the host cores (the GPU results are computed
first and inherited by the workers; only verdicts come back).
"""
import multiprocessing as mp
import os
import traceback

import numpy as np
import pytest
import torch

import oracle
from paper_2503_08217_b200 import s3r
from paper_2503_08217_b200 import scenegen as sg
from test_gpu_parity import _check_grads, _grads_like, compare_dump, gpu_dump, gpu_render

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

_G = {}     # inherited by the forked oracle workers


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = s3r.Context(0)
    c.set_debug(True)
    yield c
    c.close()


def _workers():
    n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return max(1, min(n, 16))   # each oracle worker holds ~0.8 GB at C4


def _full_job(vi):
    """Element-by-element comparison of view vi (every K1-K7 output)."""
    try:
        o = oracle.render_view(_G["scene"], _G["views"][vi], "f32")
        compare_dump(_G["dumps"][vi], o)
        return vi, None
    except Exception:                       # noqa: BLE001
        return vi, traceback.format_exc(limit=3)


def _counts_job(vi):
    """Per-view counts (K1-K4 decisions) of view vi against the oracle."""
    try:
        o = oracle.render_view(_G["scene"], _G["views"][vi], "f32", pairs=False, image=False)
        st = _G["stats"][vi]
        for k in ("n_temporal", "n_visible", "n_lod_small", "n_lod_dropped", "n_rendered",
                  "n_pairs", "n_bad_instance"):
            assert st[k] == o["stats"][k], (k, st[k], o["stats"][k])
        return vi, None
    except Exception:                       # noqa: BLE001
        return vi, traceback.format_exc(limit=3)


def _run_pool(fn, items):
    oracle.lib()                            # built and loaded before the fork
    with mp.get_context("fork").Pool(min(_workers(), len(items))) as pool:
        res = pool.map(fn, items)
    bad = [(vi, err) for vi, err in res if err]
    assert not bad, bad[:3]
    return len(res)


def test_c4_drive_full_size(ctx):
    """C4 (10 M Gaussians, 127 instances, 2 km, ~10 % temporal pass, 1550x2048,
    P:312) as bench.py renders it on one GPU: the configured 256 views in one
    s3r_render_batch.  Per-view counts of all 256 views against the oracle; two
    sampled views element by element (keys, decisions, order, pairs, ranges,
    images bit-identical)."""
    scene, views = sg.make_config("drive")
    assert scene.n == 10_000_000 and scene.num_instances == 128 and len(views) == 256
    ds, tabs, outs, rc = gpu_render(ctx, scene, views, visible=False)
    assert rc == 0
    pick = [int(v) for v in sorted(np.random.default_rng(4).choice(len(views), 2, replace=False))]
    _G.clear()
    _G.update(scene=scene, views=views, stats=[ctx.stats(i) for i in range(len(views))],
              dumps={vi: gpu_dump(ctx, views[vi], vi, outs[vi]) for vi in pick})
    del outs, ds, tabs
    torch.cuda.empty_cache()
    assert _run_pool(_counts_job, list(range(len(views)))) == 256
    assert _run_pool(_full_job, pick) == 2
    frac = np.mean([s["n_temporal"] for s in _G["stats"]]) / scene.n
    assert 0.05 < frac < 0.15, frac          # the configured ~10 % temporal pass


def test_c2_street_full_size(ctx):
    """C2 at its configured size (200 k Gaussians, 10 instances, 960x640, ~40 %
    temporal pass) as bench.py renders it: all 100 frames in one batch, every
    view element by element."""
    scene, views = sg.make_config("street")
    assert scene.n == 200_000 and len(views) == 100
    ds, tabs, outs, rc = gpu_render(ctx, scene, views)
    assert rc == 0
    _G.clear()
    _G.update(scene=scene, views=views,
              dumps={vi: gpu_dump(ctx, v, vi, outs[vi]) for vi, v in enumerate(views)})
    del outs
    assert _run_pool(_full_job, list(range(len(views)))) == 100
    frac = np.mean([d["stats"]["n_temporal"] for d in _G["dumps"].values()]) / scene.n
    assert 0.35 < frac < 0.45, frac


def test_c5_backward_full_size_av2_view(ctx):
    """C5 (training step on the C3 scene): the 64-view training batch bench.py
    times, MSE cotangent (noisy targets, s3r_mse) on one sampled full-size view
    and zero on the others; per-Gaussian gradients and that view's pose
    gradient against the fp64 oracle adjoint (1e-3 gates of _check_grads)."""
    scene, views = sg.make_config("av2")
    ds = s3r.DeviceScene.from_numpy(scene)
    tabs = s3r.view_tables(ctx, views)
    outs = s3r.alloc_outputs(views, depth=False, final_T=False)
    vi = int(np.random.default_rng(5).integers(len(views)))
    v = views[vi]
    ctx.set_training(True)
    try:
        ctx.render_batch(ds, views, list(tabs), outs)
        rng = np.random.default_rng(6)
        tgt = torch.clamp(outs[vi]["rgb"] + 0.05 * torch.from_numpy(
            rng.standard_normal(outs[vi]["rgb"].shape).astype(np.float32)).cuda(), 0, 1)
        g_img = torch.empty_like(outs[vi]["rgb"])
        loss = torch.zeros(1, device="cuda")
        ctx.mse(outs[vi]["rgb"], tgt, 1.0 / g_img.numel(), g_img, loss)
        cots = [{"rgb": g_img if i == vi else torch.zeros_like(outs[i]["rgb"])}
                for i in range(len(views))]
        grads = _grads_like(ds)
        grads["table"] = torch.zeros((len(views), scene.num_instances, 12), device="cuda")
        ctx.render_backward(ds, views, list(tabs), cots, grads)
        torch.cuda.synchronize()
    finally:
        ctx.set_training(False)
    g_gpu = np.concatenate([grads[k].cpu().numpy() for k in
                            ("means_opacity", "scales", "rotations", "colors")], 1)
    gt_ref = np.zeros((scene.num_instances, 12))
    g_ref = oracle.backward(scene, v, g_img.cpu().numpy().astype(np.float64), g_table=gt_ref)
    assert np.count_nonzero(np.abs(g_ref).sum(1)) > 10_000
    _check_grads(g_gpu, g_ref)
    got = grads["table"][vi].cpu().numpy().astype(np.float64)
    for i in range(scene.num_instances):
        ref = np.abs(gt_ref[i]).max()
        if ref > 0:
            assert np.abs(got[i] - gt_ref[i]).max() <= 1e-3 * ref, i
    others = torch.cat([grads["table"][:vi], grads["table"][vi + 1:]])
    assert float(others.abs().max()) == 0.0


def _opaque_scene(seed):
    scene, views = sg.make_random_dynamic(seed, 3000, 3, 300, 173, 129, 4, lod=(2.0, 0.5, 12.0))
    rng = np.random.default_rng(seed)
    hi = rng.random(scene.n) < 0.4
    # opacity in (0.99, 1): alpha = min(0.99, o exp(power)) clamps near the centre
    scene.means_opacity[hi, 3] = (0.99 + 0.0099 * rng.random(hi.sum())).astype(np.float32)
    return scene, views, hi


@pytest.mark.parametrize("seed", [81, 82])
def test_alpha_clamp_forward_and_backward(ctx, seed):
    """Opacities in (0.99, 1) so that the alpha = 0.99 clamp of Eq.2 (reading
    R14) bites near splat centres: forward bit-exact vs the oracle, backward
    (clamped alpha passes no gradient) within the 1e-3 gates."""
    from test_gpu_parity import check_view
    scene, views, hi = _opaque_scene(seed)
    _, tabs, outs, rc = gpu_render(ctx, scene, views)
    assert rc == 0
    n_clamp = 0
    for vi, v in enumerate(views):
        o = check_view(ctx, scene, v, tabs[vi], outs[vi], vi)
        n_clamp += int(np.count_nonzero((o["flags"] & oracle.F_RENDERED).astype(bool) & hi))
    assert n_clamp > 500, n_clamp
    rng = np.random.default_rng(seed)
    cot = [{"rgb": rng.standard_normal((v.height, v.width, 3))} for v in views]
    ds = s3r.DeviceScene.from_numpy(scene)
    outs = s3r.alloc_outputs(views)
    ctx.set_training(True)
    try:
        ctx.render_batch(ds, views, list(tabs), outs)
        cots = [{"rgb": torch.from_numpy(c["rgb"].astype(np.float32)).cuda()} for c in cot]
        grads = _grads_like(ds)
        ctx.render_backward(ds, views, list(tabs), cots, grads)
        torch.cuda.synchronize()
    finally:
        ctx.set_training(False)
    g_gpu = np.concatenate([grads[k].cpu().numpy() for k in
                            ("means_opacity", "scales", "rotations", "colors")], 1)
    g_ref = np.zeros((scene.n, 16))
    for v, c in zip(views, cot):
        oracle.backward(scene, v, c["rgb"], grads=g_ref)
    _check_grads(g_gpu, g_ref)


def test_binding_rejects_bad_buffers(ctx):
    """The binding's argument checks with real device tensors: a wrong-shaped
    output, a float64 table and a too-short gradient buffer raise ValueError
    before anything is launched."""
    scene, views = sg.make_toy()
    ds = s3r.DeviceScene.from_numpy(scene)
    tabs = s3r.view_tables(ctx, views)
    outs = s3r.alloc_outputs(views)
    bad = [{"rgb": torch.empty((views[0].height, views[0].width), device="cuda")}]
    with pytest.raises(ValueError, match="rgb"):
        ctx.render_batch(ds, views, list(tabs), bad)
    with pytest.raises(ValueError, match="3x4"):
        ctx.render_batch(ds, views, [tabs[0].double()], outs)
    ctx.set_training(True)
    try:
        ctx.render_batch(ds, views, list(tabs), outs)
        g = _grads_like(ds)
        g["colors"] = g["colors"][:-1]
        with pytest.raises(ValueError, match="colors"):
            ctx.render_backward(ds, views, list(tabs), [{"rgb": torch.zeros_like(outs[0]["rgb"])}], g)
    finally:
        ctx.set_training(False)
