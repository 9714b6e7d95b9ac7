"""Capacity mode (s3r_set_capacity): the batch is sized on the device
(k_plan.cu) instead of by two host readbacks, so a render can be captured in a
CUDA graph.  Outputs must be bit-identical to the synchronous mode; a view
that does not fit is rendered empty and reported by s3r_check."""
import numpy as np
import pytest
import torch

from paper_2503_08217_b200 import s3r
from paper_2503_08217_b200 import scenegen as sg

pytestmark = pytest.mark.gpu

KEYS = ("rgb", "depth", "final_T", "visible")
STATS = ("n_temporal", "n_visible", "n_lod_small", "n_lod_dropped", "n_rendered", "n_pairs",
         "n_bin_pairs")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def _render(ctx, ds, views, tabs, n):
    outs = s3r.alloc_outputs(views, n_visible=n)
    ctx.render_batch(ds, views, tabs, outs)
    torch.cuda.synchronize()
    return outs


@pytest.mark.parametrize("case", ["dynamic", "street"])
def test_capacity_mode_matches_sync_mode(dev, case):
    if case == "dynamic":
        scene, views = sg.make_random_dynamic(31, 6000, 4, 400, 211, 147, 7, lod=(3.0, 0.5, 12.0))
        views[3].t = views[2].t
    else:
        scene, views = sg.make_config("street", scale=0.25, n_views=12)
    a, b = s3r.Context(0), s3r.Context(0)
    try:
        tabs = list(s3r.view_tables(a, views))
        dsa = s3r.DeviceScene.from_numpy(scene)
        oa = _render(a, dsa, views, tabs, scene.n)
        sa = [a.stats(i) for i in range(len(views))]
        cap = a.capacity_from_last(1.0)          # exactly the need: every view fits
        b.set_capacity(cap)
        dsb = s3r.DeviceScene.from_numpy(scene)
        ob = _render(b, dsb, views, tabs, scene.n)
        assert b.check() == 0
        sb = [b.stats(i) for i in range(len(views))]
        for x, y in zip(oa, ob):
            for k in KEYS:
                assert torch.equal(x[k], y[k]), k
        assert torch.equal(dsa.life, dsb.life)
        for x, y in zip(sa, sb):
            for k in STATS:
                assert x[k] == y[k], k
        # the device-planned batch reports the same needs
        assert b.capacity_from_last(1.0) == cap
        # dumps need the host-side layout
        with pytest.raises(s3r.S3RError):
            b.dump(0, views[0].width, views[0].height, keys=False)
    finally:
        a.close()
        b.close()


def test_capacity_overflow_renders_empty_and_reports(dev):
    scene, views = sg.make_random_dynamic(32, 4000, 3, 300, 160, 120, 6, lod=(3.0, 0.5, 12.0))
    a, b = s3r.Context(0), s3r.Context(0)
    try:
        tabs = list(s3r.view_tables(a, views))
        oa = _render(a, s3r.DeviceScene.from_numpy(scene), views, tabs, scene.n)
        sa = [a.stats(i) for i in range(len(views))]
        need = a.capacity_from_last(1.0)
        # records for the first three views only: the later ones are dropped
        nt = [s["n_temporal"] for s in sa]
        cap = dict(need, records=sum(nt[:3]))
        b.set_capacity(cap)
        ob = _render(b, s3r.DeviceScene.from_numpy(scene), views, tabs, scene.n)
        assert b.check() == s3r.S3R_ECAPACITY
        assert b.check() == 0                     # the error word was consumed
        for i in range(3):
            for k in KEYS:
                assert torch.equal(oa[i][k], ob[i][k]), (i, k)
        for i in range(3, len(views)):
            assert float(ob[i]["rgb"].abs().max()) == 0.0
            assert torch.all(ob[i]["final_T"] == 1.0)
        # a too small per-view splat capacity drops the views above it
        big = max(range(len(views)), key=lambda i: sa[i]["n_rendered"])
        b.set_capacity(dict(need, rendered_view=sa[big]["n_rendered"] - 1))
        ob = _render(b, s3r.DeviceScene.from_numpy(scene), views, tabs, scene.n)
        assert b.check() == s3r.S3R_ECAPACITY
        assert float(ob[big]["rgb"].abs().max()) == 0.0
        for i in range(len(views)):
            if sa[i]["n_rendered"] < sa[big]["n_rendered"]:
                assert torch.equal(oa[i]["rgb"], ob[i]["rgb"]), i
        with pytest.raises(s3r.S3RError):
            b.set_capacity(dict(need, records=0))
    finally:
        a.close()
        b.close()


def test_self_planned_small_views(dev):
    """Capacity mode whose reservation makes every view small (C1): the one-CTA
    kernel plans its own view (no k_plan_bins); bit-identical to the
    synchronous mode, and a view above the reserved splat count renders empty
    with S3R_ECAPACITY."""
    scene, (v0,) = sg.make_toy()
    import dataclasses
    views = [v0, dataclasses.replace(v0, lod_seed=5), dataclasses.replace(v0, lod_seed=9)]
    a, b = s3r.Context(0), s3r.Context(0)
    try:
        tabs = list(s3r.view_tables(a, views))
        oa = _render(a, s3r.DeviceScene.from_numpy(scene), views, tabs, scene.n)
        sa = [a.stats(i) for i in range(len(views))]
        need = a.capacity_from_last(1.0)
        assert need["rendered_view"] <= 2048
        b.set_capacity(need)
        ob = _render(b, s3r.DeviceScene.from_numpy(scene), views, tabs, scene.n)
        assert b.check() == 0
        for x, y in zip(oa, ob):
            for k in KEYS:
                assert torch.equal(x[k], y[k]), k
        sb = [b.stats(i) for i in range(len(views))]
        for x, y in zip(sa, sb):
            for k in ("n_temporal", "n_visible", "n_rendered", "n_pairs"):
                assert x[k] == y[k], k
        big = max(range(len(views)), key=lambda i: sa[i]["n_rendered"])
        b.set_capacity(dict(need, rendered_view=sa[big]["n_rendered"] - 1))
        ob = _render(b, s3r.DeviceScene.from_numpy(scene), views, tabs, scene.n)
        assert b.check() == s3r.S3R_ECAPACITY
        assert float(ob[big]["rgb"].abs().max()) == 0.0
        for i in range(len(views)):
            if sa[i]["n_rendered"] < sa[big]["n_rendered"]:
                assert torch.equal(oa[i]["rgb"], ob[i]["rgb"]), i
    finally:
        a.close()
        b.close()


@pytest.mark.parametrize("case", ["toy", "street"])
def test_cuda_graph_replay(dev, case):
    """A capacity-mode render captured once in a CUDA graph and replayed equals
    the eager render bit for bit (and the graph re-renders fresh inputs: the
    scene tensors are read at replay time)."""
    if case == "toy":
        scene, views = sg.make_toy()
    else:
        scene, views = sg.make_config("street", scale=0.25, n_views=10)
    ctx = s3r.Context(0)
    try:
        tabs = list(s3r.view_tables(ctx, views))
        ds = s3r.DeviceScene.from_numpy(scene, life=False)
        ref = _render(ctx, ds, views, tabs, 0)
        ctx.set_capacity(ctx.capacity_from_last(1.1))
        outs = s3r.alloc_outputs(views)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):                # warm the capacity-mode scratch
            ctx.render_batch(ds, views, tabs, outs)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            ctx.render_batch(ds, views, tabs, outs)
        for o in outs:
            for k in ("rgb", "depth", "final_T"):
                o[k].fill_(-1.0)
        g.replay()
        torch.cuda.synchronize()
        assert ctx.check() == 0
        for x, y in zip(ref, outs):
            for k in ("rgb", "depth", "final_T"):
                assert torch.equal(x[k], y[k]), k
        # the graph reads the scene at replay: dimmed colours render dimmer
        ds.colors.mul_(0.5)
        g.replay()
        torch.cuda.synchronize()
        assert float(outs[0]["rgb"].sum()) < 0.75 * float(ref[0]["rgb"].sum())
        st = ctx.stats(0)
        assert st["n_rendered"] > 0
    finally:
        ctx.close()


@pytest.mark.parametrize("mode", ["jitter", "fast_exp", "counters"])
def test_capacity_mode_with_options(dev, mode):
    """The render options that the capacity mode keeps (LOD noisy offset, SFU
    exponential, work counters) give the synchronous mode's outputs bit for bit
    (and, for the counters, the same E_alg / E_exec per view)."""
    scene, views = sg.make_random_dynamic(34, 5000, 3, 300, 190, 131, 6, lod=(6.0, 0.4, 8.0))
    a, b = s3r.Context(0), s3r.Context(0)
    try:
        for c in (a, b):
            if mode == "jitter":
                c.set_lod_jitter(0.3, 0.2, 0.6)
            elif mode == "fast_exp":
                c.set_fast_exp(True)
            else:
                c.set_counters(True)
        tabs = list(s3r.view_tables(a, views))
        oa = _render(a, s3r.DeviceScene.from_numpy(scene), views, tabs, scene.n)
        sa = [a.stats(i) for i in range(len(views))]
        b.set_capacity(a.capacity_from_last(1.2))
        ob = _render(b, s3r.DeviceScene.from_numpy(scene), views, tabs, scene.n)
        assert b.check() == 0
        sb = [b.stats(i) for i in range(len(views))]
        for x, y in zip(oa, ob):
            for k in KEYS:
                assert torch.equal(x[k], y[k]), k
        keys = STATS + (("n_blend_evals", "n_blend_exec") if mode == "counters" else ())
        for x, y in zip(sa, sb):
            for k in keys:
                assert x[k] == y[k], k
    finally:
        a.close()
        b.close()


def test_capacity_mode_edge_cases(dev):
    """Capacity mode on the degenerate batches of test_edge_cases: an empty
    scene, a 1x1 view whose Gaussians are all filtered out by time, an empty
    view list; and graph capture without the capacity mode is refused."""
    import sys, os
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from helpers import make_scene, make_view
    cap = dict(records=64, rendered_view=64, bin_pairs=64, tile_entries=1024, temporal_view=64)
    c = s3r.Context(0)
    try:
        c.set_capacity(cap)
        s0 = make_scene(np.zeros((0, 3)), 0.1)
        v = make_view(64.0, 32.0, 40, 33)
        tabs = list(s3r.view_tables(c, [v]))
        o = _render(c, s3r.DeviceScene.from_numpy(s0), [v], tabs, 0)
        assert c.check() == 0
        assert float(o[0]["rgb"].abs().max()) == 0.0 and torch.all(o[0]["final_T"] == 1.0)
        s1 = make_scene([[0, 0, 3.0], [0.1, 0, 4.0]], 0.2, vis=[[0.5, 0.6], [0.7, 0.9]])
        v1 = make_view(64.0, 0.0, 1, 1, t=-0.0)
        tabs = list(s3r.view_tables(c, [v1]))
        o = _render(c, s3r.DeviceScene.from_numpy(s1), [v1], tabs, s1.n)
        assert c.check() == 0 and c.stats(0)["n_temporal"] == 0
        assert float(o[0]["final_T"].min()) == 1.0
        assert c.render_batch(s3r.DeviceScene.from_numpy(s1), [], [], []) == 0
        c.set_capacity(None)
        g = torch.cuda.CUDAGraph()
        ds = s3r.DeviceScene.from_numpy(s1)
        outs = s3r.alloc_outputs([v1])
        with pytest.raises(s3r.S3RError):
            with torch.cuda.graph(g):
                c.render_batch(ds, [v1], tabs, outs)
    finally:
        c.close()
