"""Randomised parity: small scenes drawn over the input space (image sizes from
1x1 to a few hundred pixels, focal lengths, Gaussian counts including 0, LOD on
and off, the noisy offset, opacities up to the 0.99 clamp, shared view times,
near-plane and behind-camera splats), each rendered on the GPU in the
synchronous and the capacity mode and compared with the CPU oracle element by
element (bit-exact), and the two modes with each other."""
import dataclasses

import numpy as np
import pytest
import torch

import oracle
from paper_2503_08217_b200 import s3r
from paper_2503_08217_b200 import scenegen as sg
from test_gpu_parity import compare_dump, gpu_dump

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    n_static = int(rng.choice([0, 1, 7, 300, 2500]))
    n_obj = int(rng.integers(0, 4))
    per = int(rng.choice([1, 50, 200]))
    W = int(rng.choice([1, 16, 17, 63, 130, 257]))
    H = int(rng.choice([1, 15, 33, 96, 191]))
    nv = int(rng.integers(1, 5))
    lod = (float(rng.choice([0.0, 2.0, 6.0])), float(rng.uniform(0, 1)), float(rng.uniform(2, 30)))
    scene, views = sg.make_random_dynamic(seed + 77, n_static, n_obj, per, max(W, 2), max(H, 2), nv,
                                          lod=lod, fresh=bool(rng.random() < 0.3))
    n = scene.n
    if n:
        hi = rng.random(n) < 0.2            # opacities in (0.99, 1): the alpha clamp
        scene.means_opacity[hi, 3] = (0.99 + 0.0099 * rng.random(hi.sum())).astype(np.float32)
        near = rng.random(n) < 0.01         # a few splats at the near plane / behind the camera
        scene.means_opacity[near, 2] = rng.choice([0.02, -1.0, 0.0105], near.sum()).astype(np.float32)
    f = float(rng.choice([0.3, 1.0, 4.0])) * max(W, 2)
    views = [dataclasses.replace(v, width=W, height=H, fx=f, fy=f * v.fy / v.fx,
                                 cx=W / 2.0 + rng.uniform(-3, 3), cy=H / 2.0 + rng.uniform(-3, 3))
             for v in views]
    if nv > 1 and rng.random() < 0.5:
        views[1] = dataclasses.replace(views[1], t=views[0].t)     # a shared time slot
    jit = tuple(float(x) for x in rng.uniform(0, 0.3, 3)) if rng.random() < 0.3 else (0.0, 0.0, 0.0)
    return scene, views, jit


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_parity(seed):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    scene, views, jit = _case(seed)
    a, b = s3r.Context(0), s3r.Context(0)
    try:
        a.set_debug(True)
        for c in (a, b):
            c.set_lod_jitter(*jit)
        tabs = list(s3r.view_tables(a, views))
        dsa = s3r.DeviceScene.from_numpy(scene)
        oa = s3r.alloc_outputs(views, n_visible=scene.n)
        a.render_batch(dsa, views, tabs, oa)
        torch.cuda.synchronize()
        assert a.check() in (s3r.S3R_OK, s3r.S3R_EINSTANCE)
        for vi, v in enumerate(views):
            vj = dataclasses.replace(v, lod_jitter=jit)
            compare_dump(gpu_dump(a, vj, vi, oa[vi]), oracle.render_view(scene, vj, "f32"))
        b.set_capacity(a.capacity_from_last(1.0))
        dsb = s3r.DeviceScene.from_numpy(scene)
        ob = s3r.alloc_outputs(views, n_visible=scene.n)
        b.render_batch(dsb, views, tabs, ob)
        torch.cuda.synchronize()
        assert b.check() == 0
        for x, y in zip(oa, ob):
            for k in x:
                assert torch.equal(x[k], y[k]), k
        assert torch.equal(dsa.life, dsb.life)
    finally:
        a.close()
        b.close()
