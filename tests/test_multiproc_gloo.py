"""The N>1 host path on CPU: world_size 2 over gloo (127.0.0.1).

Views are sharded across ranks (contiguous blocks); each rank applies its
views' M_t to a private copy of the point life; one all-reduce MAX bracketed by
l_s negation merges them (parallel.merge_life).  The merged life, and the
committed visibility, must equal a single process applying every view
(Eq.5 is order-independent, so equality is bit-exact).  The per-rank masks come
from the CPU oracle here (no GPU in this suite); the CUDA flip kernel is
covered by the gpu tests.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2503_08217_b200 import parallel
from paper_2503_08217_b200 import scenegen as sg


def _scene():
    scene, views = sg.make_random_dynamic(41, 1500, 3, 80, 96, 64, 7, fresh=True)
    for i, v in enumerate(views):
        v.t = float(np.float32(-1.0 + 2.0 * i / (len(views) - 1)))
    return scene, views


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scene, views = _scene()
        mine = parallel.shard_views(views, rank, world)
        for v in mine:
            o = oracle.render_view(scene, v, pairs=False, image=False)
            oracle.update_life(scene, o["visible"], v.t)
        life = torch.from_numpy(scene.life)

        def flip(t):
            t[:, 0].neg_()

        parallel.merge_life(life, flip)
        np.save(os.path.join(out_dir, f"life_{rank}.npy"), life.numpy().copy())
        oracle.commit_visibility(scene, 0.1)
        np.save(os.path.join(out_dir, f"vis_{rank}.npy"), scene.visibility)
    finally:
        dist.destroy_process_group()


def test_shard_bounds_partition():
    for n in (0, 1, 7, 64, 65):
        for w in (1, 2, 3, 8):
            seen = []
            for r in range(w):
                lo, hi = parallel.shard_bounds(n, r, w)
                seen.extend(range(lo, hi))
                assert hi - lo in (n // w, n // w + 1)
            assert seen == list(range(n))


def test_world2_life_merge_matches_single_process(tmp_path):
    world = 2
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    scene, views = _scene()
    for v in views:
        o = oracle.render_view(scene, v, pairs=False, image=False)
        oracle.update_life(scene, o["visible"], v.t)
    want_life = scene.life.copy()
    oracle.commit_visibility(scene, 0.1)
    for r in range(world):
        got = np.load(tmp_path / f"life_{r}.npy")
        assert np.array_equal(got, want_life)
        assert np.array_equal(np.load(tmp_path / f"vis_{r}.npy"), scene.visibility)
    assert (want_life[:, 0] <= want_life[:, 1]).sum() > 100     # observed Gaussians exist


def _grad_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scene, views = _scene()
        g = np.zeros((scene.n, 16))
        for v in parallel.shard_views(views, rank, world):
            cot = np.random.default_rng(int(1000 * (v.t + 2))).standard_normal(
                (v.height, v.width, 3))
            oracle.backward(scene, v, cot, grads=g)
        grads = {"means_opacity": torch.from_numpy(g[:, 0:4].copy()),
                 "colors": torch.from_numpy(g[:, 12:16].copy()),
                 "table": torch.full((2, 12), float(rank))}
        parallel.allreduce_grads(grads)
        np.save(os.path.join(out_dir, f"g_{rank}.npy"),
                np.concatenate([grads["means_opacity"].numpy(), grads["colors"].numpy()], 1))
        np.save(os.path.join(out_dir, f"t_{rank}.npy"), grads["table"].numpy())
    finally:
        dist.destroy_process_group()


def test_world2_gradient_allreduce_matches_single_process(tmp_path):
    """Config 5 sharded over 2 ranks: after parallel.allreduce_grads every rank
    holds the gradient of the whole batch (the single-process sum, to fp64
    rounding); the per-view pose gradient stays rank-local."""
    world = 2
    port = _free_port()
    mp.spawn(_grad_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    scene, views = _scene()
    g = np.zeros((scene.n, 16))
    for v in views:
        cot = np.random.default_rng(int(1000 * (v.t + 2))).standard_normal((v.height, v.width, 3))
        oracle.backward(scene, v, cot, grads=g)
    want = np.concatenate([g[:, 0:4], g[:, 12:16]], 1)
    assert np.abs(want).max() > 0
    for r in range(world):
        got = np.load(tmp_path / f"g_{r}.npy")
        assert np.allclose(got, want, rtol=1e-12, atol=1e-12 * np.abs(want).max())
        assert np.all(np.load(tmp_path / f"t_{r}.npy") == r)


def test_bench_view_shards():
    """bench.py's split of a step's views over ranks (BASELINE C3: 64 views over
    1/2/4/8 GPUs; C4: 256 at 32 per rank): contiguous, complete, balanced."""
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for n, g in ((64, 1), (64, 2), (64, 4), (64, 8), (256, 8), (100, 8), (7, 3)):
        shards, tot = bench.view_shards(n, g, "strong")
        assert tot == n and len(shards) == g
        assert [o for o, _ in shards] == list(np.cumsum([0] + [c for _, c in shards[:-1]]))
        assert sum(c for _, c in shards) == n
        assert max(c for _, c in shards) - min(c for _, c in shards) <= 1
    assert bench.view_shards(256, 8, "strong")[0][3] == (96, 32)
    shards, tot = bench.view_shards(64, 4, "weak", 16)
    assert tot == 64 and shards == [(0, 16), (16, 16), (32, 16), (48, 16)]
