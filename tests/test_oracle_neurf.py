"""Pins of the oracle's NeurF colour query (NEXT-4; Eq.7 rows 5-6, P:195-199;
architecture = DESIGN.md reading R22).

Pinned against torch (bf16 conversion, fp64 reference MLP through
torch.nn.functional), the math module (features of a hand-placed Gaussian),
and closed forms (time-embedding interpolation at grid points and midpoints;
the object-frame viewing direction as the unit vector from the camera centre
expressed in the object frame).
"""
import math

import numpy as np
import torch

from oracle import neurf
from paper_2503_08217_b200 import scenegen as sg
from helpers import make_scene, make_view


def test_bf16_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.normal(0, 3, 20000), rng.normal(0, 1e-3, 2000),
                        np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -(1.0 + 2 ** -8), 0.0, -0.0])])
    x = x.astype(np.float32)
    # exact ties of the bf16 grid round to even
    ties = (np.arange(1, 200, dtype=np.uint32) << 16 | 0x8000).view(np.float32)
    x = np.concatenate([x, ties, -ties])
    want = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(neurf.bf16(x).view(np.uint32), want.view(np.uint32))


def test_time_embedding():
    tab = np.arange(15, dtype=np.float64).reshape(5, 3)      # grid t = -1, -0.5, 0, 0.5, 1
    for j, t in enumerate([-1.0, -0.5, 0.0, 0.5, 1.0]):
        assert np.allclose(neurf.time_embedding(t, tab), tab[j], atol=1e-12)
    assert np.allclose(neurf.time_embedding(0.25, tab), 0.5 * (tab[2] + tab[3]), atol=1e-12)
    assert np.allclose(neurf.time_embedding(-1.0, tab), tab[0])
    assert np.allclose(neurf.time_embedding(1.0, tab), tab[4])


def test_features_hand_example():
    """Static Gaussian at (10, 20, 30) m seen by an identity camera, S = 100 m,
    D = 50 m: every feature from the math module."""
    mu = np.array([[10.0, 20.0, 30.0]])
    R = np.eye(3)[None]
    emb = np.arange(8) * 0.1
    cls = np.zeros((1, 4))
    f = neurf.features(mu, mu.copy(), R, emb, cls, 100.0, 50.0)[0]
    m = [0.1, 0.2, 0.3]
    assert np.allclose(f[0:3], m)
    for l in range(4):
        for a in range(3):
            assert math.isclose(f[3 + 6 * l + 2 * a], math.sin(2 ** l * math.pi * m[a]), abs_tol=1e-12)
            assert math.isclose(f[4 + 6 * l + 2 * a], math.cos(2 ** l * math.pi * m[a]), abs_tol=1e-12)
    assert math.isclose(f[27], 0.6)
    nrm = math.sqrt(10 ** 2 + 20 ** 2 + 30 ** 2)
    assert np.allclose(f[28:31], [10 / nrm, 20 / nrm, 30 / nrm])
    assert np.allclose(f[31:39], emb) and np.all(f[39:] == 0)
    # far away: normalize(d) saturates at 1
    f2 = neurf.features(mu * 10, mu * 10, R, emb, cls, 100.0, 50.0)[0]
    assert f2[27] == 1.0


def test_object_frame_direction():
    """dir = R^T p / |p| is the unit vector from the camera centre to mu, in
    the Gaussian's own frame (camera centre c = -R^T t there)."""
    scene, views = sg.make_random_dynamic(7, 50, 3, 40, 64, 48, 2)
    v = views[1]
    import oracle
    tab = oracle.compose(v).reshape(-1, 3, 4).astype(np.float64)
    gs = np.nonzero(scene.instance_ids > 0)[0][:30]
    for g in gs:
        M = tab[scene.instance_ids[g]]
        R, t = M[:, :3], M[:, 3]
        mu = scene.means_opacity[g, :3].astype(np.float64)
        p = R @ mu + t
        f = neurf.features(mu[None], p[None], R[None], np.zeros(8), np.zeros((1, 4)), 100.0, 50.0)
        c = -R.T @ t
        want = (mu - c) / np.linalg.norm(mu - c)
        assert np.allclose(f[0, 28:31], want, atol=1e-9)


def test_mlp_matches_torch_reference():
    rng = np.random.default_rng(3)
    prm = neurf.random_params(rng, 5)
    f = rng.normal(0, 1, (257, 64))
    f[:, 43:] = 0
    dyn = rng.random(257) < 0.4
    got = neurf.mlp(f, dyn, prm)
    F = torch.nn.functional
    want = np.zeros((257, 3))
    xb = torch.from_numpy(neurf.bf16(f.astype(np.float32))).double()
    for net in (0, 1):
        W = [torch.from_numpy(neurf.bf16(prm[k][net])).double() for k in ("w1", "w2", "w3")]
        b = [torch.from_numpy(np.asarray(prm[k][net], np.float64)) for k in ("b1", "b2", "b3")]
        h = torch.relu(F.linear(xb, W[0], b[0])).float().bfloat16().double()
        h = torch.relu(F.linear(h, W[1], b[1])).float().bfloat16().double()
        c = torch.sigmoid(F.linear(h, W[2], b[2])).numpy()
        sel = dyn == bool(net)
        want[sel] = c[sel]
    assert np.allclose(got, want, rtol=0, atol=1e-12)
    assert np.all((got > 0) & (got < 1))
    # routing: the dynamic network's weights do not touch static colours
    prm2 = dict(prm, w2=prm["w2"].copy())
    prm2["w2"][1] *= -1
    got2 = neurf.mlp(f, dyn, prm2)
    assert np.array_equal(got2[~dyn], got[~dyn]) and not np.allclose(got2[dyn], got[dyn])
