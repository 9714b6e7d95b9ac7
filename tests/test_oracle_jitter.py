"""Pins of the oracle's LOD noisy offset (NEXT-3; Eq.7 row 4):
mu <- mu + [dx, dy, dz] normalize(d) N(0,1) on the kept small Gaussians, with
reading R10 normalize(d) = min(1, d / D) and the R-ARITH Box-Muller sampler
(so_lod_normal3).

Pinned against libm / numpy (log2, sin, cos accuracy), scipy's normal
distribution (Kolmogorov-Smirnov, moments, independence), and the definition
itself: a jittered render equals the plain render of the scene whose small
Gaussian was moved by hand to mu + s n.
"""
import dataclasses
import math

import numpy as np
import pytest
from scipy import stats

import oracle
from helpers import make_scene, make_view


def test_log2_accuracy():
    xs = np.concatenate([2.0 ** -np.arange(0, 25), np.linspace(2 ** -24, 1, 20001)[1:],
                         np.float32(np.random.default_rng(0).random(5000))])
    xs = xs[xs > 0].astype(np.float32)
    for x in xs:
        want = math.log2(float(x))
        got = oracle.log2_32(float(x))
        assert abs(got - want) <= 2.5e-7 * max(1.0, abs(want)), (x, got, want)
    # exact at powers of two
    for e in range(0, 25):
        assert oracle.log2_32(2.0 ** -e) == -e


def test_sincos_turn_accuracy():
    rng = np.random.default_rng(1)
    us = np.concatenate([np.arange(0, 1, 1 / 64), rng.integers(0, 1 << 24, 20000) / 2.0 ** 24])
    for u in us:
        s, c = oracle.sincos_turn(float(u))
        assert abs(s - math.sin(2 * math.pi * u)) <= 4e-7, u
        assert abs(c - math.cos(2 * math.pi * u)) <= 4e-7, u
    assert oracle.sincos_turn(0.0) == (0.0, 1.0)
    assert oracle.sincos_turn(0.25) == (1.0, -0.0)
    assert oracle.sincos_turn(0.5) == (-0.0, -1.0)
    assert oracle.sincos_turn(0.75) == (-1.0, 0.0)


def test_normals_are_standard_normal():
    n = 60000
    z = np.stack([oracle.lod_normal3(1234, g) for g in range(n)]).astype(np.float64)
    for a in range(3):
        x = z[:, a]
        assert abs(x.mean()) < 4 / math.sqrt(n)
        assert abs(x.var() - 1) < 4 * math.sqrt(2 / n)
        assert stats.kstest(x, "norm").pvalue > 1e-3
    c = np.corrcoef(z.T)
    assert np.all(np.abs(c[np.triu_indices(3, 1)]) < 0.02)
    # independent of the Bernoulli draw (so_lod_uniform) of the same Gaussian
    u = np.array([oracle.lod_uniform(1234, g) for g in range(n)])
    assert abs(np.corrcoef(u, z[:, 0])[0, 1]) < 0.02
    # deterministic, seed-dependent
    assert np.array_equal(oracle.lod_normal3(1234, 77), oracle.lod_normal3(1234, 77))
    assert not np.array_equal(oracle.lod_normal3(1234, 77), oracle.lod_normal3(1235, 77))


def _small_far_scene():
    """A few small distant Gaussians (LOD-small at r = 4 px) in front of an
    identity camera, plus large near ones (never small)."""
    rng = np.random.default_rng(4)
    far = np.stack([rng.uniform(-20, 20, 40), rng.uniform(-12, 12, 40), rng.uniform(60, 90, 40)], 1)
    near = np.stack([rng.uniform(-2, 2, 20), rng.uniform(-1.5, 1.5, 20), rng.uniform(4, 8, 20)], 1)
    pts = np.concatenate([far, near]).astype(np.float32).astype(np.float64)
    sig = np.concatenate([np.full((40, 3), 0.02), np.full((20, 3), 0.15)])
    return make_scene(pts, sig, opacity=rng.uniform(0.3, 0.9, 60), rgb=rng.random((60, 3)))


def test_jitter_zero_is_no_jitter():
    s = _small_far_scene()
    v = make_view(200.0, 100.0, 200, 150, lod=(4.0, 0.3, 50.0), seed=9)
    a = oracle.render_view(s, v, "f32")
    b = oracle.render_view(s, dataclasses.replace(v, lod_jitter=(0.0, 0.0, 0.0)), "f32")
    assert np.array_equal(a["rgb"], b["rgb"]) and np.array_equal(a["flags"], b["flags"])
    assert not np.any(a["flags"] & oracle.F_JITTERED)


def test_jitter_is_the_definition():
    """The jittered render equals the plain render of the scene in which every
    jittered Gaussian was moved to fma(dx_a min(1, d/D), n_a, mu_a) by hand;
    M_t and the LOD decisions are those of the unmoved mean."""
    s = _small_far_scene()
    jit = (0.8, 0.5, 1.5)
    v = make_view(200.0, 100.0, 200, 150, lod=(4.0, 0.3, 50.0), seed=9)
    vj = dataclasses.replace(v, lod_jitter=jit)
    a = oracle.render_view(s, vj, "f32")
    base = oracle.render_view(s, v, "f32")
    fl = a["flags"]
    jittered = (fl & oracle.F_JITTERED) != 0
    assert jittered.sum() >= 5
    assert np.array_equal(jittered, (base["flags"] & (oracle.F_SMALL | oracle.F_DROPPED))
                          == oracle.F_SMALL)
    # M_t, the small set and the drop set do not move
    for f in (oracle.F_VISIBLE, oracle.F_SMALL, oracle.F_DROPPED):
        assert np.array_equal(fl & f, base["flags"] & f)
    # the hand-moved scene
    moved = s.copy()
    for g in np.nonzero(jittered)[0]:
        d = np.float32(base["keys"][g, 2])
        nd = min(np.float32(1.0), np.float32(d / np.float32(v.lod_D)))
        n = oracle.lod_normal3(v.lod_seed, int(g))
        for ax in range(3):
            sa = np.float32(np.float32(jit[ax]) * nd)
            moved.means_opacity[g, ax] = np.float32(float(sa) * float(n[ax])
                                                    + float(s.means_opacity[g, ax]))
    # render the moved scene without LOD (nothing re-dropped or re-jittered),
    # the Gaussians the jittered render dropped removed by their interval
    moved.visibility[(base["flags"] & oracle.F_DROPPED) != 0] = (2.0, 3.0)
    b = oracle.render_view(moved, dataclasses.replace(v, lod_r=0.0), "f32")
    keep = (fl & oracle.F_RENDERED) != 0
    assert np.array_equal(keep, (b["flags"] & oracle.F_RENDERED) != 0)
    assert np.array_equal(a["rgb"], b["rgb"]) and np.array_equal(a["depth"], b["depth"])
    assert np.array_equal(a["pair_gauss"], b["pair_gauss"])
    assert not np.array_equal(a["rgb"], base["rgb"])
