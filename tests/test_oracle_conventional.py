"""Pins of the oracle's conventional pipeline C0 (NEXT-2): the
per-frame local-to-global transformation of the dynamic Gaussians (P:20, P:45,
P:150; Fig.1a) that the streamlined stage removes.

Pinned against scipy's rotation algebra (an independent implementation), the
quaternion norm identity, and the theorem the paper rests on: the conventional
render of the world-transformed scene equals the streamlined render with
instance-specific cameras (S:679 acceptance 1), here through the oracle's own
C0 rather than a test-side transform.
"""
import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle
from helpers import make_scene, make_view
from paper_2503_08217_b200 import scenegen as sg


def _wxyz(rot: Rotation) -> np.ndarray:
    q = rot.as_quat()                  # scipy: (x, y, z, w)
    return np.array([q[3], q[0], q[1], q[2]])


def _same_rotation(q1, q2, tol):
    """q and -q are the same rotation."""
    return min(np.abs(q1 - q2).max(), np.abs(q1 + q2).max()) <= tol


# one rotation per Shepperd branch: trace > 0, then R00 / R11 / R22 largest
BRANCH_ROTS = [
    Rotation.from_rotvec([0.3, -0.2, 0.5]),
    Rotation.from_rotvec(np.array([1.0, 0.1, -0.05]) / np.linalg.norm([1.0, 0.1, -0.05]) * 3.0),
    Rotation.from_rotvec(np.array([0.1, 1.0, 0.05]) / np.linalg.norm([0.1, 1.0, 0.05]) * 3.0),
    Rotation.from_rotvec(np.array([-0.05, 0.1, 1.0]) / np.linalg.norm([-0.05, 0.1, 1.0]) * 3.0),
]


@pytest.mark.parametrize("k", range(4))
def test_quat_from_rot_branches(k):
    """quat(R) of each Shepperd branch reproduces scipy's quaternion (up to sign)."""
    rot = BRANCH_ROTS[k]
    R = rot.as_matrix()
    tr = np.trace(R)
    # the case really exercises branch k
    assert (tr > 0) == (k == 0)
    if k:
        assert int(np.argmax(np.diag(R))) == k - 1
    assert _same_rotation(oracle.quat_from_rot(R, "f64"), _wxyz(rot), 1e-14)
    assert _same_rotation(oracle.quat_from_rot(R, "f32").astype(np.float64), _wxyz(rot), 3e-7)


def test_quat_from_rot_random():
    for i in range(200):
        rot = Rotation.random(random_state=i)
        q = oracle.quat_from_rot(rot.as_matrix(), "f64")
        assert abs(np.linalg.norm(q) - 1) < 1e-14
        assert _same_rotation(q, _wxyz(rot), 1e-13)


def test_quat_mul_is_composition():
    """a (x) b is the rotation R_a R_b (scipy composition), |a (x) b| = |a| |b|."""
    rng = np.random.default_rng(3)
    for i in range(100):
        ra, rb = Rotation.random(random_state=2 * i), Rotation.random(random_state=2 * i + 1)
        s = rng.uniform(0.2, 3.0)            # an unnormalised second factor
        o = oracle.quat_mul(_wxyz(ra), s * _wxyz(rb), "f64")
        assert abs(np.linalg.norm(o) - s) < 1e-13 * s
        assert _same_rotation(o / s, _wxyz(ra * rb), 1e-13)
        o32 = oracle.quat_mul(_wxyz(ra), s * _wxyz(rb), "f32").astype(np.float64)
        assert _same_rotation(o32 / s, _wxyz(ra * rb), 4e-7)


def test_world_transform_matches_scipy():
    """C0 on a random dynamic scene: mu_w = R mu + t and R(q_w) = R R(q), per
    instance; static and out-of-range-id Gaussians are copied."""
    scene, views = sg.make_random_dynamic(5, 300, 4, 50, 64, 48, 2)
    scene.instance_ids[7] = 99               # out of range: copied
    v = views[1]
    w = oracle.world_scene(scene, v.i2g, "f64")
    mo, q, ids = scene.means_opacity.astype(np.float64), scene.rotations.astype(np.float64), \
        scene.instance_ids
    assert np.array_equal(w.instance_ids[ids == 0], ids[ids == 0])
    assert w.instance_ids[7] == 99 and np.array_equal(w.means_opacity[7], scene.means_opacity[7])
    assert np.all(w.visibility == np.array([-1.0, 1.0], np.float32))
    for g in range(scene.n):
        i = ids[g]
        if i == 0 or i >= scene.num_instances:
            assert np.array_equal(w.means_opacity[g], scene.means_opacity[g])
            assert np.array_equal(w.rotations[g], scene.rotations[g])
            continue
        P = v.i2g[i - 1].astype(np.float64)
        want_mu = P[:, :3] @ mo[g, :3] + P[:, 3]
        assert np.abs(w.means_opacity[g, :3] - want_mu).max() <= 2e-6 * max(1, np.abs(want_mu).max())
        assert w.means_opacity[g, 3] == scene.means_opacity[g, 3]
        qg = q[g] / np.linalg.norm(q[g])
        Rw = P[:, :3] @ Rotation.from_quat([qg[1], qg[2], qg[3], qg[0]]).as_matrix()
        qw = w.rotations[g].astype(np.float64)
        qw /= np.linalg.norm(qw)
        got = Rotation.from_quat([qw[1], qw[2], qw[3], qw[0]]).as_matrix()
        assert np.abs(got - Rw).max() < 2e-6


@pytest.mark.parametrize("seed", [41, 42])
def test_conventional_equals_streamlined(seed):
    """The paper's premise: with fresh intervals and no LOD the
    conventional pipeline (oracle C0 + projection through W_t of all Gaussians)
    renders the streamlined image.  fp64: the only difference is the fp32
    storage of the world scene (~6e-8 relative)."""
    scene, views = sg.make_random_dynamic(seed, 400, 3, 60, 96, 64, 3, fresh=True)
    for v in views:
        a = oracle.render_view(scene, v, "f64")
        b = oracle.render_view_conventional(scene, v, "f64")
        assert np.array_equal(a["flags"] & 2, b["flags"] & 2)      # same visible set M_t
        assert np.abs(a["rgb"] - b["rgb"]).max() < 1e-5
        assert a["stats"]["n_rendered"] > 20
        # the conventional pipeline projects every Gaussian (no temporal filter)
        assert b["stats"]["n_temporal"] == scene.n


def test_conventional_projects_temporally_invisible():
    """Without fresh intervals the conventional pipeline still projects every
    Gaussian, so its visible set contains the streamlined one."""
    scene, views = sg.make_random_dynamic(43, 400, 3, 60, 96, 64, 3)
    v = views[0]
    a = oracle.render_view(scene, dataclass_replace(v, lod_r=0.0), "f32")
    b = oracle.render_view_conventional(scene, v, "f32")
    va, vb = (a["flags"] & 2) != 0, (b["flags"] & 2) != 0
    assert np.all(vb[va]) and vb.sum() > va.sum()
    assert b["stats"]["n_lod_small"] == 0


def dataclass_replace(v, **kw):
    import dataclasses
    return dataclasses.replace(v, **kw)
