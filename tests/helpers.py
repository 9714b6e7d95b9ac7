"""Test-side construction of tiny hand-made scenes (inputs only)."""
import numpy as np

from paper_2503_08217_b200.scenegen import Scene, View


def make_scene(points, sigmas, quats=None, opacity=None, rgb=None, ids=None, vis=None,
               num_instances=None):
    points = np.asarray(points, np.float64).reshape(-1, 3)
    n = points.shape[0]
    sigmas = np.broadcast_to(np.asarray(sigmas, np.float64), (n, 3))
    quats = np.tile([1.0, 0, 0, 0], (n, 1)) if quats is None else np.broadcast_to(quats, (n, 4))
    opacity = np.full(n, 0.5) if opacity is None else np.broadcast_to(opacity, (n,))
    rgb = np.full((n, 3), 0.5) if rgb is None else np.broadcast_to(rgb, (n, 3))
    ids = np.zeros(n, np.int32) if ids is None else np.asarray(ids, np.int32)
    vis = np.tile([-1.0, 1.0], (n, 1)) if vis is None else np.broadcast_to(vis, (n, 2))
    K1 = (int(ids.max()) + 1 if n else 1) if num_instances is None else num_instances
    return Scene(
        name="hand",
        means_opacity=np.concatenate([points, np.asarray(opacity)[:, None]], 1).astype(np.float32),
        scales=np.concatenate([sigmas, np.zeros((n, 1))], 1).astype(np.float32),
        rotations=np.ascontiguousarray(quats, np.float32),
        colors=np.concatenate([rgb, np.zeros((n, 1))], 1).astype(np.float32),
        instance_ids=ids,
        visibility=np.ascontiguousarray(vis, np.float32),
        life=np.tile(np.array([[1.0, -1.0]], np.float32), (n, 1)),
        num_instances=K1,
    )


def make_view(f, c, w, h, t=0.0, w2c=None, i2g=None, lod=(0.0, 0.5, 10.0), seed=0, fy=None, cy=None):
    w2c = np.concatenate([np.eye(3), np.zeros((3, 1))], 1) if w2c is None else w2c
    i2g = np.zeros((0, 3, 4)) if i2g is None else i2g
    return View(t=t, width=w, height=h, fx=f, fy=f if fy is None else fy, cx=c,
                cy=c if cy is None else cy, w2c=np.asarray(w2c, np.float32),
                i2g=np.asarray(i2g, np.float32), lod_r=lod[0], lod_pmax=lod[1], lod_D=lod[2],
                lod_seed=seed)


def quat_mul(a, b):
    """Hamilton product (w,x,y,z) — used by tests to build the conventional pipeline."""
    w1, x1, y1, z1 = a
    w2, x2, y2, z2 = b
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
                     w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
                     w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])
