"""Seeded synthetic street scenes — the INPUT generator shared by tests and bench.

This module creates inputs only.  It holds none of the method's arithmetic
(no projection, no filtering, no LOD, no blending, no pose composition): it
draws Gaussians, object trajectories and camera rigs with the shapes of the
paper's workloads (BASELINE.json configs) and returns plain
numpy arrays.  Both the CPU oracle (oracle/) and the CUDA path
(paper_2503_08217_b200/s3r.py) consume them.

World frame: x forward along the street, y left, z up.  Cameras use the
OpenCV convention (x right, y down, z forward).  All matrices are 3x4
row-major [R|t]: ``w2c`` maps world -> camera, ``i2g[k]`` maps object k's
local frame -> world (W_{t,i2g} of P:159).

Temporal-visibility intervals are synthetic "committed" intervals (what Eq.6
would give after a sweep): a static Gaussian at street position x_g is visible
while the ego camera is within [x_g - back, x_g + front]; a dynamic Gaussian
inherits its object's lifetime intersected with the same window.  Time is the
frame index mapped to [-1, 1].
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Tuple

import numpy as np

TILE = 16


@dataclasses.dataclass
class Scene:
    name: str
    means_opacity: np.ndarray   # (N,4) f32: x,y,z (local frame of instance), opacity
    scales: np.ndarray          # (N,4) f32: sigma x,y,z (linear metres), pad 0
    rotations: np.ndarray       # (N,4) f32: quaternion w,x,y,z
    colors: np.ndarray          # (N,4) f32: r,g,b in [0,1], pad 0
    instance_ids: np.ndarray    # (N,)  i32: 0 static, 1..K objects
    visibility: np.ndarray      # (N,2) f32: v_s, v_e
    life: np.ndarray            # (N,2) f32: l_s, l_e (initial (1,-1))
    num_instances: int          # K+1

    @property
    def n(self) -> int:
        return int(self.means_opacity.shape[0])

    def copy(self) -> "Scene":
        return dataclasses.replace(self, **{f.name: np.array(getattr(self, f.name))
                                            for f in dataclasses.fields(self)
                                            if isinstance(getattr(self, f.name), np.ndarray)})


@dataclasses.dataclass
class View:
    t: float
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    w2c: np.ndarray             # (3,4) f32 world -> camera (W_t)
    i2g: np.ndarray             # (K,3,4) f32 object local -> world (W_{t,i2g})
    lod_r: float = 0.0
    lod_pmax: float = 0.5
    lod_D: float = 50.0
    lod_seed: int = 0
    near: float = 0.01
    lod_jitter: Tuple[float, float, float] = (0.0, 0.0, 0.0)   # Eq.7 row 4 [dx, dy, dz]
    frame: int = 0
    cam: int = 0


@dataclasses.dataclass
class Config:
    name: str
    n_static: int
    n_objects: int
    per_object: int
    width: int
    height: int
    focal: float
    yaws_deg: Tuple[float, ...]
    length_m: float
    frames: int
    window_back: float
    window_front: float
    lod: Tuple[float, float, float]
    n_views: int
    seed: int
    cam_height: float = 1.6


CONFIGS = {
    # C2 small street: 150k + 10x5k, 1 forward camera 960x640, ~40 % temporal pass
    # (window -38/+108 m: the realised mean pass over the 100 views is 40.0 %;
    # the survey's -20/+80 m gives 28.5 % once the street's ends clip the window)
    "street": Config("street", 150_000, 10, 5_000, 960, 640, 600.0, (0.0,), 250.0, 100,
                     38.0, 108.0, (4.0, 0.5, 50.0), 100, 2),
    # C3 Argoverse2-shaped: 1.7M + 30x10k, 7 ring cameras 1550x2048, ~25 % pass
    "av2": Config("av2", 1_700_000, 30, 10_000, 1550, 2048, 1700.0,
                  (0.0, 45.0, -45.0, 99.0, -99.0, 153.0, -153.0), 400.0, 150,
                  50.0, 50.0, (4.0, 0.5, 50.0), 64, 3),
    # C4 large drive: 9.365M + 127x5k, same rig, 2 km, ~10 % pass
    "drive": Config("drive", 9_365_000, 127, 5_000, 1550, 2048, 1700.0,
                    (0.0, 45.0, -45.0, 99.0, -99.0, 153.0, -153.0), 2000.0, 1000,
                    100.0, 100.0, (4.0, 0.5, 50.0), 256, 4),
}


# ----------------------------------------------------------------------------
# small helpers (input construction only)
# ----------------------------------------------------------------------------

def frame_time(frame: int, frames: int) -> float:
    """Frame index -> time in [-1, 1] (input labelling)."""
    if frames <= 1:
        return 0.0
    return -1.0 + 2.0 * frame / (frames - 1)


def _quat_axis(axis: np.ndarray, angle: np.ndarray) -> np.ndarray:
    half = 0.5 * angle
    s = np.sin(half)
    q = np.zeros(angle.shape + (4,), np.float64)
    q[..., 0] = np.cos(half)
    q[..., 1:] = axis * s[..., None]
    return q


def _random_quat(rng, n) -> np.ndarray:
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q


def _lognormal_sigma(rng, n, median=0.08, lnsd=0.6, lo=0.005, hi=2.0) -> np.ndarray:
    s = np.exp(np.log(median) + lnsd * rng.standard_normal(n))
    return np.clip(s, lo, hi)


def yaw_matrix(yaw: float) -> np.ndarray:
    c, s = np.cos(yaw), np.sin(yaw)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def camera_w2c(position: np.ndarray, yaw: float) -> np.ndarray:
    """World->camera 3x4 for a level camera at `position` looking along yaw."""
    fwd = np.array([np.cos(yaw), np.sin(yaw), 0.0])
    right = np.array([np.sin(yaw), -np.cos(yaw), 0.0])
    down = np.array([0.0, 0.0, -1.0])
    R = np.stack([right, down, fwd])
    t = -R @ position
    return np.concatenate([R, t[:, None]], axis=1)


def _interval_to_t(lo_frame: np.ndarray, hi_frame: np.ndarray, frames: int):
    lo = np.clip(-1.0 + 2.0 * lo_frame / max(frames - 1, 1), -1.0, 1.0)
    hi = np.clip(-1.0 + 2.0 * hi_frame / max(frames - 1, 1), -1.0, 1.0)
    return lo, hi


# ----------------------------------------------------------------------------
# street scenes (C2, C3, C4)
# ----------------------------------------------------------------------------

def make_street_scene(cfg: Config, scale: float = 1.0, seed: Optional[int] = None):
    """Build the scene + object trajectories for a street config.

    scale < 1 shrinks the Gaussian counts (parity tests); geometry is unchanged.
    Returns (Scene, traj) where traj = (x0[K], u[K], lane_y[K], yaw[K], f0[K], f1[K]).
    """
    rng = np.random.default_rng(cfg.seed if seed is None else seed)
    L, F = cfg.length_m, cfg.frames
    n_static = max(1, int(round(cfg.n_static * scale)))
    per_obj = max(1, int(round(cfg.per_object * scale)))
    K = cfg.n_objects

    n_ground = int(n_static * 0.40)
    n_far = int(n_static * 0.15)
    n_facade = n_static - n_ground - n_far
    xs_lo, xs_hi = 0.0, L

    mu, sig, quat = [], [], []
    # ground: z = 0, |y| <= 12, flattened along z, random yaw
    x = rng.uniform(xs_lo, xs_hi, n_ground)
    y = rng.uniform(-12.0, 12.0, n_ground)
    mu.append(np.stack([x, y, np.zeros_like(x)], 1))
    s = _lognormal_sigma(rng, n_ground)
    sig.append(np.stack([s * rng.uniform(0.6, 1.4, n_ground), s, 0.1 * s], 1))
    quat.append(_quat_axis(np.array([0.0, 0.0, 1.0]), rng.uniform(0, 2 * np.pi, n_ground)))
    # facades: 10 <= |y| <= 14, 0 <= z <= 20, flattened along y
    x = rng.uniform(xs_lo, xs_hi, n_facade)
    side = np.where(rng.random(n_facade) < 0.5, -1.0, 1.0)
    y = side * rng.uniform(10.0, 14.0, n_facade)
    z = 20.0 * rng.random(n_facade) ** 1.5
    mu.append(np.stack([x, y, z], 1))
    s = _lognormal_sigma(rng, n_facade)
    sig.append(np.stack([s, 0.1 * s, s * rng.uniform(0.6, 1.4, n_facade)], 1))
    quat.append(_quat_axis(np.array([0.0, 1.0, 0.0]), rng.uniform(0, 2 * np.pi, n_facade)))
    # far shell: 100-300 m from a point of the trajectory, for LOD
    xc = rng.uniform(0.0, L, n_far)
    ang = rng.uniform(0, 2 * np.pi, n_far)
    rad = rng.uniform(100.0, 300.0, n_far)
    z = rng.uniform(0.0, 60.0, n_far)
    mu.append(np.stack([xc + rad * np.cos(ang), rad * np.sin(ang), z], 1))
    sig.append(np.stack([_lognormal_sigma(rng, n_far, median=0.5, hi=4.0)] * 3, 1)
               * rng.uniform(0.5, 1.5, (n_far, 3)))
    quat.append(_random_quat(rng, n_far))

    mu = np.concatenate(mu)
    sig = np.concatenate(sig)
    quat = np.concatenate(quat)
    # window rule for static content: visible while x_cam in [x_g - front, x_g + back]
    # (ego at frame f sits at x = L f / (F-1))
    xg = mu[:, 0] if n_far == 0 else np.concatenate([mu[: n_ground + n_facade, 0], xc])
    fpm = (F - 1) / L
    v_lo, v_hi = _interval_to_t((xg - cfg.window_front) * fpm, (xg + cfg.window_back) * fpm, F)
    ids = np.zeros(n_static, np.int32)
    # storage order of the static Gaussians: along the street (the order in
    # which LiDAR-initialised points are acquired along the trajectory), so the
    # Gaussians one time t keeps are a few contiguous runs of memory
    order = np.argsort(xg, kind="stable")
    mu, sig, quat, v_lo, v_hi = mu[order], sig[order], quat[order], v_lo[order], v_hi[order]

    # dynamic objects: car boxes 4.5 x 1.9 x 1.6 m in lanes y = +-3.5
    x0 = rng.uniform(-20.0, L + 20.0, K)
    lane = np.where(rng.random(K) < 0.5, -3.5, 3.5)
    u = rng.uniform(0.5, 3.0, K) * np.where(lane > 0, -1.0, 1.0)   # m/frame
    yaw = np.where(u < 0, np.pi, 0.0)
    f0 = rng.integers(0, max(1, F // 2), K).astype(np.float64)
    f1 = np.minimum(F - 1, f0 + rng.integers(max(1, F // 4), F, K)).astype(np.float64)
    dmu, dsig, dq, did, dlo, dhi = [], [], [], [], [], []
    frames = np.arange(F, dtype=np.float64)
    for k in range(K):
        # points on the box surface, local frame centred at the ground contact
        face = rng.integers(0, 3, per_obj)
        p = rng.uniform(-0.5, 0.5, (per_obj, 3)) * np.array([4.5, 1.9, 1.6])
        sgn = np.where(rng.random(per_obj) < 0.5, -0.5, 0.5)
        dims = np.array([4.5, 1.9, 1.6])
        p[np.arange(per_obj), face] = sgn * dims[face]
        p[:, 2] += 0.8
        dmu.append(p)
        s = _lognormal_sigma(rng, per_obj, median=0.05, hi=0.5)
        dsig.append(np.stack([s] * 3, 1) * rng.uniform(0.5, 1.5, (per_obj, 3)))
        dq.append(_random_quat(rng, per_obj))
        did.append(np.full(per_obj, k + 1, np.int32))
        # frames in which the car is alive and inside the ego window
        xcar = x0[k] + u[k] * frames
        xcam = L * frames / max(F - 1, 1)
        inside = (xcar >= xcam - cfg.window_back) & (xcar <= xcam + cfg.window_front)
        inside &= (frames >= f0[k]) & (frames <= f1[k])
        if inside.any():
            lo_f, hi_f = frames[inside][0], frames[inside][-1]
            lo, hi = _interval_to_t(np.array([lo_f]), np.array([hi_f]), F)
            lo, hi = float(lo[0]), float(hi[0])
        else:       # never seen: an empty interval (v_s > v_e)
            lo, hi = 1.0, -1.0
        dlo.append(np.full(per_obj, lo))
        dhi.append(np.full(per_obj, hi))

    if K:
        mu = np.concatenate([mu] + dmu)
        sig = np.concatenate([sig] + dsig)
        quat = np.concatenate([quat] + dq)
        ids = np.concatenate([ids] + did)
        v_lo = np.concatenate([v_lo] + dlo)
        v_hi = np.concatenate([v_hi] + dhi)
    N = mu.shape[0]
    opacity = rng.uniform(0.05, 0.99, N)
    rgb = rng.random((N, 3))
    scene = Scene(
        name=cfg.name,
        means_opacity=np.concatenate([mu, opacity[:, None]], 1).astype(np.float32),
        scales=np.concatenate([sig, np.zeros((N, 1))], 1).astype(np.float32),
        rotations=quat.astype(np.float32),
        colors=np.concatenate([rgb, np.zeros((N, 1))], 1).astype(np.float32),
        instance_ids=ids.astype(np.int32),
        visibility=np.stack([v_lo, v_hi], 1).astype(np.float32),
        life=np.tile(np.array([[1.0, -1.0]], np.float32), (N, 1)),
        num_instances=K + 1,
    )
    return scene, (x0, u, lane, yaw, f0, f1)


def object_i2g(traj, frame: int) -> np.ndarray:
    """W_{t,i2g} for every object at `frame` (constant-velocity trajectories)."""
    x0, u, lane, yaw, _, _ = traj
    K = len(x0)
    out = np.zeros((K, 3, 4), np.float64)
    for k in range(K):
        out[k, :, :3] = yaw_matrix(yaw[k])
        out[k, :, 3] = [x0[k] + u[k] * frame, lane[k], 0.0]
    return out.astype(np.float32)


def make_views(cfg: Config, traj, n_views: Optional[int] = None, seed: Optional[int] = None,
               width: Optional[int] = None, height: Optional[int] = None,
               frames: Optional[List[int]] = None) -> List[View]:
    """Sample views from the (frame, camera) grid, sorted by (frame, camera)."""
    rng = np.random.default_rng((cfg.seed if seed is None else seed) + 7919)
    F, ncam = cfg.frames, len(cfg.yaws_deg)
    n_views = cfg.n_views if n_views is None else n_views
    W = cfg.width if width is None else width
    H = cfg.height if height is None else height
    f = cfg.focal * (W / cfg.width)
    if frames is not None:
        grid = [(fr, c) for fr in frames for c in range(ncam)][:n_views]
    else:
        total = F * ncam
        pick = rng.choice(total, size=min(n_views, total), replace=False) if n_views <= total \
            else rng.integers(0, total, n_views)
        grid = sorted((int(p) // ncam, int(p) % ncam) for p in pick)
    views = []
    for vi, (fr, c) in enumerate(grid):
        pos = np.array([cfg.length_m * fr / max(F - 1, 1), 0.0, cfg.cam_height])
        w2c = camera_w2c(pos, np.deg2rad(cfg.yaws_deg[c])).astype(np.float32)
        r, pmax, D = cfg.lod
        views.append(View(t=frame_time(fr, F), width=W, height=H, fx=f, fy=f,
                          cx=W / 2.0, cy=H / 2.0, w2c=w2c, i2g=object_i2g(traj, fr),
                          lod_r=r, lod_pmax=pmax, lod_D=D,
                          lod_seed=int(cfg.seed * 1_000_003 + fr * 17 + c) & ((1 << 64) - 1),
                          frame=fr, cam=c))
    return views


# ----------------------------------------------------------------------------
# C1 toy and tiny hand-made scenes
# ----------------------------------------------------------------------------

def make_toy(seed: int = 1, n: int = 1024, width: int = 64, height: int = 64,
             lod=(0.5, 0.5, 6.0)) -> Tuple[Scene, List[View]]:
    """C1: 1 static instance, n Gaussians in front of an identity camera, t = 0."""
    rng = np.random.default_rng(seed)
    z = rng.uniform(2.0, 10.0, n)
    x = rng.uniform(-0.55, 0.55, n) * z * (width / 64.0)
    y = rng.uniform(-0.55, 0.55, n) * z * (height / 64.0)
    s = np.exp(rng.uniform(np.log(0.003), np.log(0.2), (n, 3)))
    scene = Scene(
        name="toy",
        means_opacity=np.stack([x, y, z, rng.uniform(0.05, 0.99, n)], 1).astype(np.float32),
        scales=np.concatenate([s, np.zeros((n, 1))], 1).astype(np.float32),
        rotations=_random_quat(rng, n).astype(np.float32),
        colors=np.concatenate([rng.random((n, 3)), np.zeros((n, 1))], 1).astype(np.float32),
        instance_ids=np.zeros(n, np.int32),
        visibility=np.tile(np.array([[-1.0, 1.0]], np.float32), (n, 1)),
        life=np.tile(np.array([[1.0, -1.0]], np.float32), (n, 1)),
        num_instances=1,
    )
    w2c = np.concatenate([np.eye(3), np.zeros((3, 1))], 1).astype(np.float32)
    view = View(t=0.0, width=width, height=height, fx=64.0, fy=64.0, cx=width / 2.0,
                cy=height / 2.0, w2c=w2c, i2g=np.zeros((0, 3, 4), np.float32),
                lod_r=lod[0], lod_pmax=lod[1], lod_D=lod[2], lod_seed=12345)
    return scene, [view]


def make_random_dynamic(seed: int, n_static: int, n_objects: int, per_object: int,
                        width: int, height: int, n_views: int, lod=(0.0, 0.5, 10.0),
                        fresh: bool = False) -> Tuple[Scene, List[View]]:
    """A small random scene with moving objects and random temporal intervals,
    for parity tests (spans several tiles, ragged image edges)."""
    rng = np.random.default_rng(seed)
    K = n_objects
    N = n_static + K * per_object
    mu = np.empty((N, 3))
    z = rng.uniform(1.0, 30.0, n_static)
    mu[:n_static, 0] = rng.uniform(-0.8, 0.8, n_static) * z
    mu[:n_static, 1] = rng.uniform(-0.6, 0.6, n_static) * z
    mu[:n_static, 2] = z
    mu[n_static:] = rng.uniform(-1.5, 1.5, (K * per_object, 3))
    ids = np.zeros(N, np.int32)
    for k in range(K):
        ids[n_static + k * per_object: n_static + (k + 1) * per_object] = k + 1
    sig = np.exp(rng.uniform(np.log(0.01), np.log(0.6), (N, 3)))
    if fresh:
        vis = np.tile(np.array([[-1.0, 1.0]]), (N, 1))
    else:
        a = rng.uniform(-1.2, 1.0, N)
        b = a + rng.uniform(0.0, 1.5, N)
        vis = np.stack([a, b], 1)
    scene = Scene(
        name="random",
        means_opacity=np.concatenate([mu, rng.uniform(0.05, 0.99, (N, 1))], 1).astype(np.float32),
        scales=np.concatenate([sig, np.zeros((N, 1))], 1).astype(np.float32),
        rotations=_random_quat(rng, N).astype(np.float32),
        colors=np.concatenate([rng.random((N, 3)), np.zeros((N, 1))], 1).astype(np.float32),
        instance_ids=ids,
        visibility=vis.astype(np.float32),
        life=np.tile(np.array([[1.0, -1.0]], np.float32), (N, 1)),
        num_instances=K + 1,
    )
    views = []
    f = 0.9 * width
    for v in range(n_views):
        yaw = rng.uniform(-0.2, 0.2)
        pos = np.array([rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-2, 0)])
        # camera looking along +z of the world: identity-like rotation with a small yaw
        c, s_ = np.cos(yaw), np.sin(yaw)
        R = np.array([[c, 0, -s_], [0, 1, 0], [s_, 0, c]])
        w2c = np.concatenate([R, (-R @ pos)[:, None]], 1).astype(np.float32)
        i2g = np.zeros((K, 3, 4), np.float32)
        for k in range(K):
            a = rng.uniform(0, 2 * np.pi)
            Rk = np.array([[np.cos(a), 0, np.sin(a)], [0, 1, 0], [-np.sin(a), 0, np.cos(a)]])
            i2g[k, :, :3] = Rk
            i2g[k, :, 3] = [rng.uniform(-6, 6), rng.uniform(-3, 3), rng.uniform(4, 25)]
        views.append(View(t=float(np.float32(rng.uniform(-1, 1))), width=width, height=height,
                          fx=f, fy=f * rng.uniform(0.9, 1.1),
                          cx=width / 2.0 + rng.uniform(-5, 5), cy=height / 2.0 + rng.uniform(-5, 5),
                          w2c=w2c, i2g=i2g, lod_r=lod[0], lod_pmax=lod[1], lod_D=lod[2],
                          lod_seed=int(rng.integers(0, 2**63)), frame=v, cam=0))
    return scene, views


def make_config(name: str, scale: float = 1.0, n_views: Optional[int] = None,
                width: Optional[int] = None, height: Optional[int] = None,
                seed: Optional[int] = None) -> Tuple[Scene, List[View]]:
    """Scene + views for a BASELINE config ("toy", "street", "av2", "drive")."""
    if name == "toy":
        return make_toy()
    cfg = CONFIGS[name]
    scene, traj = make_street_scene(cfg, scale=scale, seed=seed)
    views = make_views(cfg, traj, n_views=n_views, width=width, height=height, seed=seed)
    return scene, views
