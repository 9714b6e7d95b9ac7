"""CPU oracle of the S3R-GS streamlined per-view splatting path (ctypes wrapper).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (paper_2503_08217_b200/) never imports it.  The C sources in this
directory are the oracle; this file only marshals numpy arrays to them.

``build()`` compiles liboracle.so with gcc -O2 -ffp-contract=off (see Makefile).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import subprocess
import threading
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
# S3R_ORACLE_SO selects another build of the same sources, e.g. the ASan/UBSan
# one (Makefile target liboracle_san.so, tools/oracle_sanitize.sh)
_SO_ALT = os.environ.get("S3R_ORACLE_SO")
_SRCS = ["s3r_oracle_f32.c", "s3r_oracle_f64.c", "s3r_oracle_bwd.c", "s3r_oracle_impl.inc",
         "s3r_oracle.h", "Makefile"]
_lock = threading.Lock()
_lib = None

F_TEMPORAL, F_VISIBLE, F_SMALL, F_DROPPED, F_RENDERED, F_BADID, F_JITTERED = 1, 2, 4, 8, 16, 32, 64
TILE = 16


def build(force: bool = False) -> str:
    """Compile liboracle.so if missing or older than its sources."""
    newest = max(os.path.getmtime(os.path.join(_HERE, s)) for s in _SRCS)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        subprocess.run(["make", "-s", "-B", "liboracle.so"], cwd=_HERE, check=True)
    return _SO


class Scene(C.Structure):
    _fields_ = [("n", C.c_int64), ("num_instances", C.c_int32),
                ("means_opacity", C.c_void_p), ("scales", C.c_void_p),
                ("rotations", C.c_void_p), ("colors", C.c_void_p),
                ("instance_ids", C.c_void_p), ("visibility", C.c_void_p),
                ("life", C.c_void_p)]


class View(C.Structure):
    _fields_ = [("t", C.c_float), ("width", C.c_int32), ("height", C.c_int32),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("near_plane", C.c_float), ("instance_w2c", C.c_void_p),
                ("lod_r", C.c_float), ("lod_pmax", C.c_float), ("lod_D", C.c_float),
                ("lod_seed", C.c_uint64), ("lod_jitter", C.c_float * 3)]


class Stats(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("n_scene", "n_temporal", "n_visible", "n_lod_small",
                                         "n_lod_dropped", "n_rendered", "n_pairs",
                                         "n_bad_instance")]


class Out(C.Structure):
    _fields_ = [("rgb", C.c_void_p), ("depth", C.c_void_p), ("final_T", C.c_void_p),
                ("visible", C.c_void_p), ("temporal_idx", C.c_void_p), ("keys", C.c_void_p),
                ("splat_keys", C.c_void_p), ("flags", C.c_void_p), ("rect", C.c_void_p), ("pair_tile", C.c_void_p),
                ("pair_gauss", C.c_void_p), ("pair_capacity", C.c_int64),
                ("ranges", C.c_void_p), ("stats", Stats)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if _SO_ALT:
                L = C.CDLL(os.path.abspath(_SO_ALT))
            else:
                build()
                L = C.CDLL(_SO)
            P = C.c_void_p
            sig = {
                "so_normalize_time": (C.c_double, [C.c_int64, C.c_int64]),
                "so_exp2_f32": (C.c_float, [C.c_float]),
                "so_exp_f64": (C.c_double, [C.c_double]),
                "so_splitmix64": (C.c_uint64, [C.c_uint64]),
                "so_lod_uniform": (C.c_float, [C.c_uint64, C.c_int64]),
                "so_compose_instance_cameras": (None, [P, P, C.c_int32, P]),
                "so_temporal_filter_f32": (C.c_int64, [P, C.c_float, P]),
                "so_temporal_filter_f64": (C.c_int64, [P, C.c_double, P]),
                "so_project_f32": (C.c_int, [P, P, C.c_int64, P]),
                "so_project_f64": (C.c_int, [P, P, C.c_int64, P]),
                "so_drop_probability_f32": (C.c_float, [C.c_float, C.c_float, C.c_float]),
                "so_drop_probability_f64": (C.c_double, [C.c_double, C.c_double, C.c_double]),
                "so_render_view_f32": (C.c_int, [P, P, P]),
                "so_render_view_f64": (C.c_int, [P, P, P]),
                "so_blend_bruteforce_f32": (C.c_int, [P, P, P, P, P, P, P, P]),
                "so_blend_bruteforce_f64": (C.c_int, [P, P, P, P, P, P, P, P]),
                "so_backward_f64": (C.c_int, [P, P, P, P, P, P, P]),
                "so_update_life_f32": (None, [P, P, C.c_float]),
                "so_lod_normal3": (None, [C.c_uint64, C.c_int64, P]),
                "so_lod_uniform_k": (C.c_float, [C.c_uint64, C.c_int64, C.c_int]),
                "so_log2_f32": (C.c_float, [C.c_float]),
                "so_sincos_turn_f32": (None, [C.c_float, P, P]),
                "so_quat_from_rot_f32": (None, [P, P]),
                "so_quat_from_rot_f64": (None, [P, P]),
                "so_quat_mul_f32": (None, [P, P, P]),
                "so_quat_mul_f64": (None, [P, P, P]),
                "so_world_transform_f32": (C.c_int64, [P, P, P, P]),
                "so_world_transform_f64": (C.c_int64, [P, P, P, P]),
                "so_commit_visibility": (None, [P, C.c_float]),
                "so_reset_visibility": (None, [P]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _SceneRef:
    """Keeps contiguous numpy arrays alive behind a ctypes Scene struct."""

    def __init__(self, scene, life: bool = True):
        self.arrs = {k: np.ascontiguousarray(getattr(scene, k)) for k in
                     ("means_opacity", "scales", "rotations", "colors", "instance_ids")}
        # visibility / life are mutated in place: keep the caller's arrays if contiguous
        self.visibility = scene.visibility
        self.life = scene.life if life else None
        assert self.visibility.flags.c_contiguous and self.visibility.dtype == np.float32
        if self.life is not None:
            assert self.life.flags.c_contiguous and self.life.dtype == np.float32
        self.s = Scene(scene.n, scene.num_instances, _ptr(self.arrs["means_opacity"]),
                       _ptr(self.arrs["scales"]), _ptr(self.arrs["rotations"]),
                       _ptr(self.arrs["colors"]), _ptr(self.arrs["instance_ids"]),
                       _ptr(self.visibility), _ptr(self.life))


def compose(view) -> np.ndarray:
    """Instance camera table (K+1, 12) f32 for a scenegen.View."""
    K = view.i2g.shape[0]
    w2c = np.ascontiguousarray(view.w2c, np.float32).reshape(12)
    i2g = np.ascontiguousarray(view.i2g, np.float32).reshape(max(K, 0) * 12)
    out = np.zeros((K + 1, 12), np.float32)
    lib().so_compose_instance_cameras(_ptr(w2c), _ptr(i2g) if K else None, K, _ptr(out))
    return out


class _ViewRef:
    def __init__(self, view, table: Optional[np.ndarray] = None):
        self.table = np.ascontiguousarray(compose(view) if table is None else table, np.float32)
        jit = tuple(float(x) for x in getattr(view, "lod_jitter", (0.0, 0.0, 0.0)))
        self.v = View(view.t, view.width, view.height, view.fx, view.fy, view.cx, view.cy,
                      view.near, _ptr(self.table), view.lod_r, view.lod_pmax, view.lod_D,
                      view.lod_seed & ((1 << 64) - 1), (C.c_float * 3)(*jit))


def render_view(scene, view, precision: str = "f32", table: Optional[np.ndarray] = None,
                pairs: bool = True, image: bool = True) -> Dict[str, np.ndarray]:
    """One streamlined render (O1-O6) of one view.  Returns numpy arrays:
    rgb (H,W,3), depth (H,W), final_T (H,W), visible (N,) u8, temporal_idx,
    keys (N,6) (NaN where not projected), flags (N,), rect (N,4),
    pair_tile / pair_gauss (P,), ranges (tiles,2), stats (dict), rc."""
    L = lib()
    real = np.float32 if precision == "f32" else np.float64
    sr, vr = _SceneRef(scene, life=False), _ViewRef(view, table)
    N, W, H = scene.n, view.width, view.height
    TX, TY = (W + TILE - 1) // TILE, (H + TILE - 1) // TILE
    o = {
        "visible": np.zeros(N, np.uint8), "temporal_idx": np.zeros(max(N, 1), np.int32),
        "keys": np.zeros((N, 6), real), "splat_keys": np.full((N, 6), np.nan, real),
        "flags": np.zeros(N, np.uint8),
        "rect": np.zeros((N, 4), np.int16), "ranges": np.zeros((TX * TY, 2), np.int32),
    }
    if image:
        o.update(rgb=np.zeros((H, W, 3), real), depth=np.zeros((H, W), real),
                 final_T=np.zeros((H, W), real))
    out = Out()
    for k in ("rgb", "depth", "final_T", "visible", "temporal_idx", "keys", "splat_keys", "flags",
              "rect", "ranges"):
        if k in o:
            setattr(out, k, _ptr(o[k]))
    fn = L.so_render_view_f32 if precision == "f32" else L.so_render_view_f64
    rc = fn(C.byref(sr.s), C.byref(vr.v), C.byref(out))
    if pairs:
        P = out.stats.n_pairs
        o["pair_tile"] = np.zeros(max(P, 1), np.int32)
        o["pair_gauss"] = np.zeros(max(P, 1), np.int32)
        out.pair_tile, out.pair_gauss = _ptr(o["pair_tile"]), _ptr(o["pair_gauss"])
        out.pair_capacity = P
        # a second, identical run fills the pair list (the oracle is deterministic)
        out.rgb = out.depth = out.final_T = None
        rc = fn(C.byref(sr.s), C.byref(vr.v), C.byref(out))
        o["pair_tile"], o["pair_gauss"] = o["pair_tile"][:P], o["pair_gauss"][:P]
    o["temporal_idx"] = o["temporal_idx"][: out.stats.n_temporal]
    o["stats"] = {k: getattr(out.stats, k) for k, _ in Stats._fields_}
    o["rc"] = rc
    o["table"] = vr.table
    return o


def blend_bruteforce(scene, view, flags, keys, rect, precision="f32", table=None):
    L = lib()
    real = np.float32 if precision == "f32" else np.float64
    sr, vr = _SceneRef(scene, life=False), _ViewRef(view, table)
    H, W = view.height, view.width
    rgb, depth, T = np.zeros((H, W, 3), real), np.zeros((H, W), real), np.zeros((H, W), real)
    keys = np.ascontiguousarray(keys, real)
    flags = np.ascontiguousarray(flags, np.uint8)
    rect = np.ascontiguousarray(rect, np.int16)
    fn = L.so_blend_bruteforce_f32 if precision == "f32" else L.so_blend_bruteforce_f64
    fn(C.byref(sr.s), C.byref(vr.v), _ptr(flags), _ptr(keys), _ptr(rect), _ptr(rgb),
       _ptr(depth), _ptr(T))
    return rgb, depth, T


def backward(scene, view, g_rgb, g_depth=None, g_T=None, table=None, grads=None,
             g_table=None) -> np.ndarray:
    """fp64 adjoint: dL/d(raw params) (n, 16) for one view given dL/d(rgb, depth, T)
    (accumulated into `grads` if given); g_table (num_instances, 12) float64, if
    given, accumulates dL/d(instance camera table) (the NEXT-1 pose gradient)."""
    L = lib()
    sr, vr = _SceneRef(scene, life=False), _ViewRef(view, table)
    g = np.zeros((scene.n, 16), np.float64) if grads is None else grads
    f = lambda a: None if a is None else np.ascontiguousarray(a, np.float64)
    a_rgb, a_d, a_t = f(g_rgb), f(g_depth), f(g_T)
    if g_table is not None:
        assert g_table.dtype == np.float64 and g_table.flags.c_contiguous
    rc = L.so_backward_f64(C.byref(sr.s), C.byref(vr.v), _ptr(a_rgb), _ptr(a_d), _ptr(a_t),
                           _ptr(g), _ptr(g_table))
    assert rc == 0
    return g


def quat_from_rot(R, precision="f32") -> np.ndarray:
    """C0 quat(R) (Shepperd), (w, x, y, z)."""
    real = np.float32 if precision == "f32" else np.float64
    R = np.ascontiguousarray(R, real).reshape(9)
    q = np.zeros(4, real)
    getattr(lib(), "so_quat_from_rot_" + precision)(_ptr(R), _ptr(q))
    return q


def quat_mul(a, b, precision="f32") -> np.ndarray:
    real = np.float32 if precision == "f32" else np.float64
    a, b = np.ascontiguousarray(a, real), np.ascontiguousarray(b, real)
    o = np.zeros(4, real)
    getattr(lib(), "so_quat_mul_" + precision)(_ptr(a), _ptr(b), _ptr(o))
    return o


def world_scene(scene, i2g, precision="f32"):
    """C0 of the conventional pipeline: the scene moved to the world frame for
    one frame's poses i2g (K, 3, 4) — every Gaussian static (id 0, K = 0),
    visibility fresh (-1, 1) so that no temporal filter applies."""
    K1 = scene.num_instances
    tab = np.zeros((max(K1, 1), 12), np.float32)
    if K1 > 1:
        tab[1:] = np.asarray(i2g, np.float32).reshape(-1, 12)[: K1 - 1]
    sr = _SceneRef(scene, life=False)
    mo = np.zeros((scene.n, 4), np.float32)
    rot = np.zeros((scene.n, 4), np.float32)
    getattr(lib(), "so_world_transform_" + precision)(C.byref(sr.s), _ptr(tab), _ptr(mo),
                                                       _ptr(rot))
    w = scene.copy()
    w.means_opacity, w.rotations = mo, rot
    bad = (scene.instance_ids < 0) | (scene.instance_ids >= K1)
    w.instance_ids = np.where(bad, scene.instance_ids, 0).astype(np.int32)
    w.num_instances = 1
    w.visibility = np.tile(np.array([-1.0, 1.0], np.float32), (scene.n, 1))
    return w


def render_view_conventional(scene, view, precision="f32", **kw) -> Dict[str, np.ndarray]:
    """The conventional pipeline (NEXT-2) for one view: C0 world transform with
    the view's i2g poses, then O2-O6 for ALL Gaussians through W_t, no LOD."""
    w = world_scene(scene, view.i2g, precision)
    v = dataclasses.replace(view, i2g=np.zeros((0, 3, 4), np.float32), lod_r=0.0)
    o = render_view(w, v, precision, **kw)
    o["world_scene"] = w
    return o


def lod_normal3(seed: int, g: int) -> np.ndarray:
    """NEXT-3 noise: the three standard normals of Gaussian g (R-ARITH Box-Muller)."""
    o = np.zeros(3, np.float32)
    lib().so_lod_normal3(seed & ((1 << 64) - 1), g, _ptr(o))
    return o


def log2_32(x: float) -> float:
    return lib().so_log2_f32(x)


def sincos_turn(u: float):
    s, c = C.c_float(), C.c_float()
    lib().so_sincos_turn_f32(u, C.byref(s), C.byref(c))
    return s.value, c.value


def lod_uniform_k(seed: int, g: int, k: int) -> float:
    return lib().so_lod_uniform_k(seed & ((1 << 64) - 1), g, k)


def temporal_filter(scene, t, precision="f32") -> np.ndarray:
    L = lib()
    sr = _SceneRef(scene, life=False)
    idx = np.zeros(max(scene.n, 1), np.int32)
    fn = L.so_temporal_filter_f32 if precision == "f32" else L.so_temporal_filter_f64
    m = fn(C.byref(sr.s), t, _ptr(idx))
    return idx[:m]


def project(scene, view, g, precision="f32", table=None):
    """(status, keys[6]) for one Gaussian: status 0 ok, 1 behind near plane, 2 bad id."""
    L = lib()
    real = np.float32 if precision == "f32" else np.float64
    sr, vr = _SceneRef(scene, life=False), _ViewRef(view, table)
    k = np.zeros(6, real)
    fn = L.so_project_f32 if precision == "f32" else L.so_project_f64
    st = fn(C.byref(sr.s), C.byref(vr.v), int(g), _ptr(k))
    return st, k


def drop_probability(d, pmax, D, precision="f32"):
    L = lib()
    fn = L.so_drop_probability_f32 if precision == "f32" else L.so_drop_probability_f64
    return fn(d, pmax, D)


def exp2_32(x: float) -> float:
    """The contract's s3r_exp2 (DESIGN.md R-ARITH)."""
    return lib().so_exp2_f32(x)


def splitmix64(x: int) -> int:
    return lib().so_splitmix64(x & ((1 << 64) - 1))


def lod_uniform(seed: int, g: int) -> float:
    return lib().so_lod_uniform(seed & ((1 << 64) - 1), g)


def normalize_time(frame: int, frames: int) -> float:
    return lib().so_normalize_time(frame, frames)


def update_life(scene, visible: np.ndarray, t: float) -> None:
    sr = _SceneRef(scene, life=True)
    vis = np.ascontiguousarray(visible, np.uint8)
    lib().so_update_life_f32(C.byref(sr.s), _ptr(vis), t)


def commit_visibility(scene, margin: float = 0.1) -> None:
    sr = _SceneRef(scene, life=True)
    lib().so_commit_visibility(C.byref(sr.s), margin)


def reset_visibility(scene) -> None:
    sr = _SceneRef(scene, life=True)
    lib().so_reset_visibility(C.byref(sr.s))
