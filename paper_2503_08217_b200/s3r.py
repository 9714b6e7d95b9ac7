"""Thin Python binding of libs3r.so (include/s3r.h) — argument marshalling only.

Every step of the path runs in the CUDA kernels behind the C ABI; this module
turns torch tensors into pointers and the header's structs into ctypes
structs.  PyTorch provides device memory and streams.  There is no fallback:
if libs3r.so is missing and cannot be built, or no CUDA device is present,
the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("S3R_LIB") or os.path.join(_HERE, "libs3r.so")   # S3R_LIB: A/B builds
_lock = threading.Lock()
_lib = None

S3R_OK, S3R_EINVAL, S3R_EINSTANCE, S3R_ENOMEM, S3R_ECUDA, S3R_ESTATE, S3R_EINTERNAL, \
    S3R_ECAPACITY = 0, -1, -2, -3, -4, -5, -6, -7
STAGES = ["filter", "project", "depth_sort", "bin", "raster", "color"]
TILE = 16
# every symbol include/s3r.h declares
EXPORTS = ["s3r_version", "s3r_create", "s3r_destroy", "s3r_last_error", "s3r_set_debug",
           "s3r_set_counters", "s3r_set_timing", "s3r_get_stage_times", "s3r_compose_instance_cameras", "s3r_render",
           "s3r_render_batch", "s3r_render_batch_host", "s3r_get_stats",
           "s3r_dump_intermediates", "s3r_commit_visibility", "s3r_reset_visibility",
           "s3r_life_flip", "s3r_check", "s3r_set_training", "s3r_render_backward",
           "s3r_mse", "s3r_set_pipeline", "s3r_set_lod_jitter", "s3r_set_neural_colors",
           "s3r_set_overlap", "s3r_set_fast_exp", "s3r_set_capacity", "s3r_capacity_from_last"]
S3R_PIPELINE_STREAMLINED, S3R_PIPELINE_CONVENTIONAL = 0, 1


class S3RError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"s3r error {code}: {msg}")
        self.code = code


class Scene_(C.Structure):
    _fields_ = [("n", C.c_int64), ("num_instances", C.c_int32),
                ("means_opacity", C.c_void_p), ("scales", C.c_void_p),
                ("rotations", C.c_void_p), ("colors", C.c_void_p),
                ("instance_ids", C.c_void_p), ("visibility", C.c_void_p), ("life", C.c_void_p)]


class View_(C.Structure):
    _fields_ = [("t", C.c_float), ("width", C.c_int32), ("height", C.c_int32),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("near_plane", C.c_float), ("instance_w2c", C.c_void_p),
                ("lod_r", C.c_float), ("lod_pmax", C.c_float), ("lod_D", C.c_float),
                ("lod_seed", C.c_uint64)]


class Outputs_(C.Structure):
    _fields_ = [("rgb", C.c_void_p), ("depth", C.c_void_p), ("final_T", C.c_void_p),
                ("visible", C.c_void_p)]


class Stats_(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("n_scene", "n_temporal", "n_visible", "n_lod_small",
                                         "n_lod_dropped", "n_rendered", "n_pairs",
                                         "n_bad_instance", "n_bin_pairs", "n_blend_evals",
                                         "n_blend_exec")]


class Capacity_(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("records", "rendered_view", "bin_pairs", "tile_entries",
                                         "temporal_view")]


class Cot_(C.Structure):
    _fields_ = [("rgb", C.c_void_p), ("depth", C.c_void_p), ("final_T", C.c_void_p)]


class Grads_(C.Structure):
    _fields_ = [("means_opacity", C.c_void_p), ("scales", C.c_void_p),
                ("rotations", C.c_void_p), ("colors", C.c_void_p), ("table", C.c_void_p)]


class Debug_(C.Structure):
    _fields_ = [("temporal_idx", C.c_void_p), ("keys", C.c_void_p), ("flags", C.c_void_p),
                ("rect", C.c_void_p), ("depth_order", C.c_void_p), ("pair_tile", C.c_void_p),
                ("pair_gauss", C.c_void_p), ("ranges", C.c_void_p), ("splat_rgb", C.c_void_p)]


class Neurf_(C.Structure):
    _fields_ = [("w1", C.c_void_p), ("b1", C.c_void_p), ("w2", C.c_void_p), ("b2", C.c_void_p),
                ("w3", C.c_void_p), ("b3", C.c_void_p), ("time_emb", C.c_void_p),
                ("n_time", C.c_int32), ("class_emb", C.c_void_p), ("num_instances", C.c_int32),
                ("pos_scale", C.c_float)]


def lib_path() -> str:
    return _SO


def lib():
    """Load libs3r.so (building it in-tree with nvcc if absent)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_SO):
                from . import build as _b
                _b.build()
            L = C.CDLL(_SO)
            P, I, I64 = C.c_void_p, C.c_int, C.c_int64
            sig = {
                "s3r_version": (I, []),
                "s3r_create": (I, [I, C.POINTER(C.c_void_p)]),
                "s3r_destroy": (None, [P]),
                "s3r_last_error": (C.c_char_p, [P]),
                "s3r_set_debug": (I, [P, I]),
                "s3r_set_counters": (I, [P, I]),
                "s3r_set_timing": (I, [P, I]),
                "s3r_get_stage_times": (I, [P, P, P]),
                "s3r_compose_instance_cameras": (I, [P, P, P, C.c_int32, C.c_int32, P, P]),
                "s3r_render": (I, [P, P, P, P, P]),
                "s3r_render_batch": (I, [P, P, P, C.c_int32, P, P]),
                "s3r_render_batch_host": (I, [P, P, P, C.c_int32, P, P]),
                "s3r_get_stats": (I, [P, C.c_int32, P]),
                "s3r_dump_intermediates": (I, [P, C.c_int32, P, P]),
                "s3r_commit_visibility": (I, [P, P, C.c_float, P]),
                "s3r_reset_visibility": (I, [P, P, P]),
                "s3r_life_flip": (I, [P, P, I64, P]),
                "s3r_set_training": (I, [P, I]),
                "s3r_set_pipeline": (I, [P, I]),
                "s3r_set_overlap": (I, [P, I]),
                "s3r_set_fast_exp": (I, [P, I]),
                "s3r_set_lod_jitter": (I, [P, C.c_float, C.c_float, C.c_float]),
                "s3r_set_neural_colors": (I, [P, P, P]),
                "s3r_render_backward": (I, [P, P, P, C.c_int32, P, P, P]),
                "s3r_mse": (I, [P, P, P, I64, C.c_float, P, P, P]),
                "s3r_check": (I, [P, P]),
                "s3r_set_capacity": (I, [P, P]),
                "s3r_capacity_from_last": (I, [P, C.c_float, P]),
            }
            for name, (res, args) in sig.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def _req(t, name: str, dtype, shape, device=None, optional: bool = False):
    """Argument check before a pointer crosses the ABI: the kernels index these
    buffers by the sizes in the structs, so a wrong dtype / shape / device or a
    non-contiguous view would make them read or write out of bounds.  Raises
    ValueError (never stripped, unlike assert)."""
    if t is None:
        if optional:
            return
        raise ValueError(f"{name}: required tensor is None")
    if not torch.is_tensor(t):
        raise ValueError(f"{name}: expected a torch.Tensor, got {type(t).__name__}")
    if t.dtype != dtype:
        raise ValueError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    if device is not None and (not t.is_cuda or t.device.index != device):
        raise ValueError(f"{name}: on {t.device}, expected cuda:{device}")


def _req_table(t, name: str, K1: int, device):
    if not (torch.is_tensor(t) and t.dtype == torch.float32 and t.numel() == 12 * K1
            and t.is_contiguous() and t.is_cuda and t.device.index == device):
        raise ValueError(f"{name}: expected a contiguous float32 cuda:{device} tensor of "
                         f"{K1} x 12 floats (per-instance 3x4 local->camera)")


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


@dataclass
class DeviceScene:
    """Scene tensors on one CUDA device (SoA, 16-byte rows)."""
    means_opacity: torch.Tensor   # (N,4) f32
    scales: torch.Tensor          # (N,4) f32
    rotations: torch.Tensor       # (N,4) f32
    colors: torch.Tensor          # (N,4) f32
    instance_ids: torch.Tensor    # (N,) i32
    visibility: torch.Tensor      # (N,2) f32
    life: Optional[torch.Tensor]  # (N,2) f32 or None
    num_instances: int

    @property
    def n(self) -> int:
        return int(self.means_opacity.shape[0])

    @staticmethod
    def from_numpy(scene, device="cuda", life: bool = True) -> "DeviceScene":
        f = lambda a, dt=torch.float32: torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dt)
        return DeviceScene(f(scene.means_opacity), f(scene.scales), f(scene.rotations),
                           f(scene.colors), f(scene.instance_ids, torch.int32),
                           f(scene.visibility), f(scene.life) if life else None,
                           int(scene.num_instances))

    def check(self, device: Optional[int] = None):
        n = self.n
        for k in ("means_opacity", "scales", "rotations", "colors"):
            _req(getattr(self, k), f"scene.{k}", torch.float32, (n, 4), device)
        _req(self.instance_ids, "scene.instance_ids", torch.int32, (n,), device)
        _req(self.visibility, "scene.visibility", torch.float32, (n, 2), device)
        _req(self.life, "scene.life", torch.float32, (n, 2), device, optional=True)

    def struct(self, device: Optional[int] = None) -> Scene_:
        self.check(device)
        return Scene_(self.n, self.num_instances, _ptr(self.means_opacity), _ptr(self.scales),
                      _ptr(self.rotations), _ptr(self.colors), _ptr(self.instance_ids),
                      _ptr(self.visibility), _ptr(self.life))


def view_struct(v, table: torch.Tensor) -> View_:
    """scenegen.View (or any object with the same fields) + its device table."""
    return View_(float(v.t), int(v.width), int(v.height), float(v.fx), float(v.fy), float(v.cx),
                 float(v.cy), float(getattr(v, "near", 0.01)), _ptr(table), float(v.lod_r),
                 float(v.lod_pmax), float(v.lod_D), int(v.lod_seed) & ((1 << 64) - 1))


class Context:
    """One s3r_ctx on one CUDA device."""

    def __init__(self, device: int = 0):
        if not torch.cuda.is_available():
            raise RuntimeError("s3r needs a CUDA device (no CPU fallback)")
        self.L = lib()
        self.device = device
        h = C.c_void_p()
        rc = self.L.s3r_create(device, C.byref(h))
        if rc != S3R_OK:
            raise S3RError(rc, "s3r_create failed")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.s3r_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int, allow=(S3R_OK,)):
        if rc not in allow:
            raise S3RError(rc, self.L.s3r_last_error(self.h).decode())
        return rc

    # -- configuration
    def set_debug(self, on: bool):
        self._check(self.L.s3r_set_debug(self.h, int(on)))

    def set_counters(self, on: bool):
        self._check(self.L.s3r_set_counters(self.h, int(on)))

    def set_timing(self, on: bool):
        self._check(self.L.s3r_set_timing(self.h, int(on)))

    def stage_times(self) -> Dict[str, float]:
        ms = (C.c_double * len(STAGES))()
        cnt = C.c_int64()
        self._check(self.L.s3r_get_stage_times(self.h, ms, C.byref(cnt)))
        out = {k: ms[i] for i, k in enumerate(STAGES)}
        out["renders"] = cnt.value
        return out

    # -- path
    def compose(self, w2c: torch.Tensor, i2g: Optional[torch.Tensor], stream=None) -> torch.Tensor:
        """(V,3,4) world->camera and (V,K,3,4) object->world -> (V,K+1,12) tables."""
        w2c = w2c.contiguous()
        V = w2c.shape[0]
        K = 0 if i2g is None else int(i2g.shape[1])
        out = torch.empty((V, K + 1, 12), dtype=torch.float32, device=w2c.device)
        i2g_c = None if (i2g is None or K == 0) else i2g.contiguous()
        self._check(self.L.s3r_compose_instance_cameras(self.h, _ptr(w2c), _ptr(i2g_c), V, K,
                                                        _ptr(out), _stream(stream)))
        return out

    def _check_views(self, scene: DeviceScene, views, tables, outs):
        if not (len(views) == len(tables) == len(outs)):
            raise ValueError(f"{len(views)} views, {len(tables)} tables, {len(outs)} outputs")
        for i, (v, t, o) in enumerate(zip(views, tables, outs)):
            _req_table(t, f"tables[{i}]", scene.num_instances, self.device)
            H, W = int(v.height), int(v.width)
            _req(o.get("rgb"), f"outs[{i}]['rgb']", torch.float32, (H, W, 3), self.device)
            _req(o.get("depth"), f"outs[{i}]['depth']", torch.float32, (H, W), self.device, True)
            _req(o.get("final_T"), f"outs[{i}]['final_T']", torch.float32, (H, W), self.device,
                 True)
            _req(o.get("visible"), f"outs[{i}]['visible']", torch.uint8, (scene.n,), self.device,
                 True)

    def render_batch(self, scene: DeviceScene, views: Sequence, tables: Sequence[torch.Tensor],
                     outs: Sequence[Dict[str, torch.Tensor]], stream=None) -> int:
        n = len(views)
        self._check_views(scene, views, tables, outs)
        vs = (View_ * max(n, 1))(*[view_struct(v, t) for v, t in zip(views, tables)])
        os_ = (Outputs_ * max(n, 1))(*[Outputs_(_ptr(o["rgb"]), _ptr(o.get("depth")),
                                                _ptr(o.get("final_T")), _ptr(o.get("visible")))
                                       for o in outs])
        sc = scene.struct(self.device)
        return self._check(self.L.s3r_render_batch(self.h, C.byref(sc), vs, n, os_,
                                                   _stream(stream)),
                           allow=(S3R_OK, S3R_EINSTANCE))

    def render_batch_host(self, scene, views: Sequence, tables: Sequence[np.ndarray],
                          outs: Sequence[Dict[str, np.ndarray]], stream=None) -> int:
        """All buffers in host memory (numpy, ideally pinned); copies inside the call."""
        def hp(a):
            return None if a is None else C.c_void_p(a.ctypes.data)
        n = len(views)
        vs = (View_ * max(n, 1))(*[View_(float(v.t), v.width, v.height, v.fx, v.fy, v.cx, v.cy,
                                         float(getattr(v, "near", 0.01)), hp(t), v.lod_r,
                                         v.lod_pmax, v.lod_D, int(v.lod_seed) & ((1 << 64) - 1))
                                   for v, t in zip(views, tables)])
        os_ = (Outputs_ * max(n, 1))(*[Outputs_(hp(o["rgb"]), hp(o.get("depth")),
                                                hp(o.get("final_T")), hp(o.get("visible")))
                                       for o in outs])
        sc = Scene_(scene.n, scene.num_instances, hp(scene.means_opacity), hp(scene.scales),
                    hp(scene.rotations), hp(scene.colors), hp(scene.instance_ids),
                    hp(scene.visibility), hp(scene.life))
        return self._check(self.L.s3r_render_batch_host(self.h, C.byref(sc), vs, n, os_,
                                                        _stream(stream)),
                           allow=(S3R_OK, S3R_EINSTANCE))

    def stats(self, view_index: int) -> Dict[str, int]:
        s = Stats_()
        self._check(self.L.s3r_get_stats(self.h, view_index, C.byref(s)))
        return {k: getattr(s, k) for k, _ in Stats_._fields_}

    def dump(self, view_index: int, width: int, height: int, keys: bool = True,
             stream=None) -> Dict[str, torch.Tensor]:
        st = self.stats(view_index)
        dev = torch.device("cuda", self.device)
        nt, nr, npairs = st["n_temporal"], st["n_rendered"], st["n_pairs"]
        ntiles = ((width + TILE - 1) // TILE) * ((height + TILE - 1) // TILE)
        d = {"temporal_idx": torch.empty(nt, dtype=torch.int32, device=dev),
             "pair_tile": torch.empty(npairs, dtype=torch.int32, device=dev),
             "ranges": torch.empty((ntiles, 2), dtype=torch.int32, device=dev),
             "splat_rgb": torch.empty((nr, 3), dtype=torch.float32, device=dev)}
        if keys:
            d.update(keys=torch.empty((nt, 6), dtype=torch.float32, device=dev),
                     flags=torch.empty(nt, dtype=torch.uint8, device=dev),
                     rect=torch.empty((nt, 4), dtype=torch.int16, device=dev),
                     depth_order=torch.empty(nr, dtype=torch.int32, device=dev),
                     pair_gauss=torch.empty(npairs, dtype=torch.int32, device=dev))
        dbg = Debug_(*[_ptr(d.get(k)) if (k in d and d[k].numel()) else None
                       for k, _ in Debug_._fields_])
        self._check(self.L.s3r_dump_intermediates(self.h, view_index, C.byref(dbg),
                                                  _stream(stream)))
        return d

    def commit_visibility(self, scene: DeviceScene, margin: float = 0.1, stream=None):
        sc = scene.struct(self.device)
        self._check(self.L.s3r_commit_visibility(self.h, C.byref(sc), margin, _stream(stream)))

    def reset_visibility(self, scene: DeviceScene, stream=None):
        sc = scene.struct(self.device)
        self._check(self.L.s3r_reset_visibility(self.h, C.byref(sc), _stream(stream)))

    def set_pipeline(self, conventional: bool):
        """NEXT-2: the conventional pipeline (world transform of every dynamic
        Gaussian, all Gaussians projected, no temporal filter, no LOD) for the
        following renders; tables then carry [W_t, W_{t,i2g}...] (see
        conventional_tables)."""
        self._check(self.L.s3r_set_pipeline(
            self.h, S3R_PIPELINE_CONVENTIONAL if conventional else S3R_PIPELINE_STREAMLINED))

    def set_overlap(self, on: bool):
        """Overlapped batch halves (s3r_set_overlap); off by default."""
        self._check(self.L.s3r_set_overlap(self.h, int(on)))

    def set_capacity(self, cap: Optional[Dict[str, int]]):
        """Capacity mode (s3r_set_capacity): batches are sized on the device from
        these reservations (keys of Capacity_), without host synchronisation, so
        a render_batch can be captured in a CUDA graph; None switches it off.
        Overflows render the view empty and surface in check() (S3R_ECAPACITY)."""
        if cap is None:
            self._check(self.L.s3r_set_capacity(self.h, None))
            return
        c = Capacity_(*[int(cap[k]) for k, _ in Capacity_._fields_])
        self._check(self.L.s3r_set_capacity(self.h, C.byref(c)))

    def capacity_from_last(self, margin: float = 1.25) -> Dict[str, int]:
        """What the last batch needed, times `margin` (s3r_capacity_from_last)."""
        c = Capacity_()
        self._check(self.L.s3r_capacity_from_last(self.h, float(margin), C.byref(c)))
        return {k: getattr(c, k) for k, _ in Capacity_._fields_}

    def set_fast_exp(self, on: bool):
        """SFU ex2.approx in the rasterizer (s3r_set_fast_exp); off by default.
        Images within 1e-4 of the oracle instead of bit-identical."""
        self._check(self.L.s3r_set_fast_exp(self.h, int(on)))

    def set_lod_jitter(self, dx: float, dy: float, dz: float):
        """NEXT-3: LOD noisy offset scale [dx, dy, dz] (Eq.7 row 4); 0 = off."""
        self._check(self.L.s3r_set_lod_jitter(self.h, float(dx), float(dy), float(dz)))

    def set_neural_colors(self, params: Optional[Dict[str, torch.Tensor]], stream=None):
        """NEXT-4: NeurF colour query (R22) with these weights (device
        fp32 tensors w1 [2,64,64], b1 [2,64], w2, b2, w3 [2,3,64], b3 [2,3],
        time_emb [n_time,8], class_emb [K+1,4], and the float pos_scale), or
        None to switch it off."""
        if params is None:
            self._check(self.L.s3r_set_neural_colors(self.h, None, _stream(stream)))
            return
        t = {k: v.contiguous() for k, v in params.items() if torch.is_tensor(v)}
        for k, v in t.items():
            if not (v.is_cuda and v.dtype == torch.float32 and v.device.index == self.device):
                raise ValueError(f"neural colours: {k} must be float32 on cuda:{self.device}")
        self._neurf_keep = t
        p = Neurf_(_ptr(t["w1"]), _ptr(t["b1"]), _ptr(t["w2"]), _ptr(t["b2"]), _ptr(t["w3"]),
                   _ptr(t["b3"]), _ptr(t["time_emb"]), int(t["time_emb"].shape[0]),
                   _ptr(t["class_emb"]), int(t["class_emb"].shape[0]),
                   float(params["pos_scale"]))
        self._check(self.L.s3r_set_neural_colors(self.h, C.byref(p), _stream(stream)))
        torch.cuda.synchronize(self.device)

    # -- training (config 5)
    def set_training(self, on: bool):
        self._check(self.L.s3r_set_training(self.h, int(on)))

    def render_backward(self, scene: DeviceScene, views: Sequence, tables: Sequence[torch.Tensor],
                        cots: Sequence[Dict[str, torch.Tensor]], grads: Dict[str, torch.Tensor],
                        stream=None):
        """Accumulate dL/d(scene params) of the last (training) forward into grads
        (keys means_opacity, scales, rotations, colors: (N,4) float32 tensors)."""
        n = len(views)
        if not (len(views) == len(tables) == len(cots)):
            raise ValueError(f"{len(views)} views, {len(tables)} tables, {len(cots)} cotangents")
        N, dv = scene.n, self.device
        for i, (v, t, c) in enumerate(zip(views, tables, cots)):
            _req_table(t, f"tables[{i}]", scene.num_instances, dv)
            H, W = int(v.height), int(v.width)
            _req(c.get("rgb"), f"cots[{i}]['rgb']", torch.float32, (H, W, 3), dv, True)
            _req(c.get("depth"), f"cots[{i}]['depth']", torch.float32, (H, W), dv, True)
            _req(c.get("final_T"), f"cots[{i}]['final_T']", torch.float32, (H, W), dv, True)
        for k in ("means_opacity", "scales", "rotations", "colors"):
            _req(grads.get(k), f"grads['{k}']", torch.float32, (N, 4), dv)
        _req(grads.get("table"), "grads['table']", torch.float32, (n, scene.num_instances, 12),
             dv, True)
        vs = (View_ * max(n, 1))(*[view_struct(v, t) for v, t in zip(views, tables)])
        cs = (Cot_ * max(n, 1))(*[Cot_(_ptr(c["rgb"]), _ptr(c.get("depth")),
                                       _ptr(c.get("final_T"))) for c in cots])
        g = Grads_(_ptr(grads["means_opacity"]), _ptr(grads["scales"]),
                   _ptr(grads["rotations"]), _ptr(grads["colors"]), _ptr(grads.get("table")))
        sc = scene.struct(self.device)
        self._check(self.L.s3r_render_backward(self.h, C.byref(sc), vs, n, cs, C.byref(g),
                                               _stream(stream)))

    def mse(self, x: torch.Tensor, y: torch.Tensor, scale: float, grad: torch.Tensor,
            loss: torch.Tensor, stream=None):
        """grad = 2 scale (x - y); loss += scale sum (x - y)^2 (device scalar)."""
        _req(x, "x", torch.float32, tuple(x.shape), self.device)
        _req(y, "y", torch.float32, tuple(x.shape), self.device)
        _req(grad, "grad", torch.float32, tuple(x.shape), self.device)
        _req(loss, "loss", torch.float32, (1,), self.device)
        self._check(self.L.s3r_mse(self.h, _ptr(x), _ptr(y), int(x.numel()), float(scale),
                                   _ptr(grad), _ptr(loss), _stream(stream)))

    def life_flip(self, life: torch.Tensor, stream=None):
        """Negate l_s in place (see s3r_life_flip): brackets an all-reduce MAX."""
        _req(life, "life", torch.float32, (life.shape[0], 2) if life.dim() == 2 else (-1,),
             self.device)
        self._check(self.L.s3r_life_flip(self.h, _ptr(life), int(life.shape[0]),
                                         _stream(stream)))

    def check(self, stream=None) -> int:
        return self._check(self.L.s3r_check(self.h, _stream(stream)),
                           allow=(S3R_OK, S3R_EINSTANCE, S3R_ECAPACITY))


def alloc_outputs(views: Sequence, device="cuda", depth=True, final_T=True, n_visible: int = 0
                  ) -> List[Dict[str, torch.Tensor]]:
    outs = []
    for v in views:
        o = {"rgb": torch.empty((v.height, v.width, 3), dtype=torch.float32, device=device)}
        if depth:
            o["depth"] = torch.empty((v.height, v.width), dtype=torch.float32, device=device)
        if final_T:
            o["final_T"] = torch.empty((v.height, v.width), dtype=torch.float32, device=device)
        if n_visible:
            o["visible"] = torch.empty(n_visible, dtype=torch.uint8, device=device)
        outs.append(o)
    return outs


def conventional_tables(views: Sequence, device="cuda") -> torch.Tensor:
    """Per-view tables of the conventional pipeline: slot 0 = W_t (world ->
    camera), slot i = W_{t,i2g} (instance i local -> world), float[V][K+1][12]."""
    K = views[0].i2g.shape[0] if len(views) else 0
    t = np.zeros((len(views), K + 1, 12), np.float32)
    for j, v in enumerate(views):
        t[j, 0] = np.asarray(v.w2c, np.float32).reshape(12)
        if K:
            t[j, 1:] = np.asarray(v.i2g, np.float32).reshape(K, 12)
    return torch.from_numpy(t).to(device)


def view_tables(ctx: Context, views: Sequence, device="cuda", stream=None) -> torch.Tensor:
    """Instance camera tables for scenegen views, composed on the device."""
    w2c = torch.from_numpy(np.stack([np.asarray(v.w2c, np.float32) for v in views])).to(device)
    K = views[0].i2g.shape[0] if len(views) else 0
    i2g = torch.from_numpy(np.stack([np.asarray(v.i2g, np.float32).reshape(K, 3, 4)
                                     for v in views])).to(device) if K else None
    return ctx.compose(w2c, i2g, stream)
