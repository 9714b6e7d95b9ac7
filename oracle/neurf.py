"""NeurF colour query — CPU ORACLE (NEXT-4 of SURVEY.md §8(f)).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): imported by tests/ and
bench.py's reference leg, never by the product path.

PAPER.md Eq.7 rows 5-6: c = NeurF_sta(mu, d, dir, emb(t))
for static Gaussians and c = NeurF_dyn(mu, d, dir, emb(t), class) for dynamic
ones, queried for "the final visible 3D Gaussians" after the LOD cull (P:155,
P:188).  The paper fixes only the inputs; the architecture is reading R22 of
DESIGN.md (trained weights are out of scope, so the weights are inputs):

  features f in R^64 (44 used, zero padded), per rendered Gaussian, in the
  Gaussian's own frame (instance-local for dynamic ones, world for static):
    f[0:3]   mu / S
    f[3:27]  for l in 0..3, for axis a in x,y,z: sin(2^l pi mu_a / S), cos(...)
             (index 3 + 6 l + 2 a + {0: sin, 1: cos})
    f[27]    min(1, d / D)            (reading R10's normalize(d); d = camera depth)
    f[28:31] dir = R_i^T p / |p|      (p = W_{t,i} mu the camera-frame position,
                                       R_i the rotation of the instance camera)
    f[31:39] emb(t): linear interpolation of an [n_time][8] table on the uniform
             grid t_j = -1 + 2 j / (n_time - 1)
    f[39:43] class embedding of the instance ([K+1][4] table; 0 for static)
  MLP per network (sta / dyn): h1 = relu(W1 f + b1), h2 = relu(W2 h1 + b2),
  c = sigmoid(W3 h2 + b3), W1, W2 in R^{64x64}, W3 in R^{3x64}.
  Precision (the tensor-core contract): f, W*, h1, h2 rounded to bf16
  (round-to-nearest-even) where the kernel stores them; every dot product and
  bias / activation exact (here fp64; the kernel accumulates in fp32).
"""
from __future__ import annotations

import numpy as np

FEAT, HID, NFREQ, NEMB_T, NEMB_C = 64, 64, 4, 8, 4


def bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 values to bfloat16 (nearest, ties to even), returned as
    float32 — the conversion cvt.rn.bf16.f32 performs."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def time_embedding(t: float, table: np.ndarray) -> np.ndarray:
    """emb(t): linear interpolation on t_j = -1 + 2 j / (n - 1) (clamped)."""
    table = np.asarray(table, np.float64)
    n = table.shape[0]
    if n == 1:
        return table[0].copy()
    x = (float(t) + 1.0) * 0.5 * (n - 1)
    j = int(min(max(np.floor(x), 0), n - 2))
    w = min(max(x - j, 0.0), 1.0)
    return (1.0 - w) * table[j] + w * table[j + 1]


def features(mu: np.ndarray, p: np.ndarray, R: np.ndarray, emb_t: np.ndarray,
             cls: np.ndarray, S: float, D: float) -> np.ndarray:
    """f (n, 64) in fp64.  mu: own-frame means (n,3); p: camera-frame positions
    (n,3); R: instance-camera rotations (n,3,3); emb_t (8,); cls (n,4)."""
    n = mu.shape[0]
    f = np.zeros((n, FEAT))
    m = mu / S
    f[:, 0:3] = m
    for l in range(NFREQ):
        for a in range(3):
            arg = (2.0 ** l) * np.pi * m[:, a]
            f[:, 3 + 6 * l + 2 * a] = np.sin(arg)
            f[:, 3 + 6 * l + 2 * a + 1] = np.cos(arg)
    f[:, 27] = np.minimum(1.0, p[:, 2] / D)
    ph = p / np.linalg.norm(p, axis=1, keepdims=True)
    f[:, 28:31] = np.einsum("nji,nj->ni", R, ph)          # R^T p_hat
    f[:, 31:39] = emb_t[None, :]
    f[:, 39:43] = cls
    return f


def mlp(f: np.ndarray, dyn: np.ndarray, params: dict) -> np.ndarray:
    """c (n, 3) = NeurF_{sta|dyn}(f), bf16 rounding at the stored tensors."""
    out = np.zeros((f.shape[0], 3))
    fb = bf16(f.astype(np.float32)).astype(np.float64)
    for net in (0, 1):
        sel = dyn == bool(net)
        if not np.any(sel):
            continue
        W1 = bf16(params["w1"][net]).astype(np.float64)
        W2 = bf16(params["w2"][net]).astype(np.float64)
        W3 = bf16(params["w3"][net]).astype(np.float64)
        b1, b2, b3 = (np.asarray(params[k][net], np.float64) for k in ("b1", "b2", "b3"))
        h1 = np.maximum(fb[sel] @ W1.T + b1, 0.0)
        h1 = bf16(h1.astype(np.float32)).astype(np.float64)
        h2 = np.maximum(h1 @ W2.T + b2, 0.0)
        h2 = bf16(h2.astype(np.float32)).astype(np.float64)
        z = h2 @ W3.T + b3
        out[sel] = 1.0 / (1.0 + np.exp(-z))
    return out


def query_colors(scene, view, table: np.ndarray, gs: np.ndarray, params: dict,
                 mu: np.ndarray | None = None) -> np.ndarray:
    """Colours (len(gs), 3) of Gaussians gs of `scene` seen by `view` through
    the instance camera table (K+1, 12).  mu: own-frame means to use (default:
    the scene's; the LOD noisy offset passes the moved ones)."""
    gs = np.asarray(gs, np.int64)
    ids = scene.instance_ids[gs]
    mu = scene.means_opacity[gs, :3].astype(np.float64) if mu is None else np.asarray(mu, np.float64)
    M = np.asarray(table, np.float64).reshape(-1, 3, 4)[ids]
    R = M[:, :, :3]
    p = np.einsum("nij,nj->ni", R, mu) + M[:, :, 3]
    emb_t = time_embedding(view.t, params["time_emb"])
    cls = np.asarray(params["class_emb"], np.float64)[ids]
    f = features(mu, p, R, emb_t, cls, float(params["pos_scale"]), float(view.lod_D))
    return mlp(f, ids > 0, params)


def random_params(rng: np.random.Generator, num_instances: int, n_time: int = 16,
                  pos_scale: float = 100.0) -> dict:
    """Random weights of the shapes R22 fixes (no trained weights exist here):
    He-style scales so that the activations stay O(1)."""
    s1, s2 = np.sqrt(2.0 / 44), np.sqrt(2.0 / HID)
    p = {"w1": rng.normal(0, s1, (2, HID, FEAT)).astype(np.float32),
         "b1": rng.normal(0, 0.1, (2, HID)).astype(np.float32),
         "w2": rng.normal(0, s2, (2, HID, HID)).astype(np.float32),
         "b2": rng.normal(0, 0.1, (2, HID)).astype(np.float32),
         "w3": rng.normal(0, s2, (2, 3, HID)).astype(np.float32),
         "b3": rng.normal(0, 0.1, (2, 3)).astype(np.float32),
         "time_emb": rng.normal(0, 1, (n_time, NEMB_T)).astype(np.float32),
         "class_emb": rng.normal(0, 1, (num_instances, NEMB_C)).astype(np.float32),
         "pos_scale": float(pos_scale)}
    p["w1"][:, :, 43:] = 0.0          # padded feature columns carry no weight
    p["class_emb"][0] = 0.0
    return p
