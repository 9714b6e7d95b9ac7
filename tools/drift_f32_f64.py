"""fp32 contract vs fp64 shadow at full density.

The fp64 shadow is Eq.2 as written (libm exp, natural power form, T(1 - alpha),
no flush); the fp32 contract is the R-ARITH evaluation the GPU reproduces bit
for bit (exp2 form, degree-4 polynomial, 2^-24 flush, T - w).  On full-size
views of C3 (av2) and C4 (drive) this reports, per view: max |delta| of RGB /
depth / final T, the number of pixels over 1e-4, the pixels whose termination
status (final T < 1e-4) differs, and the Gaussians whose integer decisions
(visible / small / dropped / rendered) differ; and, key-fed (the fp64 blend
of the fp32 contract's own keys), the same image deltas, which isolate the blend
arithmetic from the fp32 projection (--keyfed; a brute-force gather, for small
views only).  CPU only (oracle), one worker process per view.

    python tools/drift_f32_f64.py [--views 2] [--out profiles/r02_f32_vs_f64_drift.json]
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

_G = {}


def keyfed_np(scene, view, o):
    """fp64 Eq.2 (alpha = min(0.99, o exp(power)), include-then-stop
    at T < 1e-4, no flush) over the oracle's fp32 tile lists and splat keys
    (mx, my, z, a, b, c; conic from the dilated 2D covariance, reading R5),
    all tiles at once, one list position at a time."""
    W, H = view.width, view.height
    TX, TY = (W + 15) // 16, (H + 15) // 16
    nt = TX * TY
    rg = o["ranges"].astype(np.int64)
    cnt = rg[:, 1] - rg[:, 0]
    L = int(cnt.max()) if nt else 0
    k = np.nan_to_num(o["splat_keys"].astype(np.float64))   # NaN rows: not rendered (never used)
    op = scene.means_opacity[:, 3].astype(np.float64)
    col = scene.colors[:, :3].astype(np.float64)
    a_, b_, c_ = k[:, 3] + 0.3, k[:, 4], k[:, 5] + 0.3
    det = a_ * c_ - b_ * b_
    with np.errstate(all="ignore"):
        A, B, Cc = c_ / det, -b_ / det, a_ / det
    # pixel coordinates of every tile's 256 pixels
    ly, lx = np.divmod(np.arange(256), 16)
    tx, ty = np.arange(nt) % TX, np.arange(nt) // TX
    px = (tx[:, None] * 16 + lx[None, :]).astype(np.float64)
    py = (ty[:, None] * 16 + ly[None, :]).astype(np.float64)
    T = np.ones((nt, 256))
    C = np.zeros((nt, 256, 3))
    D = np.zeros((nt, 256))
    live = np.ones((nt, 256), bool)
    pg = o["pair_gauss"]
    for j in range(L):
        has = cnt > j
        g = np.where(has, pg[np.minimum(rg[:, 0] + j, len(pg) - 1)], 0)
        dx = k[g, 0][:, None] - px
        dy = k[g, 1][:, None] - py
        power = np.minimum(0.0, -0.5 * (A[g][:, None] * dx * dx + Cc[g][:, None] * dy * dy)
                           - B[g][:, None] * dx * dy)
        alpha = np.minimum(0.99, op[g][:, None] * np.exp(power))
        m = live & has[:, None]
        w = np.where(m, alpha * T, 0.0)
        C += w[:, :, None] * col[g][:, None, :]
        D += w * k[g, 2][:, None]
        T = np.where(m, T * (1.0 - alpha), T)
        live &= ~(m & (T < 1e-4))
    img = np.zeros((TY * 16, TX * 16, 3))
    dep = np.zeros((TY * 16, TX * 16))
    Ti = np.ones((TY * 16, TX * 16))
    for arr, out in ((C, img), (D, dep), (T, Ti)):
        v = arr.reshape(TY, TX, 16, 16, *arr.shape[2:]).swapaxes(1, 2)
        out[...] = v.reshape(TY * 16, TX * 16, *arr.shape[2:])
    return img[:H, :W], dep[:H, :W], Ti[:H, :W]


def _one(job):
    import oracle
    cfg, vi = job
    scene, view = _G[cfg]["scene"], _G[cfg]["views"][vi]
    t0 = time.perf_counter()
    a = oracle.render_view(scene, view, "f32")
    b = oracle.render_view(scene, view, "f64")
    dt = time.perf_counter() - t0
    r = {"config": cfg, "view": int(vi), "oracle_s_both": round(dt, 1),
         "pixels": int(a["rgb"].shape[0] * a["rgb"].shape[1])}
    drgb = np.abs(a["rgb"].astype(np.float64) - b["rgb"]).max(-1)
    ddep = np.abs(a["depth"].astype(np.float64) - b["depth"])
    dT = np.abs(a["final_T"].astype(np.float64) - b["final_T"])
    r["rgb_max_abs"] = float(drgb.max())
    r["depth_max_abs"] = float(ddep.max())
    r["final_T_max_abs"] = float(dT.max())
    r["rgb_px_over_1e-4"] = int((drgb > 1e-4).sum())
    r["depth_px_over_1e-4"] = int((ddep > 1e-4).sum())
    r["rgb_p99999"] = float(np.quantile(drgb, 0.99999))
    r["depth_p99999"] = float(np.quantile(ddep, 0.99999))
    ta, tb = a["final_T"] < 1e-4, b["final_T"] < 1e-4
    flip = ta != tb
    r["termination_status_flips"] = int(flip.sum())
    r["terminated_px_f64"] = int(tb.sum())
    nf = ~flip
    r["rgb_max_abs_no_flip"] = float(drgb[nf].max())
    r["depth_max_abs_no_flip"] = float(ddep[nf].max())
    r["rgb_px_over_1e-4_no_flip"] = int((drgb[nf] > 1e-4).sum())
    r["depth_px_over_1e-4_no_flip"] = int((ddep[nf] > 1e-4).sum())
    r["max_depth_value"] = float(b["depth"].max())
    fa, fb = a["flags"], b["flags"]
    r["decision_flips"] = int((fa != fb).sum())
    r["n_rendered_f32"] = int(a["stats"]["n_rendered"])
    r["n_rendered_f64"] = int(b["stats"]["n_rendered"])
    r["n_pairs_f32"] = int(a["stats"]["n_pairs"])
    r["n_pairs_f64"] = int(b["stats"]["n_pairs"])
    m = ~np.isnan(a["keys"][:, 0]) & ~np.isnan(b["keys"][:, 0])
    ka, kb = a["keys"][m].astype(np.float64), b["keys"][m]
    scale = np.maximum(np.abs(kb), np.abs(kb[:, 3:4]) + np.abs(kb[:, 5:6]))
    r["keys_max_rel"] = float((np.abs(ka - kb) / np.maximum(scale, 1.0)).max()) if m.any() else 0.0
    # key-fed (numpy, float64): Eq.2 as written, blended over the fp32 contract's
    # own tile lists and splat keys, so only the blend arithmetic differs
    # (exp2 polynomial + 2^-24 flush + T - w vs exp + T (1 - alpha))
    rgb, dep, T = keyfed_np(scene, view, a)
    krgb = np.abs(a["rgb"].astype(np.float64) - rgb).max(-1)
    kdep = np.abs(a["depth"].astype(np.float64) - dep)
    kflip = (a["final_T"] < 1e-4) != (T < 1e-4)
    r["keyfed_np"] = {"rgb_max_abs": float(krgb.max()), "depth_max_abs": float(kdep.max()),
                      "final_T_max_abs": float(np.abs(a["final_T"] - T).max()),
                      "rgb_px_over_1e-4": int((krgb > 1e-4).sum()),
                      "depth_px_over_1e-4": int((kdep > 1e-4).sum()),
                      "depth_max_rel": float((kdep / np.maximum(dep, 1e-3)).max()),
                      "termination_status_flips": int(kflip.sum()),
                      "rgb_max_abs_no_flip": float(krgb[~kflip].max())}
    if not _G.get("keyfed"):
        r["oracle_s_total"] = round(time.perf_counter() - t0, 1)
        return r
    # key-fed: the fp64 blend (Eq.2 as written) of the fp32 contract's own keys,
    # decisions and rectangles; isolates the blend arithmetic (exp2 polynomial,
    # 2^-24 flush, T - w) from the fp32 projection of world coordinates
    rgb, dep, T = oracle.blend_bruteforce(scene, view, a["flags"], a["keys"], a["rect"], "f64")
    krgb = np.abs(a["rgb"].astype(np.float64) - rgb).max(-1)
    kdep = np.abs(a["depth"].astype(np.float64) - dep)
    kflip = (a["final_T"] < 1e-4) != (T < 1e-4)
    r["keyfed"] = {"rgb_max_abs": float(krgb.max()), "depth_max_abs": float(kdep.max()),
                   "final_T_max_abs": float(np.abs(a["final_T"] - T).max()),
                   "rgb_px_over_1e-4": int((krgb > 1e-4).sum()),
                   "depth_px_over_1e-4": int((kdep > 1e-4).sum()),
                   "depth_max_rel": float((kdep / np.maximum(dep, 1e-30)).max()),
                   "termination_status_flips": int(kflip.sum()),
                   "rgb_max_abs_no_flip": float(krgb[~kflip].max())}
    r["oracle_s_total"] = round(time.perf_counter() - t0, 1)
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=2)
    ap.add_argument("--configs", default="av2,drive")
    ap.add_argument("--workers", type=int, default=min(8, os.cpu_count() or 1))
    ap.add_argument("--keyfed", action="store_true",
                    help="also the brute-force fp64 blend of the fp32 keys (O(pixels x N): "
                         "small views only)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_f32_vs_f64_drift.json"))
    a = ap.parse_args()
    from paper_2503_08217_b200 import scenegen as sg
    _G["keyfed"] = a.keyfed
    jobs = []
    for cfg in a.configs.split(","):
        scene, views = sg.make_config(cfg)
        pick = np.linspace(0, len(views) - 1, a.views).round().astype(int)
        _G[cfg] = {"scene": scene, "views": views}
        jobs += [(cfg, int(i)) for i in pick]
    with mp.get_context("fork").Pool(min(a.workers, len(jobs))) as pool:
        res = pool.map(_one, jobs)
    for r in res:
        print(json.dumps(r))
    json.dump({"what": __doc__.split("\n\n")[0], "views": res}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
