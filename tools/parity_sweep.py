"""Full-size parity sweep: the bench's batches (C3 av2, C4 drive, C2 street, in
the launch configuration bench.py times: all of a config's views in one
s3r_render_batch) against the CPU oracle on K sampled views each (C2: all 100), element by
element — temporal list, fp32 keys, decisions, rectangles, M_t, depth order,
(tile, Gaussian) pairs, tile ranges, images.  The oracle renders run in forked
worker processes on the host cores, each comparing its view against the GPU
dumps taken before the fork; and every view of the batch rendered again on the
product path (no dumps, capacity mode) must equal the checked render bit for
bit.  Writes a JSON summary (default profiles/r02_parity_sweep.json).  Test infrastructure: needs a B200.

    python tools/parity_sweep.py [OUT.json] [--views K]
"""
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

_G = {}


def _compare(vi):
    import oracle
    scene, view, table, gpu = _G["scene"], _G["views"][vi], _G["tabs"][vi], _G["gpu"][vi]
    t0 = time.perf_counter()
    o = oracle.render_view(scene, view, "f32")       # the oracle composes its own table
    dt = time.perf_counter() - t0
    d, st, out = gpu["dump"], gpu["stats"], gpu["out"]
    ti = o["temporal_idx"]
    r = {"view": int(vi), "oracle_s": round(dt, 2)}
    r["counts_equal"] = all(int(st[k]) == int(o["stats"][k]) for k in
                            ("n_temporal", "n_visible", "n_lod_small", "n_lod_dropped",
                             "n_rendered", "n_pairs"))
    r["temporal_idx_equal"] = bool(np.array_equal(d["temporal_idx"], ti))
    same_len = len(d["temporal_idx"]) == len(ti)
    r["keys_bit_mismatches"] = int((~((d["keys"] == o["keys"][ti]) |
                                      (np.isnan(d["keys"]) & np.isnan(o["keys"][ti])))).sum()) \
        if same_len else -1
    r["flags_equal"] = bool(same_len and np.array_equal(d["flags"], o["flags"][ti]))
    r["rect_equal"] = bool(same_len and np.array_equal(d["rect"], o["rect"][ti]))
    r["visible_equal"] = bool(np.array_equal(out["visible"], o["visible"]))
    import oracle as orc
    rend = np.nonzero(o["flags"] & orc.F_RENDERED)[0]
    want = rend[np.lexsort((rend, o["splat_keys"][rend, 2]))]
    r["depth_order_equal"] = bool(np.array_equal(d["depth_order"], want))
    r["pairs_equal"] = bool(np.array_equal(d["pair_tile"], o["pair_tile"]) and
                            np.array_equal(d["pair_gauss"], o["pair_gauss"]))
    cg = d["ranges"][:, 1] - d["ranges"][:, 0]
    co = o["ranges"][:, 1] - o["ranges"][:, 0]
    ne = co > 0
    r["ranges_equal"] = bool(np.array_equal(cg, co) and np.array_equal(d["ranges"][ne], o["ranges"][ne]))
    for k in ("rgb", "depth", "final_T"):
        r[f"{k}_max_abs"] = float(np.abs(out[k] - o[k]).max())
        r[f"{k}_bit_equal"] = bool(np.array_equal(out[k], o[k]))
    r["n_rendered"] = int(o["stats"]["n_rendered"])
    r["n_pairs"] = int(o["stats"]["n_pairs"])
    return r


def main():
    import torch
    import oracle
    from paper_2503_08217_b200 import s3r, scenegen as sg
    out_path = os.path.join(ROOT, "profiles", "r02_parity_sweep.json")
    k_views = 8
    args = sys.argv[1:]
    if "--views" in args:
        i = args.index("--views")
        k_views = int(args[i + 1])
        del args[i:i + 2]
    if args:
        out_path = args[0]
    oracle.lib()
    cores = len(os.sched_getaffinity(0))
    result = {"what": __doc__.split("\n\n")[0], "cores": cores, "configs": {}}
    for cfg in ("av2", "drive", "street"):
        scene, views = sg.make_config(cfg)
        ctx = s3r.Context(0)
        ctx.set_debug(True)
        ds = s3r.DeviceScene.from_numpy(scene)
        tabs = s3r.view_tables(ctx, views)
        outs = s3r.alloc_outputs(views, n_visible=scene.n)
        t0 = time.perf_counter()
        ctx.render_batch(ds, views, list(tabs), outs)
        torch.cuda.synchronize()
        assert ctx.check() == 0
        gpu_s = time.perf_counter() - t0
        rng = np.random.default_rng(7)
        kv = len(views) if cfg == "street" else k_views      # C2: every view
        pick = sorted(rng.choice(len(views), min(kv, len(views)), replace=False).tolist())
        gpu = {}
        for vi in pick:
            v = views[vi]
            dump = {k: t.cpu().numpy() for k, t in ctx.dump(vi, v.width, v.height).items()}
            gpu[vi] = {"dump": dump, "stats": ctx.stats(vi),
                       "out": {k: outs[vi][k].cpu().numpy() for k in
                               ("rgb", "depth", "final_T", "visible")}}
        _G.update(scene=scene, views=views, tabs=[t.cpu().numpy() for t in tabs], gpu=gpu)
        ctx.close()
        # the product path (no debug dumps: the lean K2; the capacity mode sized
        # from this batch, as bench.py runs it) must give every view's images
        # and M_t bit for bit
        pctx = s3r.Context(0)
        pds = s3r.DeviceScene.from_numpy(scene)
        ptabs = list(s3r.view_tables(pctx, views))
        pouts = s3r.alloc_outputs(views, n_visible=scene.n)
        pctx.render_batch(pds, views, ptabs, pouts)          # sizes the reservation
        pctx.set_capacity(pctx.capacity_from_last(1.1))
        pds = s3r.DeviceScene.from_numpy(scene)
        pouts = s3r.alloc_outputs(views, n_visible=scene.n)
        pctx.render_batch(pds, views, ptabs, pouts)
        torch.cuda.synchronize()
        product_ok = pctx.check() == 0 and all(
            torch.equal(outs[i][k], pouts[i][k]) for i in range(len(views))
            for k in ("rgb", "depth", "final_T", "visible"))
        pctx.close()
        del pouts, pds
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(min(cores, len(pick))) as pool:
            per = pool.map(_compare, pick)
        wall = time.perf_counter() - t0
        bool_keys = [k for k in per[0] if isinstance(per[0][k], bool)]
        summary = {k: all(p[k] for p in per) for k in bool_keys}
        summary["product_path_all_views_bit_equal"] = bool(product_ok)
        summary.update(keys_bit_mismatches=sum(p["keys_bit_mismatches"] for p in per),
                       rgb_max_abs=max(p["rgb_max_abs"] for p in per),
                       depth_max_abs=max(p["depth_max_abs"] for p in per),
                       final_T_max_abs=max(p["final_T_max_abs"] for p in per))
        result["configs"][cfg] = {"n_gaussians": scene.n, "views_in_batch": len(views),
                                  "views_checked": pick, "image": f"{views[0].width}x{views[0].height}",
                                  "gpu_batch_s_with_debug": round(gpu_s, 2),
                                  "oracle_wall_s": round(wall, 1), "summary": summary,
                                  "per_view": per}
        print(cfg, json.dumps(summary), flush=True)
        _G.clear()
    json.dump(result, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
