"""Per-view cost vs scene length, streamlined vs conventional pipeline (the
paper's Fig.1c / Fig.4 claim, on B200; SURVEY.md §8(f)
NEXT-2).  The C3 (av2) rig and density, street length L in metres with the
Gaussian count, the object count and the frame count proportional to L; 32
views sampled per length.  Writes gpurun_out/scaling_sweep.json (copied to
profiles/r0N_scaling_sweep.json per round).

    python tools/scaling_sweep.py [lengths...]
"""
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2503_08217_b200 import s3r  # noqa: E402
from paper_2503_08217_b200 import scenegen as sg  # noqa: E402


def timed(ctx, ds, views, tabs, outs, conventional, reps=3):
    ctx.set_pipeline(conventional)
    try:
        ctx.render_batch(ds, views, tabs, outs)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            ctx.render_batch(ds, views, tabs, outs)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        ctx.set_counters(True)
        ctx.render_batch(ds, views, tabs, outs)
        torch.cuda.synchronize()
        st = [ctx.stats(i) for i in range(len(views))]
        ctx.set_counters(False)
    finally:
        ctx.set_pipeline(False)
    n = len(views)
    return {"ms_per_view": ms / n,
            "n_projected_per_view": sum(s["n_temporal"] for s in st) / n,
            "n_rendered_per_view": sum(s["n_rendered"] for s in st) / n,
            "n_pairs_per_view": sum(s["n_pairs"] for s in st) / n}


def main():
    lengths = [float(x) for x in sys.argv[1:]] or [100.0, 200.0, 400.0, 800.0, 1600.0]
    base = sg.CONFIGS["av2"]
    ctx = s3r.Context(0)
    rows = []
    for L in lengths:
        f = L / base.length_m
        cfg = dataclasses.replace(base, name=f"av2_L{int(L)}", n_static=int(base.n_static * f),
                                  n_objects=max(1, int(round(base.n_objects * f))),
                                  frames=max(8, int(base.frames * f)), length_m=L, n_views=32)
        t0 = time.time()
        scene, traj = sg.make_street_scene(cfg)
        views = sg.make_views(cfg, traj, n_views=32, seed=cfg.seed + 7)
        ds = s3r.DeviceScene.from_numpy(scene)
        st_tabs = list(s3r.view_tables(ctx, views))
        cv_tabs = list(s3r.conventional_tables(views))
        outs = s3r.alloc_outputs(views, depth=False, final_T=False)
        s = timed(ctx, ds, views, st_tabs, outs, False)
        c = timed(ctx, ds, views, cv_tabs, outs, True)
        row = {"length_m": L, "n_gaussians": scene.n, "instances": scene.num_instances - 1,
               "streamlined": s, "conventional": c,
               "speedup": c["ms_per_view"] / s["ms_per_view"], "gen_s": time.time() - t0}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del ds, outs
        torch.cuda.empty_cache()
    out = {"what": "per-view render time vs street length, C3 rig/density, 32 views per "
                   "length, one B200 (tools/scaling_sweep.py)", "rows": rows}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "scaling_sweep.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
