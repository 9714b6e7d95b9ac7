"""A small exercise of every kernel for compute-sanitizer (memcheck / racecheck
/ synccheck / initcheck):  compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_08217_b200 import s3r  # noqa: E402
from paper_2503_08217_b200 import scenegen as sg  # noqa: E402


def main():
    ctx = s3r.Context(0)
    ctx.set_debug(True)
    scene, views = sg.make_random_dynamic(5, 1500, 3, 120, 70, 45, 3, lod=(3.0, 0.5, 12.0))
    ds = s3r.DeviceScene.from_numpy(scene)
    tabs = list(s3r.view_tables(ctx, views))
    outs = s3r.alloc_outputs(views, n_visible=scene.n)
    ctx.render_batch(ds, views, tabs, outs)                      # K1..K7
    for i, v in enumerate(views):
        ctx.dump(i, v.width, v.height)                           # debug dumps
    ctx.commit_visibility(ds, 0.1)
    ctx.reset_visibility(ds)
    ctx.life_flip(ds.life)
    ctx.set_lod_jitter(0.2, 0.2, 0.4)                            # NEXT-3
    ctx.render_batch(ds, views, tabs, outs)
    ctx.set_lod_jitter(0.0, 0.0, 0.0)
    ctx.set_pipeline(True)                                       # NEXT-2
    ctx.render_batch(ds, views, list(s3r.conventional_tables(views)), outs)
    ctx.set_pipeline(False)
    from bench import random_neurf_params                        # NEXT-4
    ctx.set_neural_colors(random_neurf_params(scene.num_instances, torch.device("cuda")))
    ctx.render_batch(ds, views, tabs, outs)
    ctx.set_neural_colors(None)
    ctx.set_training(True)                                       # config 5
    ctx.render_batch(ds, views, tabs, outs)
    loss = torch.zeros(1, device="cuda")
    cots = []
    for o in outs:
        g = torch.empty_like(o["rgb"])
        ctx.mse(o["rgb"], torch.zeros_like(o["rgb"]), 1.0 / o["rgb"].numel(), g, loss)
        cots.append({"rgb": g})
    grads = {k: torch.zeros_like(getattr(ds, k)) for k in
             ("means_opacity", "scales", "rotations", "colors")}
    grads["table"] = torch.zeros((len(views), scene.num_instances, 12), device="cuda")
    ctx.render_backward(ds, views, tabs, cots, grads)
    ctx.set_training(False)
    hs = scene.copy()                                            # host entry point
    hout = [{"rgb": np.zeros((v.height, v.width, 3), np.float32)} for v in views]
    ctx.render_batch_host(hs, views, [t.cpu().numpy() for t in tabs], hout)
    torch.cuda.synchronize()
    print("sanitize run ok", float(loss))


if __name__ == "__main__":
    main()
