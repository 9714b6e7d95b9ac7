"""The README.md Python usage example, runnable as is on a B200 (checked by hand)."""
import sys, os
sys.path.insert(0, os.getcwd())

import torch
from paper_2503_08217_b200 import s3r, scenegen as sg

scene, views = sg.make_config("av2", n_views=16)     # or your own arrays (see s3r.DeviceScene)
ctx = s3r.Context(0)
ds = s3r.DeviceScene.from_numpy(scene)               # SoA float4 arrays on the GPU
tables = s3r.view_tables(ctx, views)                 # per-instance local->camera 3x4
outs = s3r.alloc_outputs(views)                      # rgb, depth, final_T, visible per view
ctx.render_batch(ds, views, list(tables), outs)      # point life updated in ds.life
ctx.commit_visibility(ds, 0.1)                       # end of a sweep (Eq.6)

ctx.set_training(True)                               # config 5
ctx.render_batch(ds, views, list(tables), outs)
grads = {k: torch.zeros_like(getattr(ds, k)) for k in ("means_opacity", "scales", "rotations", "colors")}
ctx.render_backward(ds, views, list(tables), [{"rgb": torch.ones_like(o["rgb"])} for o in outs], grads)

print('readme ok', float(grads['means_opacity'].abs().sum()))
