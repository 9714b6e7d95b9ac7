"""Where does the e2e (host-buffer) step's time go?  C3, 64 views."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2503_08217_b200 import s3r
from paper_2503_08217_b200 import scenegen as sg

scene, views = sg.make_config("av2", n_views=64)
ctx = s3r.Context(0)
ds = s3r.DeviceScene.from_numpy(scene)
tabs = s3r.view_tables(ctx, views)
outs = s3r.alloc_outputs(views, depth=False, final_T=False)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
hs = scene.copy()
for k in ("means_opacity", "scales", "rotations", "colors", "instance_ids", "visibility", "life"):
    setattr(hs, k, pin(getattr(hs, k)))
htabs = [t.cpu().pin_memory().numpy() for t in tabs]
hout = [{"rgb": torch.empty((v.height, v.width, 3), dtype=torch.float32, pin_memory=True).numpy()}
        for v in views]
hrgb = [torch.from_numpy(h["rgb"]) for h in hout]

def timeit(f, n=4):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3

print("device render      %.1f ms" % timeit(lambda: ctx.render_batch(ds, views, list(tabs), outs)))
def d2h():
    for o, h in zip(outs, hrgb):
        h.copy_(o["rgb"], non_blocking=True)
print("D2H rgb (64 views) %.1f ms" % timeit(d2h))
print("host render (API)  %.1f ms" % timeit(lambda: ctx.render_batch_host(hs, views, htabs, hout)))
for nv in (8, 16, 32):
    print(f"host render {nv} views %.1f ms" % timeit(
        lambda: ctx.render_batch_host(hs, views[:nv], htabs[:nv], hout[:nv])))
s = torch.cuda.Stream()
print("host render, own stream %.1f ms" % timeit(
    lambda: ctx.render_batch_host(hs, views, htabs, hout, stream=s)))
cs = torch.cuda.Stream()
def overlap():
    with torch.cuda.stream(cs):
        for o, h in zip(outs[:32], hrgb[:32]):
            h.copy_(o["rgb"], non_blocking=True)
    ctx.render_batch(ds, views, list(tabs), outs, stream=s)
print("torch D2H(32) || device render: %.1f ms" % timeit(overlap))
