import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle
from paper_2503_08217_b200 import s3r, scenegen as sg
from helpers import make_scene, make_view

ctx = s3r.Context(0)
def run(scene, views, cot):
    ds = s3r.DeviceScene.from_numpy(scene)
    tabs = s3r.view_tables(ctx, views)
    outs = s3r.alloc_outputs(views)
    ctx.set_training(True)
    ctx.render_batch(ds, views, list(tabs), outs)
    cots = [{k: torch.from_numpy(np.ascontiguousarray(c[k], np.float32)).cuda() for k in c} for c in cot]
    grads = {k: torch.zeros_like(getattr(ds, k)) for k in ("means_opacity", "scales", "rotations", "colors")}
    ctx.render_backward(ds, views, list(tabs), cots, grads)
    torch.cuda.synchronize()
    g = np.concatenate([grads[k].cpu().numpy() for k in ("means_opacity", "scales", "rotations", "colors")], 1)
    ref = np.zeros((scene.n, 16))
    for v, t, c in zip(views, tabs, cot):
        oracle.backward(scene, v, c["rgb"], c.get("depth"), c.get("final_T"), table=t.cpu().numpy(), grads=ref)
    for i, name in enumerate(["mx","my","mz","op","sx","sy","sz","-","qw","qx","qy","qz","r","g","b","-"]):
        r = np.abs(ref[:, i]).max()
        d = np.abs(g[:, i] - ref[:, i]).max()
        print(f"{name}: ref {r:.4g} diff {d:.4g} rel {d/max(r,1e-30):.3g}")
    return g, ref

# single Gaussian, identity camera
s = make_scene([[0.1, -0.05, 3.0]], [[0.05, 0.08, 0.04]], quats=[[0.9, 0.1, 0.3, 0.2]], opacity=0.5, rgb=[[0.2, 0.5, 0.8]])
v = make_view(80.0, 32.0, 64, 48, cy=24.0)
rng = np.random.default_rng(0)
print("== single, rgb cot only")
run(s, [v], [{"rgb": rng.standard_normal((48, 64, 3))}])
print("== single, depth only")
run(s, [v], [{"rgb": np.zeros((48, 64, 3)), "depth": rng.standard_normal((48, 64))}])
print("== two overlapping")
s = make_scene([[0.1, -0.05, 3.0], [0.12, 0.0, 4.0]], [[0.05, 0.08, 0.04], [0.1, 0.1, 0.1]], opacity=[0.5, 0.6], rgb=[[0.2, 0.5, 0.8], [0.9, 0.1, 0.3]])
run(s, [v], [{"rgb": rng.standard_normal((48, 64, 3)), "final_T": rng.standard_normal((48,64))}])
