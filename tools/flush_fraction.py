"""Fraction of a full-size C3 view's tile-pixel evaluations that are flushed (e2 < -24)
and how many remain at warp-block / half-block / quarter-block culling granularity
(oracle keys, numpy).  DESIGN.md §7.  PYTHONPATH=. python tools/flush_fraction.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, oracle, time
from paper_2503_08217_b200 import scenegen as sg
scene, views = sg.make_config("av2")
v = views[10]
o = oracle.render_view(scene, v, "f32")
k = o["splat_keys"].astype(np.float64)
a_, b_, c_ = k[:,3]+0.3, k[:,4], k[:,5]+0.3
det = a_*c_ - b_*b_
with np.errstate(all='ignore'):
    A, B, C = c_/det, -b_/det, a_/det
LOG2E = 1.4426950408889634
qa, qb, qc = -0.5*A*LOG2E, -B*LOG2E, -0.5*C*LOG2E
TX = (v.width+15)//16
pt, pg = o["pair_tile"], o["pair_gauss"]
ly, lx = np.divmod(np.arange(256), 16)
tot = 0; live_px = 0; live_wb = 0; live_hb = 0; live_qb = 0
t0=time.time()
for s in range(0, len(pt), 20000):
    t = pt[s:s+20000]; g = pg[s:s+20000]
    px = (t % TX)[:,None]*16 + lx[None,:]; py = (t // TX)[:,None]*16 + ly[None,:]
    dx = k[g,0][:,None] - px; dy = k[g,1][:,None] - py
    e2 = qa[g][:,None]*dx*dx + qb[g][:,None]*dx*dy + qc[g][:,None]*dy*dy
    on = e2 >= -24
    tot += on.size; live_px += on.sum()
    on4 = on.reshape(-1, 16, 16)   # [pair, row, col]
    # warp blocks: 8 cols x 16 rows (2 per tile)
    wb = on4.reshape(-1,16,2,8).any(axis=(1,3)); live_wb += wb.sum()*128
    # half blocks 8x8 (pair rows 0-7 / 8-15 of a warp block)
    hb = on4.reshape(-1,2,8,2,8).any(axis=(2,4)); live_hb += hb.sum()*64
    # quarter blocks 8x4
    qb4 = on4.reshape(-1,4,4,2,8).any(axis=(2,4)); live_qb += qb4.sum()*32
print("pairs", len(pt), "evals (tile pixels)", tot, "unflushed %.3f" % (live_px/tot),
      "executed at 8x16 warp blocks %.3f, 8x8 %.3f, 8x4 %.3f" % (live_wb/tot, live_hb/tot, live_qb/tot), time.time()-t0)
