"""Build kernel variants (tools/ab_raster.py build SET) and time them on a GPU
(tools/ab_raster.py run SET): one bench.py run per variant, stage times and the
config-5 training step printed.  SET names one of the dicts in VARIANT_SETS."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VARIANT_SETS = {
    "r2scat": {
        "base": [],
        "scatmask": ["S3R_SCATTER_MASK=1"],
    },
    "r2occ": {
        "base": [],
        "m18rb192": ["S3R_RASTER_MINB=18", "S3R_RASTER_RB=192"],
        "m20rb160": ["S3R_RASTER_MINB=20", "S3R_RASTER_RB=160"],
        "m20rb128": ["S3R_RASTER_MINB=20", "S3R_RASTER_RB=128"],
        "m16rb192": ["S3R_RASTER_RB=192"],
    },
    "r2smem": {
        "base": [],
        "scot14": ["S3R_BWD_SMEMCOT=1"],
        "scot16": ["S3R_BWD_SMEMCOT=1", "S3R_BWD_MINB=16"],
        "scot18": ["S3R_BWD_SMEMCOT=1", "S3R_BWD_MINB=18", "S3R_BWD_RB=128"],
        "scot20": ["S3R_BWD_SMEMCOT=1", "S3R_BWD_MINB=20", "S3R_BWD_RB=128"],
        "rb128": ["S3R_BWD_RB=128"],
    },
    "r2bwd": {
        "base": [],
        "stage0": ["S3R_RASTER_STAGE=0"],
        "vred": ["S3R_BWD_VRED=1"],
        "ulast": ["S3R_BWD_ULAST=1"],
        "vredulast": ["S3R_BWD_VRED=1", "S3R_BWD_ULAST=1"],
    },
    "r2raster": {
        "base": [],
        "fastlive": ["S3R_RASTER_FASTLIVE=1"],
        "uvote": ["S3R_RASTER_UVOTE=1"],
        "aluexp": ["S3R_RASTER_ALUEXP=1"],
        "flalu": ["S3R_RASTER_FASTLIVE=1", "S3R_RASTER_ALUEXP=1"],
        "fluvalu": ["S3R_RASTER_FASTLIVE=1", "S3R_RASTER_UVOTE=1", "S3R_RASTER_ALUEXP=1"],
        "stage1": ["S3R_RASTER_STAGE=1"],
        "stage2": ["S3R_RASTER_STAGE=2"],
    },
    "flush": {
        "base": [],
        "flush32": ["S3R_FLUSH_E2=-32.0f"],
        "flush20": ["S3R_FLUSH_E2=-20.0f"],
    },
    "minb": {
        "base": [],
        "minb12": ["S3R_RASTER_MINB=12"],
        "minb14": ["S3R_RASTER_MINB=14"],
        "minb16": ["S3R_RASTER_MINB=16"],
    },
    "mb": {
        "base": [],
        "minb14": ["S3R_RASTER_MINB=14"],
        "minb15": ["S3R_RASTER_MINB=15"],
    },
    "live": {
        "base": [],
        "live1": ["S3R_LIVE_EVERY=1"],
        "live8": ["S3R_LIVE_EVERY=8"],
        "live0": ["S3R_LIVE_EVERY=0"],
        "live0_mb0": ["S3R_LIVE_EVERY=0", "S3R_RASTER_MINB=0"],
    },
    "cull": {
        "base": [],
        "nocull": ["S3R_CULL=0"],
    },
    "clist": {
        "base": [],
        "adj": ["S3R_RASTER_ADJ=1"],
    },
    "mufu": {
        "base": [],
        "mufu": ["S3R_RASTER_MUFU=1"],
    },
    "ov": {
        "base": [],
        "ov": [],
    },
    "rpr": {
        "base": [],
        "noadj": ["S3R_BWD_ADJ=0"],
    },
    "bex": {
        "base": [],
        "ex2pair": ["S3R_BWD_EX2=2"],
        "exact": ["S3R_BWD_EX2=0"],
    },
    "k2": {
        "base": [],
        "k2m5": ["S3R_K2_MINB=5"],
        "k2m6": ["S3R_K2_MINB=6"],
    },
    "fwd8": {
        "base": [],
        "f8m20": ["S3R_RASTER_RPIX=8", "S3R_RASTER_MINB=20"],
        "f8m24": ["S3R_RASTER_RPIX=8", "S3R_RASTER_MINB=24"],
        "f8m32": ["S3R_RASTER_RPIX=8", "S3R_RASTER_MINB=32"],
    },
    "bwd8": {
        "base": [],
        "rp8m16": ["S3R_BWD_RPIX=8", "S3R_BWD_MINB=16"],
        "rp8m20": ["S3R_BWD_RPIX=8", "S3R_BWD_MINB=20"],
        "rp8m24": ["S3R_BWD_RPIX=8", "S3R_BWD_MINB=24"],
    },
    "front": {
        "base": [],
        "noprecull": ["S3R_K2_PRECULL=0"],
        "k2m3": ["S3R_K2_MINB=3"],
        "k2m5": ["S3R_K2_MINB=5"],
    },
    "bin": {
        "base": [],
        "scat0": ["S3R_SCATTER_MASK=0"],
    },
    "nobr": {
        "base": [],
        "bnobr": ["S3R_BWD_NOBR=1"],
        "bnobr_m16": ["S3R_BWD_NOBR=1", "S3R_BWD_MINB=16"],
        "fnobr": ["S3R_RASTER_NOBR=1"],
    },
    "nobr2": {
        "base": [],
        "m16": ["S3R_BWD_MINB=16"],
        "bnobr_m16": ["S3R_BWD_NOBR=1", "S3R_BWD_MINB=16"],
        "bnobr_m14": ["S3R_BWD_NOBR=1", "S3R_BWD_MINB=14"],
        "bnobr_m12": ["S3R_BWD_NOBR=1", "S3R_BWD_MINB=12"],
        "bnobr_m18": ["S3R_BWD_NOBR=1", "S3R_BWD_MINB=18"],
    },
    "bmb": {
        "base": [],
        "m13": ["S3R_BWD_MINB=13"],
        "m15": ["S3R_BWD_MINB=15"],
        "m16": ["S3R_BWD_MINB=16"],
    },
    "rpr2": {
        "base": [],
        "rpr2": ["S3R_BWD_RPR=2"],
        "rpr2m12": ["S3R_BWD_RPR=2", "S3R_BWD_MINB=12"],
        "rpr2m10": ["S3R_BWD_RPR=2", "S3R_BWD_MINB=10"],
    },
    "bin2": {
        "base": [],
        "xpf1": ["S3R_XPF=1"],
        "xpf2": ["S3R_XPF=2"],
        "scat1d": ["S3R_SCAT2D=0"],
        "xpf1_scat1d": ["S3R_XPF=1", "S3R_SCAT2D=0"],
    },
    "vote": {
        "base": [],
        "vote2": ["S3R_VOTE_EVERY=2"],
        "vote4": ["S3R_VOTE_EVERY=4"],
        "xt128": ["S3R_XT=128"],
    },
    "k2pr": {
        "base": [],
        "pr2": ["S3R_K2_PR=2"],
        "pr8": ["S3R_K2_PR=8"],
        "pr2m6": ["S3R_K2_PR=2", "S3R_K2_MINB=6"],
    },
    "trainmb": {
        "base": [],
        "tmb14": ["S3R_RASTER_TRAIN_MINB=14"],
        "tmb12": ["S3R_RASTER_TRAIN_MINB=12"],
    },
    "sort": {
        "base": [],
        "it4": ["S3R_SORT_ITEMS=4"],
        "mb3": ["S3R_SORT_MINB=3"],
        "mb4": ["S3R_SORT_MINB=4"],
        "it4mb6": ["S3R_SORT_ITEMS=4", "S3R_SORT_MINB=6"],
    },
    "split": {
        "base": [],
        "nosplit": ["S3R_K2_SPLIT=0"],
        "k2a4": ["S3R_K2A_MINB=4"],
        "k2a8": ["S3R_K2A_MINB=8"],
    },
    "bex2": {
        "base": [],
        "ex2a": ["S3R_BWD_EX2=1"],
        "ex2b": ["S3R_BWD_EX2=2"],
    },
    "lmask": {
        "base": [],
        "lmask0": ["S3R_LMASK=0"],
    },
    "fnobr": {
        "base": [],
        "fnobr": ["S3R_RASTER_NOBR=1"],
        "fnobr14": ["S3R_RASTER_NOBR=1", "S3R_RASTER_MINB=14"],
        "fnobr12": ["S3R_RASTER_NOBR=1", "S3R_RASTER_MINB=12"],
    },
    "persist": {
        "base": [],
        "persist": ["S3R_RASTER_PERSIST=1"],
    },
    "frange": {
        "base": [],
        "frange0": ["S3R_FILTER_RANGE=0"],
    },
    "rowskip": {
        "base": [],
        "rowskip": ["S3R_BWD_ROWSKIP=1"],
    },
    "xt": {
        "base": [],
        "xt32": ["S3R_XT=32"],
        "xt64": ["S3R_XT=64"],
    },
    "rmb": {
        "base": [],
        "rm14": ["S3R_RASTER_MINB=14"],
        "rm12": ["S3R_RASTER_MINB=12"],
    },
    "pose": {
        "base": [],
        "pg1": ["S3R_POSE_GROUPS=1"],
        "pg8": ["S3R_POSE_GROUPS=8"],
    },
    "lean": {
        "base": [],
        "lean1": ["S3R_RASTER_LEAN=1"],
        "lean3": ["S3R_RASTER_LEAN=3"],
        "lean7": ["S3R_RASTER_LEAN=7"],
    },
    "xm": {
        "base": [],
        "xm2": ["S3R_XMASK=2"],
    },
    "hyb": {
        "base": [],
        "hyb": ["S3R_SCAT_HYBRID=1"],
        "hyb16": ["S3R_SCAT_HYBRID=1", "S3R_SCAT_SMALL=16"],
        "hyb4": ["S3R_SCAT_HYBRID=1", "S3R_SCAT_SMALL=4"],
    },
    "hyb2": {
        "hyb16": ["S3R_SCAT_HYBRID=1", "S3R_SCAT_SMALL=16"],
        "hyb24": ["S3R_SCAT_HYBRID=1", "S3R_SCAT_SMALL=24"],
        "hyb32": ["S3R_SCAT_HYBRID=1", "S3R_SCAT_SMALL=32"],
    },
    "k2lean": {
        "base": [],
        "nolean": ["S3R_K2_LEAN=0"],
    },
    "xpref": {
        "base": [],
        "nopref": ["S3R_XPREF=0"],
    },
    "grpbig": {
        "base": [],
        "wb1184": ["S3R_FILTER_WANT_BIG=1184"],
        "wb2368": ["S3R_FILTER_WANT_BIG=2368"],
    },
    "half": {
        "base": [],
        "th16": ["S3R_RASTER_SMALL_TH=16"],
        "th4": ["S3R_RASTER_SMALL_TH=4"],   # C1: 18.1 k vs 18.3-18.6 k at 8
    },
    "smask": {
        "base": [],
        "nosmask": ["S3R_SMALL_MASK=0"],
    },
    "bwd": {
        "base": [],
        "bmb13": ["S3R_BWD_MINB=13"],
        "bmb14": ["S3R_BWD_MINB=14"],
        "bmb12": ["S3R_BWD_MINB=12"],
        "bmb11": ["S3R_BWD_MINB=11"],
    },
}

if __name__ == "__main__":
    cmd, vset = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "flush"
    variants = VARIANT_SETS[vset]
    if cmd == "build":
        from paper_2503_08217_b200 import build as B
        for name, d in variants.items():
            print(B.build_variant(name, d))
    else:
        for name in variants:
            env = dict(os.environ, S3R_LIB=os.path.join(ROOT, "paper_2503_08217_b200",
                                                        f"libs3r_{name}.so"))
            if name.startswith("ov"):
                env["S3R_OVERLAP"] = "1"
            r = subprocess.run([sys.executable, "bench.py", "--steps", "5", "--warmup", "3",
                                "--no-e2e", "--no-cpu-baseline", "--pool", "1",
                                "--config", os.environ.get("AB_CONFIG", "av2")] +
                               (["--no-train", "--no-neurf", "--no-conventional", "--no-fast-exp"]
                                if os.environ.get("AB_FWD_ONLY") else []), cwd=ROOT,
                               env=env, capture_output=True, text=True, timeout=400)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])
                t = d.get("train") or {}
                print(name, round(d["value"], 1),
                      {k: round(v["ms"], 3) for k, v in d["stages"].items()},
                      "train", round(t.get("value", 0), 1), "fwd", round(t.get("forward_ms", 0), 2),
                      "bwd", round(t.get("backward_ms", 0), 2), flush=True)
            except Exception:
                print(name, "FAILED", r.stderr[-800:], flush=True)
