"""Build raster variants (tools/ab_raster.py build) and time them on a GPU
(tools/ab_raster.py run): one bench.py run per variant, stage times printed."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VARIANTS = {
    "base": [],
    "flush32": ["S3R_FLUSH_E2=-32.0f"],
    "flush24": ["S3R_FLUSH_E2=-24.0f"],
    "flush20": ["S3R_FLUSH_E2=-20.0f"],
}

if __name__ == "__main__":
    if sys.argv[1] == "build":
        from paper_2503_08217_b200 import build as B
        for name, d in VARIANTS.items():
            print(B.build_variant(name, d))
    else:
        for name in VARIANTS:
            env = dict(os.environ, S3R_LIB=os.path.join(ROOT, "paper_2503_08217_b200",
                                                        f"libs3r_{name}.so"))
            r = subprocess.run([sys.executable, "bench.py", "--steps", "5", "--warmup", "3",
                                "--no-e2e", "--no-cpu-baseline"], cwd=ROOT, env=env,
                               capture_output=True, text=True, timeout=400)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])
                print(name, round(d["value"], 1), {k: round(v["ms"], 3) for k, v in d["stages"].items()},
                      flush=True)
            except Exception:
                print(name, "FAILED", r.stderr[-500:], flush=True)
