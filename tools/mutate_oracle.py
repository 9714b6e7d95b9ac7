"""Mutation check of the oracle's pins: each mutant below
is a plausible mistake in the Eq.2 edge rules (reading R14: alpha clamp 0.99,
include-then-stop at T < 1e-4) or in their adjoint, or (MUTANTS_PATH) in the
other steps of the path: the temporal filter, the projection, the decisions,
the adaptive LOD and the point life / commit.  For each one the repo is
copied to a scratch directory, the mutation applied to oracle/, liboracle.so
rebuilt, and the CPU oracle pins run; a mutant must make at least one pin fail (all failing pins are recorded).

    python tools/mutate_oracle.py [--out profiles/r02_oracle_mutants.json]
"""
import argparse
import json
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
IMPL = "oracle/s3r_oracle_impl.inc"
BWD = "oracle/s3r_oracle_bwd.c"

EXP2_W = "        REAL w = alpha * T;\n        Cr = FMA(q->r, w, Cr);"
MUTANTS = {
    # forward (both precisions: the f32 contract and the f64 shadow)
    "fwd_threshold_1e-3": [(IMPL, "if (T < R(1e-4)) break;", "if (T < R(1e-3)) break;", 2)],
    "fwd_threshold_2e-4": [(IMPL, "if (T < R(1e-4)) break;", "if (T < R(2e-4)) break;", 2)],
    "fwd_stop_before_include": [
        (IMPL, "        REAL alpha = FMIN(R(0.99), q->o * so_exp2_f32(e2));\n        REAL w = alpha * T;\n",
         "        REAL alpha = FMIN(R(0.99), q->o * so_exp2_f32(e2));\n        REAL w = alpha * T;\n"
         "        if (T - w < R(1e-4)) break;\n", 1),
        (IMPL, "        REAL alpha = FMIN(R(0.99), q->o * EXPF(power));\n        REAL w = alpha * T;\n",
         "        REAL alpha = FMIN(R(0.99), q->o * EXPF(power));\n        REAL w = alpha * T;\n"
         "        if (T * (R(1.0) - alpha) < R(1e-4)) break;\n", 1)],
    "fwd_no_termination": [(IMPL, "if (T < R(1e-4)) break;", "if (T < R(0.0)) break;", 2)],
    "fwd_no_alpha_clamp": [
        (IMPL, "FMIN(R(0.99), q->o * so_exp2_f32(e2))", "(q->o * so_exp2_f32(e2))", 1),
        (IMPL, "FMIN(R(0.99), q->o * EXPF(power))", "(q->o * EXPF(power))", 1)],
    "fwd_alpha_clamp_0.999": [
        (IMPL, "FMIN(R(0.99), q->o * so_exp2_f32(e2))", "FMIN(R(0.999), q->o * so_exp2_f32(e2))", 1),
        (IMPL, "FMIN(R(0.99), q->o * EXPF(power))", "FMIN(R(0.999), q->o * EXPF(power))", 1)],
    "fwd_flush_below_-20": [(IMPL.replace("impl.inc", "f32.c"), "if (!(x >= -24.0f)) return 0.0f;",
                              "if (!(x >= -20.0f)) return 0.0f;", 1)],
    # adjoint (fp64)
    "bwd_clamp_passes_gradient": [(BWD, "if (q->o * G >= 0.99) continue;", "if (0) continue;", 1)],
    "bwd_threshold_1e-3": [(BWD, "if (T < 1e-4) break;", "if (T < 1e-3) break;", 1)],
    "bwd_stop_before_include": [
        (BWD, "                T = T * (1.0 - a);\n                last = i + 1;\n",
         "                if (T * (1.0 - a) < 1e-4) break;\n                T = T * (1.0 - a);\n"
         "                last = i + 1;\n", 1)],
    "bwd_no_termination": [(BWD, "if (T < 1e-4) break;", "if (T < 0.0) break;", 1)],
}
F32C = "oracle/s3r_oracle_f32.c"
# the other steps of the path: filter (a1), projection (a2, Eq.1), decisions,
# adaptive LOD (a3, Eq.7 rows 1-3), point life and commit (a6, Eq.5 / Eq.6)
MUTANTS_PATH = {
    "filter_exclusive_upper": [(IMPL, "if (vs <= t && t <= ve) {", "if (vs <= t && t < ve) {", 1)],
    "filter_exclusive_lower": [(IMPL, "if (vs <= t && t <= ve) {", "if (vs < t && t <= ve) {", 1)],
    "proj_rotation_sign": [(IMPL, "Rq[1] = R(2.0) * (xy - wz);", "Rq[1] = R(2.0) * (xy + wz);", 1)],
    "proj_jacobian_sign": [(IMPL, "REAL j02 = -((fx * uc) / pz);", "REAL j02 = ((fx * uc) / pz);", 1)],
    "proj_tangent_clamp_1.3": [(IMPL, "REAL hix = ((R(1.15) * Wf) - cx) / fx;",
                                "REAL hix = ((R(1.3) * Wf) - cx) / fx;", 1)],
    "proj_mean_uses_fy": [(IMPL, "keys[0] = FMA(fx, u, cx);", "keys[0] = FMA(fy, u, cx);", 1)],
    "decide_no_dilation": [(IMPL, "REAL ad = a + R(0.3);\n    REAL cd = c + R(0.3);",
                            "REAL ad = a + R(0.0);\n    REAL cd = c + R(0.0);", 1)],
    "decide_conic_b_sign": [(IMPL, "d->conB = (-b) / det;", "d->conB = b / det;", 1)],
    "decide_radius_2sigma": [(IMPL, "REAL rf = CEIL(R(3.0) * SQRT(lamd));",
                              "REAL rf = CEIL(R(2.0) * SQRT(lamd));", 1)],
    "lod_scale_of_dilated": [(IMPL, "REAL sc = SO(so_scale2d)(k[3], k[5], d.disc);",
                              "REAL sc = SO(so_scale2d)(k[3] + R(0.3), k[5] + R(0.3), d.disc);", 1)],
    "lod_slope_sign": [(IMPL, "REAL p = FMA(pmax - R(0.01), m, pmax);",
                        "REAL p = FMA(pmax + R(0.01), m, pmax);", 1)],
    "lod_far_side": [(IMPL, "REAL m = FMIN(R(0.0), (d - D) / D);", "REAL m = FMAX(R(0.0), (d - D) / D);", 1)],
    "lod_drop_inverted": [(IMPL, "if (uu < p) {", "if (uu >= p) {", 1)],
    "life_start_max": [(F32C, "if (t < s->life[2 * g + 0]) s->life[2 * g + 0] = t;",
                        "if (t > s->life[2 * g + 0]) s->life[2 * g + 0] = t;", 1)],
    "commit_no_margin": [(F32C, "s->visibility[2 * g + 0] = fmaxf(-1.0f, ls - margin);",
                          "s->visibility[2 * g + 0] = fmaxf(-1.0f, ls);", 1)],
    "commit_single_observation_unseen": [(F32C, "if (ls > le) {", "if (ls >= le) {", 1)],
    # tile binning and depth order (a4, reading R11 / R12)
    "order_ties_descending_index": [(IMPL, "if (a->g != b->g) return a->g < b->g ? -1 : 1;",
                                     "if (a->g != b->g) return a->g > b->g ? -1 : 1;", 1)],
    "order_back_to_front": [(IMPL, "if (a->z != b->z) return a->z < b->z ? -1 : 1;",
                             "if (a->z != b->z) return a->z > b->z ? -1 : 1;", 1)],
    "rect_last_tile_dropped": [(IMPL, "d->tx1 = x1 / SO_TILE;", "d->tx1 = (x1 - 1) / SO_TILE;", 1)],
    "rect_box_floor_low": [(IMPL, "REAL xlo = CEIL(mx - rf), xhi = FLOOR(mx + rf);",
                            "REAL xlo = FLOOR(mx - rf), xhi = FLOOR(mx + rf);", 1)],
    # R-ARITH exp2, instance cameras, adjoint terms, NEXT-3 noisy
    # offset scale (R10), NEXT-4 NeurF features and layers (R22)
    "exp2_coefficient": [(F32C, "p = fmaf(p, r, 5.550733208656311e-2f);",
                          "p = fmaf(p, r, 5.6e-2f);", 1)],
    "exp2_exponent_off_by_one": [(F32C, "return ldexpf(y, (int)n);", "return ldexpf(y, (int)n - 1);", 1)],
    "compose_rotation_transposed": [(F32C, "double acc = a0 * (double)B[0 * 4 + c];",
                                     "double acc = a0 * (double)B[c * 4 + 0];", 1)],
    "compose_translation_term_dropped": [(F32C, "double acc = fma(a0, (double)B[0 * 4 + 3], a3);",
                                          "double acc = a3;", 1)],
    "bwd_conic_b_sign": [(BWD, "q->gB += -dx * dy * gP;", "q->gB += dx * dy * gP;", 1)],
    "bwd_mean_cross_term_dropped": [(BWD, "q->gmx += -(q->A * dx + q->B * dy) * gP;",
                                     "q->gmx += -(q->A * dx) * gP;", 1)],
    "jitter_depth_scale_max": [(IMPL, "REAL nd = FMIN(R(1.0), k[2] / (REAL)v->lod_D);",
                                "REAL nd = FMAX(R(1.0), k[2] / (REAL)v->lod_D);", 1)],
    "neurf_no_relu": [("oracle/neurf.py", "h1 = np.maximum(fb[sel] @ W1.T + b1, 0.0)",
                       "h1 = (fb[sel] @ W1.T + b1)", 1)],
    "neurf_frequency_without_pi": [("oracle/neurf.py", "arg = (2.0 ** l) * np.pi * m[:, a]",
                                    "arg = (2.0 ** l) * m[:, a]", 1)],
}
MUTANTS.update(MUTANTS_PATH)
TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_backward.py", "tests/test_oracle_jitter.py",
         "tests/test_oracle_neurf.py", "tests/test_oracle_conventional.py"]


def run_mutant(name, edits):
    tmp = tempfile.mkdtemp(prefix="s3r_mut_")
    try:
        for d in ("oracle", "tests", "paper_2503_08217_b200"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("*.so", "__pycache__", "build"))
        for path, old, new, count in edits:
            p = os.path.join(tmp, path)
            src = open(p).read()
            assert src.count(old) == count, (name, path, src.count(old))
            open(p, "w").write(src.replace(old, new))
        subprocess.run(["make", "-s", "-B", "liboracle.so"], cwd=os.path.join(tmp, "oracle"),
                       check=True)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "not gpu",
                            "-p", "no:cacheprovider", *TESTS], cwd=tmp, capture_output=True,
                           text=True, timeout=3000)
        failed = [ln.split(" ")[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
        return {"killed": r.returncode != 0, "failures": failed, "rc": r.returncode}
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_oracle_mutants.json"))
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    res = {}
    for name, edits in MUTANTS.items():
        if a.only and a.only not in name:
            continue
        res[name] = run_mutant(name, edits)
        print(name, res[name], flush=True)
    json.dump({"tests": TESTS, "mutants": res}, open(a.out, "w"), indent=1)
    survivors = [k for k, v in res.items() if not v["killed"]]
    print("survivors:", survivors)
    sys.exit(1 if survivors else 0)


if __name__ == "__main__":
    main()
