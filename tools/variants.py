"""Build libgvox kernel variants (compile-time knobs) and time each with
bench.py --linearize-only on the GPU box.  Usage (on the box):
  python tools/variants.py build   # here, CPU: compiles variants into build/variants/
  python tools/variants.py run     # on the GPU: times each variant
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_2407_10344_b200", "build", "variants")
VARIANTS = {
    # linearize kernel (C5, r01 results in k_linearize.cu's knob comment)
    "base": [],
    "lin_nonest": ["GVOX_LIN_NESTED=0"],
    "lin_incbase": ["GVOX_LIN_INCBASE=1"],
    "lin_b5": ["GVOX_LIN_MINB=5"],
    "lin_nofuse": ["GVOX_LIN_FUSEOM=0"],
    "lin_nounroll": ["GVOX_LIN_UNROLL2=0"],
    "lin_b6": ["GVOX_LIN_MINB=6"],
    "s3": ["GVOX_LIN_STAGES=3"],
    "nopipe": ["GVOX_LIN_PIPE=0"],
    "nocull": ["GVOX_LIN_CULL=0"],
    "tile4": ["GVOX_TILE_MIN_TILES=4"],
    "tile2": ["GVOX_TILE_MIN_TILES=2", "GVOX_TILE_MAX_PPT=128"],
    "tile1": ["GVOX_TILE_MIN_TILES=1", "GVOX_TILE_MAX_PPT=256"],
    "tile2_256": ["GVOX_TILE_MIN_TILES=2", "GVOX_TILE_MAX_PPT=256"],
    "bulk2": ["GVOX_LIN_BULK=1"],
    "bulk3": ["GVOX_LIN_BULK=1", "GVOX_LIN_STAGES=3"],
    "bulk4": ["GVOX_LIN_BULK=1", "GVOX_LIN_STAGES=4"],
    "t256_b2": ["GVOX_LIN_THREADS=256", "GVOX_LIN_MINB=2"],
    "t128_b3": ["GVOX_LIN_THREADS=128", "GVOX_LIN_MINB=3"],
    "g1": ["GVOX_LIN_G=1"],
    "t128_b2": ["GVOX_LIN_THREADS=128", "GVOX_LIN_MINB=2"],
    "t256_b1": ["GVOX_LIN_THREADS=256", "GVOX_LIN_MINB=1"],
    "t128_b5": ["GVOX_LIN_THREADS=128", "GVOX_LIN_MINB=5"],
    "small2": ["GVOX_TILE_MIN_TILES_SMALL=2"],
    "small4": ["GVOX_TILE_MIN_TILES_SMALL=4"],
    "small8": ["GVOX_TILE_MIN_TILES_SMALL=8"],
    "small16": ["GVOX_TILE_MIN_TILES_SMALL=16"],
    "small32": ["GVOX_TILE_MIN_TILES_SMALL=32"],
    "dense48": ["GVOX_DENSE_RATIO=48"],
    "dense96": ["GVOX_DENSE_RATIO=96"],
    "dense192": ["GVOX_DENSE_RATIO=192"],
    "t64_b8": ["GVOX_LIN_THREADS=64", "GVOX_LIN_MINB=8"],
    "branchless": ["GVOX_LIN_BRANCHLESS=1"],
    "t160_b3": ["GVOX_LIN_THREADS=160", "GVOX_LIN_MINB=3"],
    # overlap kernel (stage times from a full bench run)
    "ovl_base": [],
    "ovl_bar": ["GVOX_OVL_NOBAR=0"],
    "ovl_nobar": ["GVOX_OVL_NOBAR=1"],
    "ovl_nobar_b6": ["GVOX_OVL_NOBAR=1", "GVOX_OVL_MINB=6"],
    "ovl_nobar_b8": ["GVOX_OVL_NOBAR=1", "GVOX_OVL_MINB=8"],
    "acc_seg1": ["GVOX_ACC_SEG_MIN=1"],
    "acc_seg6": ["GVOX_ACC_SEG_MIN=6"],
    "acc_noseg": ["GVOX_ACC_SEG_MIN=99"],
    "acc_base": [],
    "acc_seg2": ["GVOX_ACC_SEG_MIN=2"],
    "acc_seg3": ["GVOX_ACC_SEG_MIN=3"],
    "acc_nohoist": ["GVOX_ACC_HOIST=0"],
    "acc_nomaxrun": ["GVOX_ACC_MAXRUN=0"],
    "acc_r01f": ["GVOX_ACC_HOIST=0", "GVOX_ACC_MAXRUN=0"],
    "ovl_b6": ["GVOX_OVL_MINB=6"],
    "ovl_nocull": ["GVOX_OVL_CULL=0"],
    "ovl_b5": ["GVOX_OVL_MINB=5"],
    "ovl_lvs": ["GVOX_OVL_LV_SMEM=1"],
    "ovl_b5_lvs": ["GVOX_OVL_MINB=5", "GVOX_OVL_LV_SMEM=1"],
    "ovl_b8_lvs": ["GVOX_OVL_MINB=8", "GVOX_OVL_LV_SMEM=1"],
    "ovl_b7": ["GVOX_OVL_MINB=7"],
    "ovl_b8": ["GVOX_OVL_MINB=8"],
    "ovl_win4": ["GVOX_OVL_WIN=4"],
    "ovl_win16": ["GVOX_OVL_WIN=16"],
    "ovl_win32": ["GVOX_OVL_WIN=32"],
    "ovl_win64": ["GVOX_OVL_WIN=64"],
    "ovl_ilp4": ["GVOX_OVL_ILP=4"],
    "ovl_ilp4_b6": ["GVOX_OVL_ILP=4", "GVOX_OVL_MINB=6"],
    "ovl_ilp4_lvs": ["GVOX_OVL_LV_SMEM=1"],
    "ovl_win128": ["GVOX_OVL_WIN=128"],
    "acc_ins6": ["GVOX_INS_MINB=6"],
    "acc_ins8": ["GVOX_INS_MINB=8"],
    "acc_acc4": ["GVOX_ACC_MINB=4"],
    "acc_acc4_ins6": ["GVOX_ACC_MINB=4", "GVOX_INS_MINB=6"],
    "acc_acc5": ["GVOX_ACC_MINB=5"],
    "acc_acc4_ins8": ["GVOX_ACC_MINB=4", "GVOX_INS_MINB=8"],
    "acc_acc4_ins6_fin": ["GVOX_ACC_MINB=4", "GVOX_INS_MINB=6", "GVOX_FIN_MINB=8"],
    # r02 session 3: the three-point pipeline with records gathered into shared memory
    "deep0": ["GVOX_LIN_DEEP=0"],
    "deep1": ["GVOX_LIN_DEEP=1"],
    "deep_cg": ["GVOX_LIN_DEEP=1", "GVOX_LIN_DEEP_CG=1"],
    "rpipe_b3": ["GVOX_LIN_RPIPE=1", "GVOX_LIN_MINB=3"],
    "rpipe_b2": ["GVOX_LIN_RPIPE=1", "GVOX_LIN_MINB=2"],
    "order1": ["GVOX_LIN_ORDER=1"],
    "order2": ["GVOX_LIN_ORDER=2"],
    "cullrows": ["GVOX_CULL_ROWS=1"],
    "ovl_cullrows": ["GVOX_CULL_ROWS=1"],
    "cullpf0": ["GVOX_CULL_PREFETCH=0"],
    "cullold": ["GVOX_CULL_ROWS=1", "GVOX_CULL_PREFETCH=0"],
    "cull27pf": ["GVOX_CULL_ROWS=0", "GVOX_CULL_PREFETCH=1"],
    "ovl_cullcoarse": ["GVOX_OVL_CULL_AT_LEVEL=0"],
    "acc_segmajor0": ["GVOX_INS_SEG_MAJOR=0"],
    "acc_known0": ["GVOX_INS_KNOWN_IDX=0"],
    "tmin1": ["GVOX_TILE_MIN_TILES=1"],
}


def build(names):
    sys.path.insert(0, ROOT)
    import importlib.util
    spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_2407_10344_b200", "_build.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    os.makedirs(OUT, exist_ok=True)
    for n in names:
        m.build(out=os.path.join(OUT, f"libgvox_{n}.so"), defines=VARIANTS[n], verbose=False)
        print("built", n, flush=True)


def run(names, extra, stage="linearize"):
    res = {}
    for n in names:
        env = dict(os.environ, GVOX_LIB=os.path.join(OUT, f"libgvox_{n}.so"))
        if n.startswith("ovl") or n.startswith("acc"):
            p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-e2e",
                                "--no-cpu-baseline", "--steps", "3", *extra], env=env,
                               capture_output=True, text=True)
            try:
                d = json.loads(p.stdout.strip().splitlines()[-1])
                res[n] = {k: round(v["ms_per_step"], 2) for k, v in d["stages"].items()
                          if "ms_per_step" in v}
            except Exception:
                res[n] = (p.stdout[-300:], p.stderr[-700:])
        else:
            try:
                p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--linearize-only",
                                    "--no-e2e", "--no-cpu-baseline", "--steps", "6", *extra], env=env,
                                   capture_output=True, text=True, timeout=240)
            except subprocess.TimeoutExpired:
                res[n] = "TIMEOUT"
                print(n, "TIMEOUT", flush=True)
                continue
            line = [l for l in p.stderr.splitlines() if "linearize-only" in l]
            res[n] = line[-1] if line else p.stderr[-500:]
        print(n, res[n], flush=True)
    return res


if __name__ == "__main__":
    names = sys.argv[2].split(",") if len(sys.argv) > 2 and sys.argv[2] else list(VARIANTS)
    if sys.argv[1] == "build":
        build(names)
    else:
        run(names, sys.argv[3:])
