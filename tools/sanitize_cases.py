"""Small training steps through every kernel path, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Each case runs schedule + forward + backward once and checks the result
against the fp64 oracle loosely (the sanitizer run is about memory / synchronisation errors).

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case ...]

Cases (path forced by the library's environment switches, set per case in a child process):
  persist      Tree-LSTM h=256 bf16: persistent level kernels, row GEMMs, stream-K lazy
  persist_fc   Tree-FC h=128 bf16 (persistent Tree-FC plans)
  rows         Tree-FC h=640 bf16 with CAVS_ROWS_MIN_TILES=1: row-tiled k_rows level GEMMs
  tc_level     Tree-LSTM h=128 bf16, CAVS_PERSIST=0: per-task swap-AB / skinny kernels
  fp32         Tree-LSTM h=64 fp32 (CAVS_FP32_FFMA=1 in round 1; round 2: the tcgen05 bf16x3 path)
  fp32_tc*     FP32 mode on tcgen05 (bf16x3 split operands), Tree-LSTM and Tree-FC
  rows_splitk* split-K row-tiled kernels (shares meet at a per-tile counter)
  ksl4         per-task kernels with 16-CTA K-sliced gate-split clusters
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CASES = {
    "persist": (dict(cell="tree_lstm", N=2, h=256, d=256, shape="sst_tree", K=6), "bf16", {}),
    "persist_fc": (dict(cell="tree_fc", N=2, h=128, d=128, shape="cbt8", K=3), "bf16", {}),
    "rows": (dict(cell="tree_fc", N=2, h=640, d=640, shape="cbt16", K=2), "bf16", {"CAVS_ROWS_MIN_TILES": "1"}),
    "tc_level": (dict(cell="tree_lstm", N=2, h=128, d=128, shape="sst_tree", K=5), "bf16", {"CAVS_PERSIST": "0"}),
    "fp32": (dict(cell="tree_lstm", N=2, h=64, d=64, shape="sst_tree", K=4), "fp32", {}),
    # round 2
    "ksplit_bwd": (dict(cell="tree_lstm", N=2, h=256, d=256, shape="sst_tree", K=6), "bf16", {"CAVS_PBWD": "1"}),
    "multicast": (dict(cell="tree_lstm", N=2, h=256, d=256, shape="sst_tree", K=6), "bf16", {"CAVS_PERSIST_MC": "1"}),
    "rows_pair": (dict(cell="tree_fc", N=2, h=512, d=512, shape="cbt16", K=2), "bf16",
                  {"CAVS_ROWS_MIN_TILES": "1", "CAVS_ROWS_PAIR": "1", "CAVS_PERSIST": "0"}),
    "dag": (dict(cell="tree_lstm", N=2, h=128, d=128, shape="dag", K=5), "bf16", {}),
    "ablations": (dict(cell="tree_lstm", N=2, h=128, d=128, shape="sst_tree", K=5), "bf16",
                  {"CAVS_LAZY_BATCH": "0", "CAVS_UNFUSED": "1", "CAVS_STREAMING": "1"}),
    # round 2, second half: FP32 on tcgen05 (bf16x3), split-K row kernel, K-sliced gate split
    "fp32_tc": (dict(cell="tree_lstm", N=2, h=64, d=64, shape="sst_tree", K=4), "fp32", {}),
    "fp32_tc_fc": (dict(cell="tree_fc", N=2, h=128, d=64, shape="cbt8", K=3), "fp32", {}),
    "rows_splitk": (dict(cell="tree_fc", N=2, h=256, d=128, shape="cbt16", K=3), "bf16",
                    {"CAVS_ROWS_MIN_TILES": "1", "CAVS_PERSIST": "0"}),
    "rows_splitk_lstm": (dict(cell="tree_lstm", N=2, h=256, d=128, shape="sst_tree", K=6), "bf16",
                         {"CAVS_ROWS_MIN_TILES": "1", "CAVS_PERSIST": "0", "CAVS_ROWS_SEL": "i"}),
    "ksl4": (dict(cell="tree_lstm", N=2, h=128, d=64, shape="sst_tree", K=4), "bf16",
             {"CAVS_PERSIST": "0", "CAVS_ROWS": "0", "CAVS_TC_KSL": "4"}),
}


def run_case(name):
    import numpy as np
    from gpu_harness import rel, run_gpu, run_oracle
    from workloads import gen
    spec, prec, _ = CASES[name]
    if spec["shape"] == "dag":                      # shared children and duplicate child ids
        import test_gpu_parity as T
        b = gen.batch_from_graphs(T._random_dags(spec["K"], spec["N"], 20, 1), cell=spec["cell"], N=spec["N"],
                                  h=spec["h"], d=spec["d"], seed=1, x_at="all", loss_at="all")
    else:
        b = gen.make_batch(spec["cell"], spec["N"], spec["h"], spec["d"], spec["shape"], spec["K"], seed=1)
    g = run_gpu(b, prec)
    r = run_oracle(b)
    e = max(rel(g["h_out"], r["h_out"]), rel(g["dparams"], r["dparams"]), rel(g["dx"], r["dx"]))
    tol = 2e-2 if prec == "bf16" else 1e-5
    print(f"{name}: max rel err {e:.2e} (tol {tol}) path: {g['ctx'].path_info()}")
    assert e <= tol, name
    g["ctx"].close()


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    if len(names) == 1:
        os.environ.update(CASES[names[0]][2])
        run_case(names[0])
    else:
        rc = 0
        for n in names:
            env = dict(os.environ, **CASES[n][2])
            rc |= subprocess.call([sys.executable, __file__, n], env=env)
        sys.exit(rc)
