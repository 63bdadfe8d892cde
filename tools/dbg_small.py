import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
from workloads import gen
from gpu_harness import run_gpu
b = gen.make_batch("tree_lstm", 2, 64, 64, "sst_tree", 24, seed=11)
g = run_gpu(b, "bf16")
print("ok", g["h_out"].sum())
