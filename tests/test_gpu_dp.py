"""The N > 1 data-parallel path of bench.py on one GPU: two ranks with the gloo backend sharing
cuda:0 (NCCL refuses two ranks on one device) run the sharded global batch, the grad event and the
bucketed all-reduce end to end.  NCCL over NVLink is the same code with the
backend switched; only one GPU is available to this build."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(600)
def test_bench_two_ranks_gloo_on_one_gpu():
    env = dict(os.environ, CAVS_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--no-cpu-baseline", "--pool", "2"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=540)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["global_batch"] == 256 and line["config"]["batch_per_gpu"] == 128.0
    assert line["value"] > 0 and line["e2e"]["value"] > 0
