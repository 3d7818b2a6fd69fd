"""The multi-GPU bench legs (`bench.py --gpus N`: NCCL / peer-memory
runners, GPipe, hybrid DP x PP, module configs) as 2 ranks sharing the one
GPU over gloo (`--share-gpu`): every leg must run without reporting an error
— the dry run of what the driver's 2/4/8-GPU scaling run executes."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _errors(obj, path=""):
    out = []
    if isinstance(obj, dict):
        for k, v in obj.items():
            if k == "error":
                out.append(f"{path}: {v}")
            out += _errors(v, f"{path}/{k}")
    return out


def test_two_rank_bench_dry_run():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--dist-backend", "gloo", "--share-gpu", "--n-params", "1e7", "--no-cpu"]
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    pipe = line["pipeline"]
    assert isinstance(pipe, dict) and not _errors(pipe), _errors(pipe)
    for key in ("pred_on", "pred_off", "peer_graphed", "hybrid_dp_pp", "configs"):
        assert key in pipe, key
