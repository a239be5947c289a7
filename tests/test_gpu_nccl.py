"""Group-sharded execution across GPUs: one process per GPU over NCCL,
each rank computing only its LPT share of the groups and all-gathering the output per
slab on a side stream (distributed.SlabGather). Rank 0 checks the gathered batch
against one launch over the whole batch (bf16: |diff| <= 1e-2, the differently
chunked partials' rounding). Needs >= 2 GPUs; the gather logic itself is covered
on CPU by the gloo tests in test_multiproc.py."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("config", ["c4", "c2"])
def test_nccl_group_sharding_with_overlapped_gather(config):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (one NCCL rank per GPU)")
    world = min(n, 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(HERE, "mp", "nccl_worker.py"), config]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=540)
    assert res.returncode == 0, res.stderr[-3000:]
    line = [l for l in res.stdout.splitlines() if l.startswith("{")][-1]
    r = json.loads(line)
    assert r["world"] == world and not r["nan"]
    assert all(e == 0 for e in r["device_errors"])
    assert r["max_abs_diff"] <= 1e-2
