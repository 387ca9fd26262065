"""The multi-GPU path end to end on the box's GPU: two torchrun ranks share it
with gloo collectives (the data path is the same code the NCCL run takes). Every query must be
served exactly once and the combined first tokens must equal the reference's run (golden)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_ranks_serve_every_query_once(tmp_path):
    out = tmp_path / "mr.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(HERE, "support", "multirank_c1.py"), str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    got = json.loads(out.read_text())
    with open(os.path.join(HERE, "golden", "c1_pipeline.json")) as f:
        G = json.load(f)
    assert got["labels"] == G["labels"]
    assert sorted(set(got["owner"])) == [0, 1]          # both ranks own clusters (LPT)
    assert sum(got["served"]) == 64                      # each query served by exactly one rank
    assert got["first"] == G["run_batch_first_token"]    # == the reference's run_batch
