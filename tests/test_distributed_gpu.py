"""Two processes, peer-mapped inboxes and system-scope flags (runs on a single B200: both ranks map
the same device; on a multi-GPU box the same code path uses NVLink peer stores)."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("stages", [4, 3])
def test_two_process_pipeline_matches_oracle(stages):
    env = dict(os.environ, PD_STAGES=str(stages), PD_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29517", os.path.join(REPO, "tools", "dist_check.py")]
    out = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=600)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert out.returncode == 0 and lines, out.stdout[-3000:] + out.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["world"] == 2
    assert res["ok"], res
