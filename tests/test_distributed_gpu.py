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


@pytest.mark.parametrize("model,reps,nproc", [("mlp", "1-1-1-1", 2), ("mlp", "1-1-1", 2), ("mlp", "2-1", 3),
                                              ("mlp", "1-2-1", 4), ("conv", "2-1", 3), ("gpt", "1-1", 2),
                                              ("mlp-unfused", "1-1-1-1", 2)])
def test_multi_process_pipeline_matches_oracle(model, reps, nproc):
    """Straight plans over 2 processes; replicated plans with the replicas in different processes
    (peer-mapped gradient reads in the fused allreduce+SGD, remote round flags); the VGG-style
    conv 2-1 plan and a GPT-2-style 2-stage pipeline across processes.  bf16 MLP hand-offs release
    the receiver's flag from the producing GEMM's last CTA; "mlp-unfused" covers the fallback."""
    env = dict(os.environ, PD_REPS=reps, PD_DIST_BACKEND="gloo", PD_MODEL=model.split("-")[0])
    if model.endswith("-unfused"):  # stand-alone signal kernels instead of the GEMM-fused flag release
        env["PD_FUSED_HANDOFF"] = "0"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", "--master-port=29517", os.path.join(REPO, "tools", "dist_check.py")]
    out = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=600)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert out.returncode == 0 and lines, out.stdout[-3000:] + out.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["world"] == nproc
    assert res["ok"], res
