"""bench.py's launch contract: `--gpus N` outside torchrun re-launches itself as N ranks and the
printed line reports N; under torchrun a WORLD_SIZE different from --gpus is refused."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "LOCAL_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(REPO, "bench.py")] + args, cwd=REPO, env=e,
                          capture_output=True, text=True, timeout=timeout)


def _line(out):
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert out.returncode == 0 and len(lines) == 1, out.stdout[-2000:] + out.stderr[-2000:]
    return json.loads(lines[0])


def test_reference_arm_self_launches_two_ranks():
    """CPU-only: the reference arm under the self-launch prints exactly one line (rank 0) for N=2."""
    out = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--width", "512",
                "--minibatches", "32"])
    d = _line(out)
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["cpu_baseline"]["cores"] >= 1 and d["e2e"]["h2d_bytes_per_step"] == 0


def test_world_size_mismatch_is_refused():
    out = _run(["--impl", "reference", "--gpus", "4", "--steps", "1", "--warmup", "0"],
               env={"WORLD_SIZE": "1", "RANK": "0"})
    assert out.returncode == 2 and "refusing" in out.stderr


@pytest.mark.gpu
def test_bench_two_ranks_report_two_gpus():
    """Two ranks (on a one-GPU box both map cuda:0, gloo plumbing; on a multi-GPU box one each)."""
    out = _run(["--gpus", "2", "--steps", "1", "--warmup", "1", "--width", "1024", "--batch", "256",
                "--minibatches", "32", "--no-cpu-baseline", "--e2e-steps", "1"], timeout=900)
    d = _line(out)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpus_active"] >= 1
    assert d["p2p"]["bytes_traced_step"] > 0  # stages 0-3 | 4-7 hand off across the two processes
    assert set(d["p2p"]["bytes_by_boundary"]) == {"3"} or set(d["p2p"]["bytes_by_boundary"]) == {3}
