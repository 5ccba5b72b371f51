"""CLI of the B200 backend (mirrors pipesim/cli.py): argument handling on CPU, and on the GPU an
end-to-end profile -> plan -> simulate run with the reference's artefacts, plus checkpoint/resume."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1806_03377_b200 import cli
from paper_1806_03377_b200.errors import ValidationError
from paper_1806_03377_b200.models import ConvNetSpec, GPTSpec, MLPSpec

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_model_specs():
    m = cli.parse_model("mlp:256:4:64:bf16", lr=1e-3)
    assert isinstance(m, MLPSpec) and m.widths == (256,) * 5 and m.batch == 64 and m.lr == 1e-3
    assert isinstance(cli.parse_model("vgg16:16"), ConvNetSpec)
    g = cli.parse_model("gpt:250:256:4:2:128:2")
    assert isinstance(g, GPTSpec) and g.layers == 2 and g.num_layers == 4
    assert cli.parse_model("gpt2-medium").num_layers == 26
    with pytest.raises(ValidationError):
        cli.parse_model("resnet50")


def test_usage_errors_exit_1():
    with pytest.raises(SystemExit) as e:
        cli.main(["simulate"])
    assert e.value.code == cli.EXIT_USAGE


def test_plan_command_on_measured_profile(tmp_path):
    prof = os.path.join(REPO, "profiles", "layer_profiles", "vgg16_profile.json")
    rc = cli.main(["plan", prof, "--machines", "8", "--bandwidth", "12.5e9", "--out-dir", str(tmp_path)])
    assert rc == 0
    doc = json.loads((tmp_path / "plan.json").read_text())
    assert doc["config"] == "7-1" and doc["manifest"]["command"] == "plan"


@pytest.mark.gpu
def test_profile_plan_simulate_checkpoint(tmp_path):
    env = dict(os.environ)
    run = lambda *a: subprocess.run([sys.executable, "-m", "paper_1806_03377_b200", *a], cwd=REPO, env=env,  # noqa
                                    capture_output=True, text=True, timeout=600)
    model = "mlp:256:4:64:bf16"
    r = run("profile", "--model", model, "--out", str(tmp_path / "profile.json"))
    assert r.returncode == 0, r.stderr
    r = run("plan", str(tmp_path / "profile.json"), "--machines", "2", "--straight", "--out-dir", str(tmp_path))
    assert r.returncode == 0, r.stderr
    ck = tmp_path / "ck"
    r = run("simulate", str(tmp_path / "plan.json"), str(tmp_path / "profile.json"), "--model", model,
            "--minibatches", "14", "--out-dir", str(tmp_path / "a"), "--checkpoint-dir", str(ck))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "staleness_violations: 0" in r.stdout
    for name in ("report.json", "trace.csv", "staleness.json"):
        assert (tmp_path / "a" / name).exists()
    rep = json.loads((tmp_path / "a" / "report.json").read_text())
    assert rep["manifest"]["backend"] == "b200" and rep["steady_throughput"] > 0
    files = sorted(os.listdir(ck))
    assert len(files) == json.loads((tmp_path / "plan.json").read_text())["machines_used"]
    # resume: training continues from the checkpoint (loss of the first minibatch drops below the fresh run's)
    r = run("simulate", str(tmp_path / "plan.json"), str(tmp_path / "profile.json"), "--model", model,
            "--minibatches", "14", "--out-dir", str(tmp_path / "b"), "--resume", str(ck))
    assert r.returncode == 0, r.stderr
    la = json.loads((tmp_path / "a" / "report.json").read_text())["losses"]
    lb = json.loads((tmp_path / "b" / "report.json").read_text())["losses"]
    assert np.isfinite(lb).all() and lb[0] != la[0]
    w0 = np.load(ck / files[0])
    assert "W0" in w0 and w0["W0"].dtype == np.float32


@pytest.mark.gpu
def test_compare_regimes_on_device(tmp_path):
    """The reference's five regimes (cli.py:211-261) executed on the runtime: every regime runs and
    reports a measured throughput, single_machine is the 1.00x base, the artefact has the schema."""
    env = dict(os.environ)
    run = lambda *a: subprocess.run([sys.executable, "-m", "paper_1806_03377_b200", *a], cwd=REPO, env=env,  # noqa
                                    capture_output=True, text=True, timeout=900)
    model = "mlp:256:4:64:bf16"
    r = run("profile", "--model", model, "--out", str(tmp_path / "profile.json"))
    assert r.returncode == 0, r.stderr
    r = run("compare", str(tmp_path / "profile.json"), "--model", model, "--machines", "4", "--minibatches", "16",
            "--out-dir", str(tmp_path))
    assert r.returncode == 0, r.stdout + r.stderr
    doc = json.loads((tmp_path / "compare.json").read_text())
    names = [x["regime"] for x in doc["regimes"]]
    assert names == ["single_machine", "model_parallel", "data_parallel", "straight_pipeline", "full_plan"]
    assert doc["regimes"][0]["speedup"] == 1.0 and doc["regimes"][2]["config"] == "4"
    assert all(x["throughput"] > 0 and x["predicted_throughput"] > 0 for x in doc["regimes"])
    assert doc["regimes"][1]["max_inflight"] == 1


def test_compare_minibatches_whole_rounds():
    from paper_1806_03377_b200.plans import Plan, Stage

    p71 = Plan(stages=(Stage(1, 13, 7), Stage(14, 16, 1)), bottleneck_time=1.0, noam=2, machines_used=8)
    assert cli._regime_minibatches(p71, 32) == 35
    p8 = Plan(stages=(Stage(1, 16, 8),), bottleneck_time=1.0, noam=1, machines_used=8)
    assert cli._regime_minibatches(p8, 32) == 32
    with pytest.raises(SystemExit) as e:
        cli.main(["compare", "x.json"])  # --model / --machines missing: usage error
    assert e.value.code == cli.EXIT_USAGE
