"""Benchmark: pipeline-training samples/s of the 1F1B weight-stashing executor on B200.

Contract (see task): `python bench.py --gpus N --steps K --warmup W [--impl reference]`
prints ONE JSON line on rank 0.

Workload (BASELINE.json configs[1]): 8-stage, 16-layer MLP, width 8192, bf16 storage /
fp32 accumulate, straight pipeline (one stage per GPU at N=8; 8/N stages per GPU below),
1F1B with weight stashing, minibatch 2048, synthetic data.
A bench "step" = one execution of the whole 1F1B schedule over K=256 minibatches
(pipeline fill + steady state + drain), i.e. 256*2048 = 524,288 samples; at 8 GPUs the
fill/drain bubble of a 256-minibatch schedule is 7/263 (2.7 %).
`--gpus N` without torchrun re-launches itself as N ranks (torch.distributed.run, 127.0.0.1);
under torchrun WORLD_SIZE must equal --gpus.
The working set (~15 GB of weight versions + activations) is >100x the 126 MB L2, so no
explicit L2 flush is needed between steps.
"""

from __future__ import annotations

import argparse
import faulthandler
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "pipeline training samples/s at 1/2/4/8 B200; stage TC util %; bubble %"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=["mlp", "vgg", "gpt"], default="mlp",
                   help="mlp: configs[1] MLP-8192 straight pipeline (headline); vgg: configs[2] VGG-16 7-1; "
                        "gpt: configs[3] GPT-2 medium 8-stage")
    p.add_argument("--batch", type=int, default=2048)
    p.add_argument("--minibatches", type=int, default=256)
    p.add_argument("--width", type=int, default=8192)
    p.add_argument("--layers", type=int, default=16)
    p.add_argument("--stages", type=int, default=8)
    p.add_argument("--mode", default="weight_stashing")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample-only", action="store_true",
                   help="internal: run only the CPU baseline sample and print it (child process)")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--serial", choices=["on", "off"], default="off",
                   help="timed region: issue all hosted stages on one stream (on) or one stream per stage (off); "
                        "the roofline pass is always serial so per-kernel events are not inflated by overlap")
    return p.parse_args()


GPT_BOUNDS = [(1, 4), (5, 7), (8, 10), (11, 13), (14, 17), (18, 21), (22, 25), (26, 26)]


def workload(args):
    if args.workload == "gpt":
        return {
            "workload": "cfg4: GPT-2 medium (24 layers, d 1024, 16 heads, vocab 50257 padded to 50304, untied head), "
                        "seq 1024, bf16, synthetic tokens, 8-stage 1F1B weight_stashing",
            "minibatch": args.batch,
            "minibatch_unit": "sequences of 1024 tokens",
            "minibatches_per_step": args.minibatches,
            "stages": 8,
            "stage_layers": GPT_BOUNDS,
            "stages_per_gpu": 8 // max(1, args.gpus),
            "lr": 1e-4,
            "l2": "working set > 100x L2 (126 MB); no flush needed",
            "loss": "next-token softmax cross-entropy, mean over tokens",
            "streams": "one per GPU (stages in program order)" if args.serial == "on" else "one per stage",
            "roofline_timing": "per-GEMM CUDA events over one extra serial step (no inter-stage overlap)",
        }
    if args.workload == "vgg":
        return {
            "workload": "cfg3: VGG-16 on synthetic 224x224 images, PipeDream 7-1 (conv stack replicated 7x with "
                        "round-rule peer-memory allreduce, FC stage 1x), 1F1B-RR weight_stashing",
            "minibatch": args.batch,
            "minibatches_per_step": args.minibatches,
            "stages": 2,
            "workers": 8,
            "workers_per_gpu": 8 // max(1, args.gpus),
            "lr": 1e-3,
            "l2": "working set > 100x L2 (126 MB); no flush needed",
            "loss": "softmax cross-entropy, mean over the minibatch",
            "streams": "one per GPU (workers in program order)" if args.serial == "on" else "one per worker",
            "roofline_timing": "per-GEMM CUDA events over one extra serial step (no inter-worker overlap)",
        }
    return {
        "workload": f"cfg2: {args.stages}-stage {args.layers}-layer MLP-{args.width} bf16 straight pipeline, "
                    f"1F1B {args.mode}",
        "minibatch": args.batch,
        "minibatches_per_step": args.minibatches,
        "stages": args.stages,
        "stages_per_gpu": args.stages // max(1, args.gpus),
        "lr": 1e-5,
        "l2": "working set > 100x L2 (126 MB); no flush needed",
        "loss": "1/(2B) sum (Z-T)^2",
        "streams": "one per GPU (stages in program order)" if args.serial == "on" else "one per stage",
        "roofline_timing": "per-GEMM CUDA events over one extra serial step (no inter-stage overlap)",
    }


def load_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            with open(self.path) as fh:
                for line in fh:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[5:9]) if v.lower() == "active"})
        loaded = [x for x in sm if x > 0.5 * (max(sm) if sm else 1)]
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


_CPU_CACHE: dict = {}


def cpu_sample(args, seconds=12.0, batch=128, max_minibatches=3):
    """Time the CPU oracle (numpy fp32, all host threads) on a bounded sample of the workload."""
    import numpy as np

    import paper_1806_03377_b200 as pd
    from oracle.pipeline_oracle import closed_form_version, mlp_train

    per = args.layers // args.stages
    bounds = [(s * per + 1, (s + 1) * per) for s in range(args.stages)]
    w = args.width
    key = (w, args.layers, batch)
    if key not in _CPU_CACHE:
        rng = np.random.default_rng(0)
        params = [(rng.standard_normal((w, w), dtype=np.float32) * np.float32((2.0 / w) ** 0.5),
                   np.zeros(w, dtype=np.float32)) for _ in range(args.layers)]
        X = rng.standard_normal((1, batch, w), dtype=np.float32)
        T = rng.standard_normal((1, batch, w), dtype=np.float32)
        _CPU_CACHE[key] = (params, X, T)
    params, X, T = _CPU_CACHE[key]
    n = args.stages
    versions = lambda s, mb, d: closed_form_version(args.mode, n, s, mb, d)  # noqa: E731
    done, t0 = 0, time.perf_counter()
    while True:
        k = done + 1
        mlp_train(params, X, T, 1e-5, bounds, versions, 1, dtype=np.float32, prune=True)
        done = k
        el = time.perf_counter() - t0
        if el >= seconds or done >= max_minibatches:
            break
    try:
        from threadpoolctl import threadpool_info

        cores = max((i.get("num_threads", 1) for i in threadpool_info()), default=os.cpu_count())
    except Exception:
        cores = os.cpu_count()
    return {"value": done * batch / el, "unit": "samples/s", "cores": cores, "kind": "port",
            "sample": f"{done} minibatch(es) of {batch} samples through all {args.layers} layers "
                      f"(fwd+bwd+SGD, numpy fp32, weight-stashing versions) in {el:.1f} s"}


def cpu_sample_vgg(args, seconds=12.0, batch=4, max_minibatches=2):
    """Time the conv-net oracle (torch CPU fp32, all host threads) on a bounded VGG-16 sample."""
    import numpy as np
    import torch

    import paper_1806_03377_b200 as pd
    from oracle.convnet_oracle import convnet_train

    torch.set_num_threads(os.cpu_count())
    spec = pd.vgg16(batch=batch)
    key = ("vgg", batch)
    if key not in _CPU_CACHE:
        rng = np.random.default_rng(0)
        params = [(rng.standard_normal(g.w_shape, dtype=np.float32) * np.float32(0.01),
                   np.zeros(g.c_out, dtype=np.float32)) for g in spec.geoms()]
        X = rng.standard_normal((1, batch, 224, 224, 3), dtype=np.float32)
        y = rng.integers(0, 1000, size=(1, batch)).astype(np.int32)
        _CPU_CACHE[key] = (params, X, y)
    params, X, y = _CPU_CACHE[key]
    done, t0 = 0, time.perf_counter()
    while True:
        convnet_train(spec.geoms(), params, X, y, 1e-3, [(1, 13), (14, 16)], lambda s, mb, d: 0, 1, emulate=None,
                      dtype=torch.float32)
        done += 1
        el = time.perf_counter() - t0
        if el >= seconds or done >= max_minibatches:
            break
    return {"value": done * batch / el, "unit": "samples/s", "cores": torch.get_num_threads(), "kind": "port",
            "sample": f"{done} minibatch(es) of {batch} images through all 16 VGG-16 layers "
                      f"(fwd+bwd+SGD, torch-CPU fp32 conv-net oracle) in {el:.1f} s"}


def cpu_sample_gpt(args, seconds=12.0, max_minibatches=1):
    """Time the GPT oracle (torch CPU fp32 autograd, all host threads) on one GPT-2 medium sequence."""
    import numpy as np
    import torch

    import paper_1806_03377_b200 as pd
    from oracle.gpt_oracle import gpt_train

    torch.set_num_threads(os.cpu_count())
    spec = pd.gpt2_medium(batch=1)
    key = ("gpt", 1)
    if key not in _CPU_CACHE:
        rng = np.random.default_rng(0)
        params = [(rng.standard_normal(g.w_shape, dtype=np.float32) * np.float32(0.02),
                   np.zeros(g.b_numel, dtype=np.float32)) for g in spec.geoms()]
        tok = rng.integers(0, spec.vocab, size=(1, 1, spec.seq + 1)).astype(np.int32)
        _CPU_CACHE[key] = (params, tok[:, :, :-1], tok[:, :, 1:])
    params, X, y = _CPU_CACHE[key]
    bounds = [(1, spec.num_layers)]
    done, t0 = 0, time.perf_counter()
    while True:
        gpt_train(spec, params, X, y, 1e-4, bounds, lambda s, mb, d: 0, 1, emulate=None, dtype=torch.float32)
        done += 1
        el = time.perf_counter() - t0
        if el >= seconds or done >= max_minibatches:
            break
    return {"value": done / el, "unit": "samples/s", "cores": torch.get_num_threads(), "kind": "port",
            "sample": f"{done} sequence(s) of 1024 tokens through all 26 GPT-2 medium layers "
                      f"(fwd+bwd+SGD, torch-CPU fp32 autograd oracle) in {el:.1f} s"}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform

    return platform.processor() or "unknown"


def reference_simulator_sample(args, seconds=3.0):
    """The reference's own CPU path for this configuration: pipesim.run + staleness_check
    (simulator.py:401-411, 423-466) on the same plan / mode / minibatch count, with the measured
    B200 layer profile (profiles/layer_profiles, reference JSON format) as its cost context.  Runs
    the unmodified package installed in baseline/_ref (pip --target, git-ignored); None if absent."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "pipesim")):
        return {"available": False, "why": "baseline/_ref/pipesim not installed"}
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import pipesim as ps

    prof_name = {"mlp": "mlp8192_profile.json", "vgg": "vgg16_profile.json", "gpt": "gpt2_medium_profile.json"}
    prof = ps.load_profile(os.path.join(REPO, "profiles", "layer_profiles", prof_name[args.workload]))
    if args.workload == "vgg":
        stages = (ps.Stage(1, 13, 7), ps.Stage(14, 16, 1))
        machines, bpe = 8, 2
    elif args.workload == "gpt":
        stages = tuple(ps.Stage(a, b, 1) for a, b in GPT_BOUNDS)
        machines, bpe = 8, 2
    else:
        per = args.layers // args.stages
        stages = tuple(ps.Stage(s * per + 1, (s + 1) * per, 1) for s in range(args.stages))
        machines, bpe = args.stages, 2
    if prof.num_layers != stages[-1].last_layer:
        return {"available": False, "why": f"profile has {prof.num_layers} layers, plan {stages[-1].last_layer}"}
    ctx = ps.build_context(prof, ps.HardwareSpec(num_machines=machines, bandwidth=900e9, bytes_per_elem=bpe))
    plan = ps.Plan(stages=stages, bottleneck_time=1.0, noam=ps.noam_for(machines, stages[0].replication),
                   machines_used=machines)
    cfg = ps.SimConfig(plan=plan, mode=ps.Mode(args.mode), num_minibatches=args.minibatches)
    runs, t0 = 0, time.perf_counter()
    while True:
        res = ps.run(cfg, ctx)
        if plan.stages[0].replication == 1 and all(st.replication == 1 for st in plan.stages):
            ps.staleness_check(res.ledger, cfg.mode, plan.num_stages)
        runs += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return {"available": True, "package": f"pipesim {ps.__version__} (unmodified, baseline/_ref)",
            "ms_per_run": el / runs * 1e3, "runs": runs, "minibatches_per_run": args.minibatches,
            "threads": 1, "what": "pipesim.run + staleness_check: the reference's discrete-event simulation of "
                                  "this schedule (simulated, not trained, minibatches)"}


def _all_host_threads():
    """Use every host core for the CPU arms even under torchrun (which exports OMP_NUM_THREADS=1)."""
    n = os.cpu_count() or 1
    import numpy  # noqa: F401  (load its BLAS before setting the pool size)

    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(limits=n)
    except Exception:
        pass
    try:
        import torch

        torch.set_num_threads(n)
    except Exception:
        pass


def _phase(msg):
    """Progress marker on stderr (stdout carries only the JSON line)."""
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def _cpu_sample_for(args):
    return (cpu_sample_vgg(args) if args.workload == "vgg" else
            cpu_sample_gpt(args) if args.workload == "gpt" else cpu_sample(args))


def cpu_baseline_isolated(args, timeout=300):
    """The CPU baseline sample in a child process (all host threads, no CUDA context): a stuck or
    slow CPU library cannot hold back the bench line; on failure the baseline is reported as such."""
    env = dict(os.environ, OMP_NUM_THREADS=str(os.cpu_count() or 1))
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "LOCAL_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    cmd = [sys.executable, os.path.abspath(__file__)] + [a for a in sys.argv[1:]] + ["--cpu-sample-only"]
    try:
        out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout)
        lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if out.returncode == 0 and lines:
            return json.loads(lines[-1])
        why = f"child exited {out.returncode}: {out.stderr.strip()[-200:]}"
    except subprocess.TimeoutExpired:
        why = f"timed out after {timeout} s"
    return {"value": None, "unit": "samples/s", "cores": os.cpu_count(), "kind": "port", "sample": why}


def run_reference(args, rank):
    if rank != 0:
        return
    import numpy as np  # noqa: F401

    _all_host_threads()

    cfg = workload(args)
    vgg = args.workload == "vgg"
    gpt = args.workload == "gpt"
    if gpt:
        one = lambda: cpu_sample_gpt(args, seconds=0.0)  # noqa: E731
    elif vgg:
        one = lambda: cpu_sample_vgg(args, seconds=0.0, max_minibatches=1)  # noqa: E731
    else:
        one = lambda: cpu_sample(args, seconds=0.0, max_minibatches=1)  # noqa: E731
    per_step = 1 if gpt else (4 if vgg else 128)
    for _ in range(args.warmup):
        one()
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(one())
    el = time.perf_counter() - t0
    samples = per_step * len(vals)
    value = samples / el
    cb = dict(vals[-1])
    cb["value"] = value
    cb["sample"] = (f"{args.steps} steps x 1 sequence of 1024 tokens, all 26 GPT-2 medium layers, torch-CPU fp32"
                    if gpt else
                    f"{args.steps} steps x 1 minibatch of 4 images, all 16 VGG-16 layers, torch-CPU fp32" if vgg else
                    f"{args.steps} steps x 1 minibatch of 128 samples, all {args.layers} layers, numpy fp32")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
           "config": cfg, "cpu_baseline": cb,
           "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def build_config(args):
    """(SimConfig, model spec) of the selected workload."""
    import paper_1806_03377_b200 as pd

    if args.workload == "gpt":
        stages = tuple(pd.Stage(a, b, 1) for a, b in GPT_BOUNDS)
        plan = pd.Plan(stages=stages, bottleneck_time=1.0, noam=8, machines_used=8)
        spec = pd.gpt2_medium(batch=args.batch, lr=1e-4, n_blocks=2, seed=0)
    elif args.workload == "vgg":
        # PipeDream's VGG-16 partition on 8 machines: conv stack x7, FC stage x1
        plan = pd.Plan(stages=(pd.Stage(1, 13, 7), pd.Stage(14, 16, 1)), bottleneck_time=1.0, noam=2, machines_used=8)
        spec = pd.vgg16(batch=args.batch, lr=1e-3, n_blocks=2, seed=0)
    else:
        per = args.layers // args.stages
        stages = tuple(pd.Stage(s * per + 1, (s + 1) * per, 1) for s in range(args.stages))
        plan = pd.Plan(stages=stages, bottleneck_time=1.0, noam=args.stages, machines_used=args.stages)
        spec = pd.mlp(args.width, args.layers, batch=args.batch, dtype="bf16", lr=1e-5, n_blocks=4, seed=0)
    return pd.SimConfig(plan=plan, mode=args.mode, num_minibatches=args.minibatches), spec


def run_ours(args, rank, world):
    import torch

    import paper_1806_03377_b200 as pd

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    dev = torch.cuda.current_device()
    cfg, spec = build_config(args)
    ex = pd.Executor(cfg, model=spec)
    ex.set_serial(args.serial == "on")
    dist = torch.distributed if world > 1 else None

    def barrier():
        if dist is not None:
            dist.barrier()

    stream = torch.cuda.current_stream()
    red_dev = "cuda" if dist is not None and dist.get_backend() == "nccl" else "cpu"

    def reduce(vals, op):
        t = torch.tensor(vals, device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=op)
        return [float(x) for x in t.cpu()]

    _phase("warmup")
    for _ in range(args.warmup):
        ex.step(stream=stream)
    torch.cuda.synchronize()
    _phase("timed region")
    # ---------------- timed region (device events, max over ranks)
    launches0 = ex.launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clocks:
        barrier()
        torch.cuda.synchronize()
        start.record(stream)
        for _ in range(args.steps):
            ex.step(stream=stream)
        end.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = start.elapsed_time(end)
    if dist is not None:
        ms = reduce([ms], dist.ReduceOp.MAX)[0]
    launches = ex.launch_count() - launches0
    # ---------------- roofline pass: one serial step with per-GEMM CUDA events on the launching stream
    _phase("serial roofline pass")
    barrier()
    ex.set_serial(True)
    ex.kernel_timing(True)
    ex.step(stream=stream)
    torch.cuda.synchronize()
    kstats = ex.kernel_stats()
    # per-stage tensor-core utilisation: the stage's GEMM FLOPs over the stage's serial kernel time
    peaks_, _ = load_peaks()
    peak_ = float(peaks_.get("bf16_tflops_sustained", peaks_.get("bf16_tflops")))
    stage_util = {}
    for w in sorted(b.wid for b in ex.bufs.values()):
        ks = ex.kernel_stats(w)
        busy = sum(v["total_ms"] for v in ks.values())
        fl = sum(v["total_flops"] for k, v in ks.items() if k in ("fwd", "dgrad", "wgrad_sgd"))
        gemm_ms = sum(v["total_ms"] for k, v in ks.items() if k in ("fwd", "dgrad", "wgrad_sgd"))
        if busy > 0:
            stage_util[str(w)] = {"tc_util_busy": round(fl / (busy * 1e-3) / 1e12 / peak_, 3),
                                  "tc_util_gemm": round(fl / (gemm_ms * 1e-3) / 1e12 / peak_, 3) if gemm_ms else None,
                                  "busy_ms": round(busy, 2)}
    ex.kernel_timing(False)
    ex.set_serial(args.serial == "on")
    samples = args.steps * args.minibatches * args.batch
    value = samples / (ms * 1e-3)
    # ---------------- traced step: bubble / utilisation with the reference's window rule
    _phase("traced step + e2e")
    barrier()
    torch.cuda.synchronize()
    ex.step(stream=stream, trace=True)
    res = ex.result()
    # ---------------- e2e through the public API with host buffers
    if args.workload == "gpt":
        X_host = torch.randint(0, spec.vocab, (spec.n_blocks, spec.batch, spec.seq), dtype=torch.int32).pin_memory()
    else:
        X_host = torch.randn(spec.n_blocks, spec.batch, spec.widths[0]).to(torch.bfloat16).pin_memory()
    if args.workload == "gpt":
        T_host = torch.randint(0, spec.vocab, (spec.n_blocks, spec.batch, spec.seq), dtype=torch.int32).pin_memory()
    elif args.workload == "vgg":
        T_host = torch.randint(0, spec.classes, (spec.n_blocks, spec.batch), dtype=torch.int32).pin_memory()
    else:
        T_host = torch.randn(spec.n_blocks, spec.batch, spec.widths[-1]).pin_memory()
    loss_host = torch.empty(args.minibatches + 1, dtype=torch.float32).pin_memory()
    hosts_first = ex.hosts_stage(0)
    hosts_last = ex.hosts_stage(cfg.plan.num_stages - 1)
    h2d = (X_host.numel() * X_host.element_size() if hosts_first else 0) + \
          (T_host.numel() * T_host.element_size() if hosts_last else 0)
    d2h = loss_host.numel() * 4 if hosts_last else 0

    def e2e_step():
        ex.load_inputs(X_host if hosts_first else None, T_host if hosts_last else None, stream=stream)
        ex.step(stream=stream)
        if hosts_last:
            loss_host.copy_(ex.loss_tensor(), non_blocking=True)

    # one untimed e2e step first: the serial roofline pass above dropped the CUDA graph, and its
    # re-capture belongs in warm-up, not in the timed region
    e2e_step()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if dist is not None:
        e2e_ms = reduce([e2e_ms], dist.ReduceOp.MAX)[0]
    e2e_value = args.e2e_steps * args.minibatches * args.batch / (e2e_ms * 1e-3)
    gpus_active = 1
    if dist is not None:  # whole-job counts
        h2d, d2h, launches = [int(x) for x in reduce([float(h2d), float(d2h), float(launches)], dist.ReduceOp.SUM)]
        devs = [None] * world
        dist.all_gather_object(devs, str(getattr(torch.cuda.get_device_properties(dev), "uuid", dev)))
        gpus_active = len({str(d) for d in devs})
    if rank != 0:
        ex.close()
        return
    # ---------------- roofline for the dominant kernel class (largest total GEMM time)
    peaks, peak_kind = load_peaks()
    peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")))
    gemm_stats = {k: v for k, v in kstats.items() if k in ("fwd", "dgrad", "wgrad_sgd")}
    kernel_time = {k: round(v["total_ms"], 3) for k, v in kstats.items()}
    dom_name, dom = max(gemm_stats.items(), key=lambda kv: kv[1]["total_ms"])
    achieved = dom["flops_per_launch"] / (dom["avg_ms"] * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tr = json.load(fh)
        if args.workload == "mlp" and tr.get("batch") == args.batch and tr.get("width") == args.width:
            traffic = tr.get(dom_name)
    per_class = {k: {"launches": v["launches"], "avg_ms": round(v["avg_ms"], 4),
                     "tflops": round(v["flops_per_launch"] / (v["avg_ms"] * 1e-3) / 1e12, 1),
                     "frac_of_sustained_peak": round(v["flops_per_launch"] / (v["avg_ms"] * 1e-3) / 1e12 / peak, 3)}
                 for k, v in gemm_stats.items()}
    flops_per_sample = spec.flops_per_sample()
    rep = res.report
    out = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "config": workload(args),
        "roofline": {"bound": "tensor",
                     "kernel": f"k_gemm_tc ({dom_name}{', conv + linear' if args.workload == 'vgg' else ''})",
                     "flops_per_launch": dom["flops_per_launch"], "avg_launch_ms": dom["avg_ms"],
                     "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": f"{peak_kind} bf16_tflops_sustained (MEASURED_PEAKS.json)"},
        "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "gemm_classes": per_class,
        "kernel_time_ms_serial_step": kernel_time,
        "stage_tc_util": stage_util,
        "stage_tc_util_definition": "per worker: GEMM algorithmic FLOPs / serial kernel time / measured sustained "
                                    "bf16 peak (tc_util_busy over all its kernels, tc_util_gemm over its GEMMs only)",
        "model_tflops": value * flops_per_sample / 1e12,
        "model_frac_of_sustained_peak": value * flops_per_sample / 1e12 / peak / world,
        "gpus_active": gpus_active,
        "bubble_fraction": res.extras.get("bubble_fraction"),
        "bubble_fraction_whole_run": res.extras.get("bubble_fraction_whole_run"),
        "bubble_definition": "1 - fraction of the reference's steady window (simulator.py:361-385) in which the GPU "
                             "runs a pass (union over its hosted stages), mean over GPUs; whole_run: the same over "
                             "each GPU's first pass start .. last pass end, including pipeline fill and drain",
        "p2p": p2p_summary(res, args),
        "per_worker_utilization": [round(u, 4) for u in rep.per_worker_utilization] if rep else None,
        "steady_minibatches_per_s": rep.steady_throughput if rep else None,
    }
    if not args.no_cpu_baseline:
        _phase("cpu baseline (child process)")
        out["cpu_baseline"] = cpu_baseline_isolated(args)
    ex.close()
    _phase("done")
    print(json.dumps(out), flush=True)


def self_launch(args) -> int:
    """`python bench.py --gpus N` outside torchrun: run N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1; rank 0's JSON line goes to stdout."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    _phase(f"launching {args.gpus} ranks: {' '.join(cmd[1:6])} ...")
    return subprocess.run(cmd).returncode


def p2p_summary(res, args):
    """Inter-stage payload bytes stored into other processes' inboxes during the traced step,
    counted by the storing kernels (pd_rt_set_records), per pipeline boundary, and the average
    rate over the traced step.  Zero at N=1 (every boundary is on one GPU)."""
    by = res.extras.get("p2p_bytes_by_boundary") or {}
    span = max((ev.time_end for ev in res.trace), default=0.0)
    return {"bytes_traced_step": res.extras.get("p2p_bytes_measured"),
            "bytes_by_boundary": by,
            "avg_gbs_by_boundary": {k: (v / span / 1e9 if span else None) for k, v in by.items()},
            "definition": "boundary s = stages s|s+1, both directions; GB/s averaged over the traced step"}


def apply_workload_defaults(args):
    if args.workload == "gpt":
        if "--batch" not in sys.argv:
            args.batch = 8  # sequences of 1024 tokens per minibatch
        if "--minibatches" not in sys.argv:
            args.minibatches = 128  # fill/drain 7/135 at 8 GPUs; >= 25 for the reference's steady window
    if args.workload == "vgg":
        if "--batch" not in sys.argv:
            args.batch = 32
        if "--minibatches" not in sys.argv:
            args.minibatches = 126  # 18 allreduce rounds of 7; >= 37 for the reference's steady window
    return args


def main():
    args = apply_workload_defaults(parse())
    # a stuck run prints every thread's Python stack on stderr (the device side traps on its own:
    # mbarrier waits give up after 20 s, flag waits after 10 s)
    faulthandler.dump_traceback_later(float(os.environ.get("PD_BENCH_WATCHDOG_S", "600")), exit=False)
    if args.cpu_sample_only:
        _all_host_threads()
        out = _cpu_sample_for(args)
        out["cpu_model"] = cpu_model()
        out["host_cpus"] = os.cpu_count()
        try:
            out["reference_simulator"] = reference_simulator_sample(args)
        except Exception as e:  # the baseline is reported, never fatal
            out["reference_simulator"] = {"available": False, "why": f"{type(e).__name__}: {e}"}
        print(json.dumps(out), flush=True)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: refusing to report a different GPU count",
              file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch

        ngpu = torch.cuda.device_count()
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % ngpu)
        # host plumbing only (IPC handle exchange, barriers, max-over-ranks); the data path is
        # peer stores + flags.  Several ranks per GPU (functional testing) cannot use NCCL.
        torch.distributed.init_process_group("nccl" if ngpu >= world else "gloo")
    run_ours(args, rank, world)
    if world > 1:
        import torch

        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
