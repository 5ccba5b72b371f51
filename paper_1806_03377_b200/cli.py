"""Command line: ``python -m paper_1806_03377_b200 {profile,plan,simulate,compare}``.

Mirrors the reference CLI (pipesim/cli.py:264-358) for the hot path, with the B200 executor as
the backend of ``simulate``: same positional arguments, options, artefact
names (report.json, trace.csv, staleness.json, each JSON carrying a run manifest), stdout lines
and exit codes (0 ok, 1 usage, 2 validation, 3 simulation).  Differences: ``--model`` names the
network the stages train (the reference has no tensors), ``profile`` measures a layer profile on
the GPU instead of synthesising one, and ``--checkpoint-dir`` / ``--resume`` write / read per-stage
weight checkpoints at the end of the run without global coordination.

Model specs: ``mlp:WIDTH:LAYERS[:BATCH[:DTYPE]]``, ``vgg16[:BATCH]``, ``gpt2-medium[:BATCH]``,
``gpt:VOCAB:D:HEADS:LAYERS:SEQ[:BATCH]``.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

from . import __version__
from .errors import SimulationError, ValidationError

EXIT_OK, EXIT_USAGE, EXIT_VALIDATION, EXIT_SIMULATION = 0, 1, 2, 3


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 1, as the reference documents (cli.py:44-49)
        self.print_usage(sys.stderr)
        print(f"{self.prog}: error: {message}", file=sys.stderr)
        raise SystemExit(EXIT_USAGE)


def parse_model(text: str, lr: float | None = None, seed: int = 0):
    """Model spec string -> MLPSpec / ConvNetSpec / GPTSpec."""
    from . import models

    parts = text.split(":")
    kw = {"seed": seed}
    if lr is not None:
        kw["lr"] = lr
    try:
        if parts[0] == "mlp":
            width, layers = int(parts[1]), int(parts[2])
            batch = int(parts[3]) if len(parts) > 3 else 32
            dtype = parts[4] if len(parts) > 4 else "bf16"
            return models.mlp(width, layers, batch=batch, dtype=dtype, **kw)
        if parts[0] == "vgg16":
            return models.vgg16(batch=int(parts[1]) if len(parts) > 1 else 32, **kw)
        if parts[0] == "gpt2-medium":
            return models.gpt2_medium(batch=int(parts[1]) if len(parts) > 1 else 8, **kw)
        if parts[0] == "gpt":
            v, d, h, n, s = (int(x) for x in parts[1:6])
            batch = int(parts[6]) if len(parts) > 6 else 8
            return models.GPTSpec(vocab=v, d=d, heads=h, layers=n, seq=s, batch=batch, **kw)
    except (IndexError, ValueError) as exc:
        raise ValidationError(f"bad model spec {text!r}: {exc}") from exc
    raise ValidationError(f"unknown model spec {text!r} (mlp:W:L[:B[:dtype]] | vgg16[:B] | gpt2-medium[:B] | "
                          "gpt:V:D:H:L:S[:B])")


def _manifest(command: str, args) -> dict:
    inputs = {k: v for k, v in sorted(vars(args).items()) if k not in ("func", "command") and v is not None}
    return {"command": command, "backend": "b200", "inputs": {k: str(v) if isinstance(v, Path) else v
                                                               for k, v in inputs.items()},
            "tool_version": __version__, "seed": getattr(args, "seed", 0)}


def _write_json(path: Path, manifest: dict, payload: dict) -> None:
    doc = {"manifest": manifest}
    doc.update(payload)
    path.write_text(json.dumps(doc, indent=2, sort_keys=True) + "\n")


def _out_dir(args) -> Path:
    out = Path(args.out_dir)
    out.mkdir(parents=True, exist_ok=True)
    return out


def cmd_profile(args) -> int:
    from .profiler import profile_model
    from .profiles import save_profile

    spec = parse_model(args.model, seed=args.seed)
    prof = profile_model(spec, minibatches=args.minibatches, steps=args.steps)
    out = Path(args.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    save_profile(prof, out)
    print(f"profile: {out}")
    print(f"layers: {prof.num_layers}")
    print(f"total_time: {prof.total_time:.6f} s")
    print(f"total_param_elems: {prof.total_param_elems}")
    return EXIT_OK


def cmd_plan(args) -> int:
    from .plans import solve
    from .profiles import HardwareSpec, build_context, comm_volume_bsp, comm_volume_pp, load_profile

    ctx = build_context(load_profile(args.profile), HardwareSpec(args.machines, args.bandwidth, args.bytes_per_elem))
    plan = solve(ctx, force_all_machines=args.force_all_machines,
                 max_replication=1 if args.straight else None)
    bsp, pp = comm_volume_bsp(ctx, args.machines), comm_volume_pp(ctx, plan)
    out = _out_dir(args)
    path = out / "plan.json"
    _write_json(path, _manifest("plan", args), plan.to_dict() | {"config": plan.config_string})
    print(f"config: {plan.config_string}")
    print(f"stages: {plan.num_stages}")
    print(f"machines_used: {plan.machines_used}")
    print(f"bottleneck_time: {plan.bottleneck_time:.9f} s")
    print(f"noam: {plan.noam}")
    print(f"predicted_throughput: {1.0 / plan.bottleneck_time:.6f} minibatches/s")
    print(f"comm_bsp_bytes: {bsp:.0f}")
    print(f"comm_pp_bytes: {pp:.0f}")
    print(f"comm_reduction: {100.0 * (1.0 - pp / bsp):.1f}%" if bsp > 0 else "comm_reduction: n/a (no comm)")
    print(f"plan_file: {path}")
    return EXIT_OK


def cmd_simulate(args) -> int:
    from .executor import Executor
    from .ledger import Mode, SimConfig, compare_analytic, staleness_check, write_trace_csv
    from .plans import load_plan
    from .profiles import HardwareSpec, build_context, load_profile

    profile = load_profile(args.profile)
    plan = load_plan(args.plan)
    if plan.num_layers != profile.num_layers:
        raise ValidationError(f"plan covers {plan.num_layers} layers but profile has {profile.num_layers}")
    ctx = build_context(profile, HardwareSpec(plan.machines_used, args.bandwidth, args.bytes_per_elem))
    cfg = SimConfig(plan=plan, mode=Mode(args.mode), num_minibatches=args.minibatches, max_inflight=args.max_inflight)
    spec = parse_model(args.model, lr=args.lr, seed=args.seed)
    ex = Executor(cfg, ctx, model=spec)
    try:
        if args.resume:
            ex.load_checkpoint(args.resume)
        for _ in range(max(0, args.steps - 1)):  # extra training steps (untraced)
            ex.step()
        ex.step(trace=True)
        result = ex.result()
        if args.checkpoint_dir:
            ex.save_checkpoint(args.checkpoint_dir)
    finally:
        ex.close()
    manifest = _manifest("simulate", args)
    out = _out_dir(args)
    _write_json(out / "report.json", manifest, result.report.to_dict() | {
        "losses": result.losses, "bubble_fraction": result.extras.get("bubble_fraction")})
    write_trace_csv(result.trace, out / "trace.csv", header_comment="manifest: " + json.dumps(manifest, sort_keys=True))
    checked = result.ledger.is_straight and cfg.effective_inflight == plan.noam
    violations = staleness_check(result.ledger, cfg.mode, plan.num_stages) if checked else []
    _write_json(out / "staleness.json", manifest, {"checked": checked, "violations": [
        {"stage": v.stage_index, "minibatch": v.minibatch_id, "direction": v.direction.value, "expected": v.expected,
         "actual": v.actual} for v in violations]})
    print(f"mode: {cfg.mode.value}")
    print(f"makespan: {result.report.makespan:.9f} s")
    print(f"steady_throughput: {result.report.steady_throughput:.6f} minibatches/s")
    print(f"throughput_vs_analytic_error: {compare_analytic(result.report, plan):.4%}")
    print(f"comm_bytes_total: {result.report.comm_bytes_total:.0f}")
    print(f"staleness_violations: {len(violations)}" if checked else
          "staleness_violations: n/a (replicated plan or reduced max-inflight)")
    print(f"report_file: {out / 'report.json'}")
    if not checked:
        return EXIT_OK
    if cfg.mode is Mode.NAIVE_PIPELINE and args.expect_naive:
        if not violations:
            print("error: naive mode unexpectedly produced a consistent ledger", file=sys.stderr)
            return EXIT_VALIDATION
        return EXIT_OK
    if violations:
        print(f"error: staleness check failed with {len(violations)} violations", file=sys.stderr)
        return EXIT_VALIDATION
    return EXIT_OK


def _regime_minibatches(plan, k: int) -> int:
    """Smallest K' >= k that is a whole number of rounds of every replicated stage (the round rule)."""
    from math import lcm

    step = 1
    for st in plan.stages:
        step = lcm(step, st.replication)
    return -(-k // step) * step


def cmd_compare(args) -> int:
    """The reference's regime comparison (cli.py:211-261: single machine, model parallel, data
    parallel, straight pipeline, full plan) with every regime EXECUTED on the B200 runtime instead
    of simulated: each plan runs through the executor (its workers spread over this job's ranks; at
    one GPU all of them share it) and the measured steady throughput is reported next to the
    planner's analytic 1 / bottleneck_time.  Speed-ups are relative to the measured single-machine
    run, as in the reference."""
    import torch

    from .executor import Executor
    from .ledger import Mode, SimConfig
    from .plans import Plan, Stage, solve
    from .profiles import HardwareSpec, build_context, load_profile, stage_time

    profile = load_profile(args.profile)
    machines = args.machines
    ctx = build_context(profile, HardwareSpec(machines, args.bandwidth, args.bytes_per_elem))
    n = profile.num_layers
    spec = parse_model(args.model, lr=args.lr, seed=args.seed)
    if getattr(spec, "num_layers", n) != n:
        raise ValidationError(f"model has {spec.num_layers} layers but profile has {n}")

    def single_stage(m: int) -> Plan:
        return Plan(stages=(Stage(1, n, m),), bottleneck_time=stage_time(ctx, 1, n, m), noam=1, machines_used=m)

    straight = solve(ctx, machines=min(machines, n), max_replication=1)
    regimes = [("single_machine", single_stage(1), None), ("model_parallel", straight, 1),
               ("data_parallel", single_stage(machines), None), ("straight_pipeline", straight, None),
               ("full_plan", solve(ctx, machines=machines), None)]
    rows = []
    for name, plan, inflight in regimes:
        k = _regime_minibatches(plan, args.minibatches)
        cfg = SimConfig(plan=plan, mode=Mode.WEIGHT_STASHING, num_minibatches=k, max_inflight=inflight)
        ex = Executor(cfg, ctx, model=spec)
        try:
            for _ in range(max(0, args.steps - 1)):
                ex.step()
            ex.step(trace=True)
            res = ex.result()
        finally:
            ex.close()
            torch.cuda.empty_cache()
        rows.append({"regime": name, "config": plan.config_string, "minibatches": k,
                     "max_inflight": cfg.effective_inflight, "throughput": res.report.steady_throughput,
                     "samples_per_s": res.report.steady_throughput * spec.batch,
                     "predicted_throughput": 1.0 / plan.bottleneck_time,
                     "bubble_fraction": res.extras.get("bubble_fraction")})
    base = rows[0]["throughput"]
    world = int(__import__("os").environ.get("WORLD_SIZE", "1"))
    print(f"{'regime':<18} {'config':<12} {'throughput/s':>14} {'speedup':>9} {'predicted/s':>12}")
    for r in rows:
        r["speedup"] = r["throughput"] / base
        print(f"{r['regime']:<18} {r['config']:<12} {r['throughput']:>14.6f} {r['speedup']:>8.2f}x "
              f"{r['predicted_throughput']:>12.6f}")
    out = _out_dir(args)
    _write_json(out / "compare.json", _manifest("compare", args), {
        "machines": machines, "n_gpus": world, "regimes": rows,
        "note": "measured on the B200 runtime; with fewer GPUs than workers, workers share GPUs"})
    print(f"compare_file: {out / 'compare.json'}")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    parser = _Parser(prog="python -m paper_1806_03377_b200", description="B200 pipeline-parallel training runtime")
    parser.add_argument("--version", action="version", version=f"paper_1806_03377_b200 {__version__}")
    sub = parser.add_subparsers(dest="command", parser_class=_Parser)
    sub.required = True

    p = sub.add_parser("profile", help="measure a per-layer profile on the GPU (reference JSON format)")
    p.add_argument("--model", required=True)
    p.add_argument("--minibatches", type=int, default=11)
    p.add_argument("--steps", type=int, default=2)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", default="profile.json")
    p.set_defaults(func=cmd_profile)

    p = sub.add_parser("plan", help="PipeDream partitioner (solve) on a profile")
    p.add_argument("profile")
    p.add_argument("--machines", type=int, required=True)
    p.add_argument("--bandwidth", type=float, default=770e9, help="bytes/s (default: measured B200 NVLink copy)")
    p.add_argument("--bytes-per-elem", type=int, default=2)
    p.add_argument("--force-all-machines", action="store_true")
    p.add_argument("--straight", action="store_true", help="replication 1 for every stage")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out-dir", default=".")
    p.set_defaults(func=cmd_plan)

    p = sub.add_parser("simulate", help="execute a plan on B200s (the drop-in for pipesim simulate)")
    p.add_argument("plan")
    p.add_argument("profile")
    p.add_argument("--model", required=True)
    p.add_argument("--bandwidth", type=float, default=770e9)
    p.add_argument("--bytes-per-elem", type=int, default=2)
    p.add_argument("--mode", default="weight_stashing", choices=["naive_pipeline", "weight_stashing", "vertical_sync"])
    p.add_argument("--minibatches", type=int, default=32)
    p.add_argument("--max-inflight", type=int, default=None)
    p.add_argument("--lr", type=float, default=None)
    p.add_argument("--steps", type=int, default=1, help="schedule executions (the last one is traced)")
    p.add_argument("--expect-naive", action="store_true")
    p.add_argument("--checkpoint-dir", default=None, help="write per-stage weight checkpoints after the run")
    p.add_argument("--resume", default=None, help="load per-stage checkpoints before the run")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out-dir", default=".")
    p.set_defaults(func=cmd_simulate)

    p = sub.add_parser("compare", help="execute the reference's five training regimes on the B200 runtime")
    p.add_argument("profile")
    p.add_argument("--model", required=True)
    p.add_argument("--machines", type=int, required=True)
    p.add_argument("--bandwidth", type=float, default=770e9)
    p.add_argument("--bytes-per-elem", type=int, default=2)
    p.add_argument("--minibatches", type=int, default=32)
    p.add_argument("--lr", type=float, default=None)
    p.add_argument("--steps", type=int, default=2, help="schedule executions per regime (the last one is traced)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out-dir", default=".")
    p.set_defaults(func=cmd_compare)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except ValidationError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_VALIDATION
    except SimulationError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_SIMULATION
