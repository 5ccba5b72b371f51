"""Reliability loop: run many back-to-back schedule executions of the bench workloads in one process
and report per-step times, so a stall (the round-1 "2 of 40 bench runs" hang) shows up as a step far
above the median or as the mbarrier / flag watchdog firing.  Every 10th step is traced (device
ledger + records path) and its ledger is checked against the program's resolution.

    python tools/reliability_loop.py --steps 100 --workloads mlp,vgg,gpt [--minibatches K]
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--workloads", default="mlp,vgg,gpt")
    p.add_argument("--minibatches", type=int, default=0, help="per step (default: mlp 64, vgg 63, gpt 32)")
    a = p.parse_args()
    import numpy as np
    import torch

    import paper_1806_03377_b200 as pd

    out = {}
    for w in a.workloads.split(","):
        k = a.minibatches or {"mlp": 64, "vgg": 63, "gpt": 32}[w]
        sys.argv = ["bench.py", "--workload", w, "--minibatches", str(k)]
        args = bench.apply_workload_defaults(bench.parse())
        cfg, spec = bench.build_config(args)
        ex = pd.Executor(cfg, model=spec)
        times, traced_ok = [], 0
        try:
            for i in range(a.steps):
                t0 = time.perf_counter()
                trace = i % 10 == 9
                ex.step(trace=trace)
                torch.cuda.synchronize()
                times.append(time.perf_counter() - t0)
                if trace:
                    res = ex.result()
                    assert res.ledger.entries == ex.program.ledger.entries
                    assert np.all(np.isfinite(res.losses))
                    traced_ok += 1
        finally:
            ex.close()
            torch.cuda.empty_cache()
        t = np.array(times[1:])
        out[w] = {"steps": a.steps, "minibatches_per_step": k, "median_s": float(np.median(t)),
                  "max_s": float(t.max()), "max_over_median": float(t.max() / np.median(t)),
                  "traced_steps_checked": traced_ok}
        print(w, json.dumps(out[w]), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
