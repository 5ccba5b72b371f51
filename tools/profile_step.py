"""Build a bench workload and run N plain steps (no timing, no trace): the target for ncu launch lists.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file out.csv \
        python tools/profile_step.py --workload gpt --minibatches 25 --steps 1
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402


def main():
    args = bench.apply_workload_defaults(bench.parse())
    import torch

    import paper_1806_03377_b200 as pd

    cfg, spec = bench.build_config(args)
    ex = pd.Executor(cfg, model=spec)
    ex.set_serial(args.serial == "on")
    for _ in range(args.steps):
        ex.step()
    torch.cuda.synchronize()
    print("launches", ex.launch_count())
    ex.close()


if __name__ == "__main__":
    main()
