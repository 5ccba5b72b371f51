"""cfg5 P2P microbench: activation hand-off bandwidth vs message size (64 KiB .. 256 MiB).

Two ranks (one process per GPU).  Rank 0 plays the producer stage, rank 1 the consumer.
For each message size it measures, on rank 0's stream with CUDA events:
  * store+flag : the runtime's hand-off path, i.e. a copy kernel storing the payload straight into
                 the peer-mapped inbox (what a GEMM epilogue does), then the system-scope release
                 flag (pd_flag_signal) that the consumer acquire-polls;
  * memcpy     : cudaMemcpyAsync device->peer-mapped device (the copy-engine path) for comparison.
Unidirectional GB/s = bytes / time.  On a single GPU (two ranks sharing it) the numbers are
same-device IPC copies, not NVLink; the JSON says which.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 tools/p2p_bench.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_03377_b200 import _native as nat  # noqa: E402


def main():
    ngpu = torch.cuda.device_count()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    torch.distributed.init_process_group("nccl" if ngpu >= world else "gloo")
    rank = torch.distributed.get_rank()
    dev = rank % ngpu
    torch.cuda.set_device(dev)
    sizes = [1 << k for k in range(16, 29)]  # 64 KiB .. 256 MiB
    cap = sizes[-1]
    inbox = torch.zeros(cap, dtype=torch.uint8, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    src = torch.randint(0, 255, (cap,), dtype=torch.uint8, device="cuda")
    handles = [None] * world
    torch.distributed.all_gather_object(handles, (nat.ipc_export(inbox), nat.ipc_export(flag)))
    rows = []
    if rank == 0:
        (h_in, o_in), (h_fl, o_fl) = handles[1]
        peer_inbox = nat.ipc_import(h_in, o_in)
        peer_flag = nat.ipc_import(h_fl, o_fl)
        lib = nat.lib()
        stream = torch.cuda.current_stream()
        for n in sizes:
            reps = max(3, min(200, (64 << 20) // n))
            for mode in ("store+flag", "memcpy"):
                def once(i):
                    if mode == "memcpy":
                        nat.check(lib.pd_memcpy_async(peer_inbox, src.data_ptr(), n, stream.cuda_stream), "memcpy")
                    else:
                        # the hand-off path: SM stores into the peer inbox (16-byte vectors), then the
                        # system-scope release flag the consumer acquire-polls
                        nat.check(lib.pd_copy(peer_inbox, src.data_ptr(), n, stream.cuda_stream), "payload store")
                        nat.check(lib.pd_flag_signal(peer_flag, i + 1, stream.cuda_stream), "flag")
                for i in range(3):
                    once(i)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record()
                for i in range(reps):
                    once(i)
                b.record()
                torch.cuda.synchronize()
                ms = a.elapsed_time(b) / reps
                rows.append({"bytes": n, "mode": mode, "us": ms * 1e3, "GBps": n / (ms * 1e-3) / 1e9})
    torch.distributed.barrier()
    if rank == 0:
        print(json.dumps({"p2p": rows, "same_device": ngpu < world,
                          "note": "same-device IPC (not NVLink)" if ngpu < world else "peer GPUs over NVLink"}))
    torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
