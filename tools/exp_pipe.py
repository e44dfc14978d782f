"""One-GPU proxy of the multi-GPU step (gpurun): a one-rank NCCL group, a C4
shard, 50 timed steps of (a) scans only, (b) scan + all-reduce on the scan
stream, (c) bench.py's PipelinedAllReduce (flag-gated side stream).

    N=400000000 python tools/exp_pipe.py
"""
import os
import socket
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench as B  # noqa: E402
from paper_1509_01506_b200 import _native, workloads  # noqa: E402

with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
dev = torch.device("cuda", 0)
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=dev)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
ctx = _native.DeviceContext(0)
ctx.set_stream(stream.cuda_stream)
ctx.set_reserved_sms(int(os.environ.get("RES", "2")))
n = int(os.environ.get("N", "400000000"))
w = workloads.make(4, n)
dh = ctx.dfa(w.dfa)
sh = ctx.upload_ascii(w.ascii)
ne = w.dfa.n_expressions
buf = torch.zeros(max(ne, 1), dtype=torch.int64, device=dev)
pin = torch.zeros(max(ne, 1), dtype=torch.int64).pin_memory()
pipe = B.PipelinedAllReduce(ne, dev, pin)


def a():
    ctx.count_shard_async(dh, sh, 0, n, 0, 0, buf.data_ptr())


def b():
    ctx.count_shard_async(dh, sh, 0, n, 0, 0, buf.data_ptr())
    dist.all_reduce(buf)


def c():
    pipe.step(lambda cp, fp, v: ctx.count_shard_async_signal(dh, sh, 0, n, 0, 0, cp, fp, v))


for name, fn, fin in (("scan only", a, None), ("scan+allreduce same stream", b, None),
                      ("pipelined (flag-gated side stream)", c, pipe.finish)):
    for rep in range(2):
        for _ in range(5):
            fn()
        if fin:
            fin()
        ctx.async_wait()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(50):
            fn()
        if fin:
            fin()
        e1.record(stream)
        ctx.async_wait()
        torch.cuda.synchronize()
        print(f"{name}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us/step (n={n})", flush=True)
dist.destroy_process_group()
