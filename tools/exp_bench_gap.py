import sys, time
sys.path.insert(0,'.')
import numpy as np, torch
from paper_1509_01506_b200 import _native, workloads
import bench
w = workloads.make(3)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
ctx = _native.context(0); ctx.set_stream(stream.cuda_stream)
dh = ctx.dfa(w.dfa); sh = ctx.upload_ascii(w.ascii)
out = torch.zeros(max(dh.n_expressions,1), dtype=torch.int64).pin_memory(); out_np = out.numpy()
def run(n, sampler=False, idle=0.0, warm=5):
    for _ in range(warm): ctx.count_async(dh, sh, out_np)
    ctx.async_wait(); torch.cuda.synchronize()
    if idle: time.sleep(idle)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    cs = bench.ClockSampler(0).prepare() if sampler else None
    if cs: cs.__enter__()
    e0.record(stream)
    for _ in range(n): ctx.count_async(dh, sh, out_np)
    e1.record(stream)
    ctx.async_wait(); torch.cuda.synchronize()
    if cs: cs.__exit__()
    return e0.elapsed_time(e1)/n
ea = torch.cuda.Event(enable_timing=True); eb = torch.cuda.Event(enable_timing=True)
for _ in range(5): ctx.count_async(dh, sh, out_np)
ctx.async_wait(); torch.cuda.synchronize()
import os
if os.environ.get("PRIMER") == "events":
    ea.record(stream); eb.record(stream); eb.synchronize(); print("primer events only", ea.elapsed_time(eb))
elif os.environ.get("PRIMER") == "kernel":
    ea.record(stream); ctx.count_async(dh, sh, out_np); eb.record(stream); ctx.async_wait(); torch.cuda.synchronize(); print("primer events+kernel", ea.elapsed_time(eb))
elif os.environ.get("PRIMER") == "wait":
    ctx.count_async(dh, sh, out_np); ctx.async_wait(); torch.cuda.synchronize(); time.sleep(0.5); print("primer: one more call, 0.5 s pause")
for label, kw in (("first region", {"warm": 5}), ("plain", {}), ):
    print(label, [round(run(20, **kw), 5) for _ in range(5 if "first" not in label else 1)], flush=True)

