"""Host enqueue cost of the async count path vs the GPU time per call."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_01506_b200 import _native, workloads  # noqa: E402

for cfg in [int(c) for c in (sys.argv[1:] or ["5", "2", "3"])]:
    w = workloads.make(cfg)
    ctx = _native.context(0)
    dh = ctx.dfa(w.dfa)
    sh = ctx.upload_ascii(w.ascii)
    out = torch.zeros(max(dh.n_expressions, 1), dtype=torch.int64).pin_memory()
    out_np = out.numpy()
    for _ in range(5):
        ctx.count_async(dh, sh, out_np)
    ctx.async_wait()
    for steps in (1, 20):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        for _ in range(steps):
            ctx.count_async(dh, sh, out_np)
        t1 = time.perf_counter()
        e1.record()
        wt = ctx.async_wait()
        torch.cuda.synchronize()
        print(f"C{cfg} steps={steps}: host enqueue {(t1 - t0) / steps * 1e6:.1f} us/call, "
              f"gpu {e0.elapsed_time(e1) / steps * 1e3:.1f} us/call, scan_ms/call {wt['scan_ms_total'] / steps * 1e3:.1f} us, "
              f"launches/call {wt['kernel_launches'] / steps:.1f}", flush=True)
    del sh, dh
