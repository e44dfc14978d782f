"""Locate (count + sorted match rows) throughput on a device-resident sequence."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_01506_b200 import _native, workloads  # noqa: E402

for cfg in [int(c) for c in (sys.argv[1:] or ["2", "4"])]:
    w = workloads.make(cfg)
    ctx = _native.context(0)
    dh = ctx.dfa(w.dfa)
    sh = ctx.upload_ascii(w.ascii)
    c0 = ctx.count(dh, sh)
    counts, rows = ctx.locate(dh, sh)
    assert counts.tolist() == c0.tolist() and rows.shape[0] == int(c0.sum())
    for name, fn in (("count", lambda: ctx.count(dh, sh)), ("locate", lambda: ctx.locate(dh, sh))):
        ts = []
        for _ in range(10):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        st = ctx.stats()
        t = float(np.median(ts))
        print(f"C{cfg} {name}: {w.n / t / 1e9:.0f} GB/s wall ({t * 1e3:.3f} ms), scan_ms {st['scan_ms']:.3f}, "
              f"total_ms {st['total_ms']:.3f}, launches {st['kernel_launches']}, rows {rows.shape[0]}")
