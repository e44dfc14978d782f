"""Wall time and device phases (KS_PHASE_TRACE=1) of ks_locate."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_01506_b200 import _native, workloads  # noqa: E402

for cfg in [int(c) for c in (sys.argv[1:] or ["2"])]:
    w = workloads.make(cfg)
    ctx = _native.context(0)
    dh = ctx.dfa(w.dfa)
    sh = ctx.upload_ascii(w.ascii)
    for _ in range(3):
        ctx.locate(dh, sh)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        c, rows = ctx.locate(dh, sh)
        ts.append(time.perf_counter() - t0)
    st = ctx.stats()
    print(f"C{cfg} locate wall {np.median(ts) * 1e3:.3f} ms, total_ms {st['total_ms']:.3f}, scan_ms {st['scan_ms']:.3f}, rows {rows.shape[0]}", flush=True)
    t0 = time.perf_counter(); ctx.count(dh, sh); t1 = time.perf_counter()
    print(f"C{cfg} count wall {(t1 - t0) * 1e3:.3f} ms", flush=True)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); ctx.count(dh, sh); ts.append(time.perf_counter() - t0)
    st = ctx.stats()
    print(f"C{cfg} count wall x5 {[round(t * 1e3, 3) for t in ts]} ms, total_ms {st['total_ms']:.3f}, scan_ms {st['scan_ms']:.3f}", flush=True)
    os.environ["KS_PHASE_TRACE"] = "1"
    print("locate phases:", flush=True)
    ctx.locate(dh, sh)
    print("count phases:", flush=True)
    ctx.count(dh, sh)
    os.environ["KS_PHASE_TRACE"] = "0"
