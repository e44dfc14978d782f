"""Per-phase device times of a count: KS_PHASE_TRACE=1 (synchronous calls)
and KS_PHASE_TRACE=2 (back-to-back async calls, printed at async_wait)."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_01506_b200 import _native, workloads  # noqa: E402

for cfg in [int(c) for c in (sys.argv[1:] or ["5"])]:
    w = workloads.make(cfg)
    ctx = _native.context(0)
    dh = ctx.dfa(w.dfa)
    sh = ctx.upload_ascii(w.ascii)
    for _ in range(3):
        ctx.count(dh, sh)
    os.environ["KS_PHASE_TRACE"] = "1"
    print(f"C{cfg} sync count:", flush=True)
    ctx.count(dh, sh)
    out = torch.zeros(max(dh.n_expressions, 1), dtype=torch.int64).pin_memory().numpy()
    os.environ["KS_PHASE_TRACE"] = "2"
    print(f"C{cfg} 4 async counts:", flush=True)
    for _ in range(4):
        ctx.count_async(dh, sh, out)
    print(ctx.async_wait(), flush=True)
    os.environ["KS_PHASE_TRACE"] = "0"
