"""Back-to-back async counts (the bench's step) per config under env
variants: GPU time per call from CUDA events around 20 enqueued calls.

    python tools/exp_b2b.py 3,4 base KS_EARLY_WAIT=1
"""
import json
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_01506_b200 import _native, workloads  # noqa: E402

cfgs = [int(c) for c in sys.argv[1].split(",")]
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
variants = sys.argv[2:] or ["base"]
for cfg in cfgs:
    w = workloads.make(cfg, int(os.environ["N"]) if os.environ.get("N") else None)
    ctx = _native.context(0)
    ctx.set_stream(stream.cuda_stream)   # events and scans on one stream
    dh = ctx.dfa(w.dfa)
    sh = ctx.upload_ascii(w.ascii)
    want = ctx.count(dh, sh)
    out = torch.zeros(max(dh.n_expressions, 1), dtype=torch.int64).pin_memory()
    out_np = out.numpy()
    for rnd in range(2):
        for v in variants:
            env = dict(kv.split("=", 1) for kv in v.split(",") if "=" in kv)
            saved = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            try:
                per = []
                for rep in range(5):
                    for _ in range(3):
                        ctx.count_async(dh, sh, out_np)
                    ctx.async_wait()
                    torch.cuda.synchronize()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    s = torch.cuda.current_stream()
                    e0.record(s)
                    for _ in range(20):
                        ctx.count_async(dh, sh, out_np)
                    e1.record(s)
                    ctx.async_wait()
                    torch.cuda.synchronize()
                    per.append(e0.elapsed_time(e1) / 20)
                    assert os.environ.get("NOCHECK") or np.array_equal(out_np[:want.size], want), v
                med = statistics.median(per)
                print(json.dumps({"cfg": cfg, "round": rnd, "variant": v, "ms_per_call": round(med, 5),
                                  "gbases_per_s": round(w.n / med / 1e6, 1)}), flush=True)
            finally:
                for k, old in saved.items():
                    if old is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = old
    del sh, dh
