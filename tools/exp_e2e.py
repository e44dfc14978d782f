"""End-to-end (pinned host ASCII -> counts) A/B of environment knobs on C3
(gpurun): median wall time of ks_count_host_ascii per variant.

    python tools/exp_e2e.py KS_RAW_EVERY=0 KS_RAW_EVERY=6 KS_PIECE_KB=32768
"""
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_01506_b200 import _native, workloads  # noqa: E402

w = workloads.make(int(os.environ.get("CFG", "3")))
ctx = _native.context(0)
dh = ctx.dfa(w.dfa)
host = torch.from_numpy(w.ascii).pin_memory().numpy()
want = ctx.count(dh, ctx.upload_ascii(w.ascii))
variants = sys.argv[1:] or ["base"]
for rnd in range(2):
    for v in variants:
        env = dict(kv.split("=", 1) for kv in v.split(",") if "=" in kv)
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            ts = []
            for i in range(6):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                got = ctx.count_host_ascii(dh, host)
                ts.append(time.perf_counter() - t0)
                assert np.array_equal(got, want), v
            med = statistics.median(ts[1:])
            st = ctx.stats()
            print(json.dumps({"round": rnd, "variant": v, "e2e_gbs": round(w.n / med / 1e9, 1),
                              "ms": round(med * 1e3, 2), "h2d_MB": round(st["h2d_bytes"] / 1e6, 1)}), flush=True)
        finally:
            for k, old in saved.items():
                if old is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = old
