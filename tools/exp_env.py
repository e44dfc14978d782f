"""A/B of environment knobs on one config (gpurun): counts must agree with the
first variant, scan-kernel time = median of `reps` synchronous calls.

    python tools/exp_env.py --config 3 --n 1073741824 base KS_L2HIST=1 KS_L2HIST=8
"""

import argparse
import json
import os
import statistics

import numpy as np
import torch
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

from paper_1509_01506_b200 import _native, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--flush", action="store_true", help="write 256 MiB before every timed call (L2 flush)")
    ap.add_argument("variants", nargs="*", default=["base"])
    args = ap.parse_args()
    w = workloads.make(args.config, args.n or None)
    ctx = _native.DeviceContext(0)
    dh = _native.DfaHandle(ctx, w.dfa)
    sh = ctx.upload_ascii(w.ascii.tobytes())
    want = None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if args.flush else None
    for rnd in range(2):
        for v in args.variants:
            env = dict(kv.split("=", 1) for kv in v.split(",") if "=" in kv)
            saved = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            try:
                counts = ctx.count(dh, sh)
                if want is None:
                    want = counts
                ok = bool((counts == want).all())
                ms = []
                for _ in range(args.reps):
                    if flush is not None:
                        flush.zero_()
                        torch.cuda.synchronize()
                    ctx.count(dh, sh)
                    ms.append(ctx.stats()["scan_ms"])
                med = statistics.median(ms)
                print(json.dumps({"round": rnd, "variant": v, "scan_ms": round(med, 4),
                                  "gbases_per_s": round(w.n / med / 1e6, 1), "counts_equal": ok,
                                  "checksum": int((counts * (1 + np.arange(counts.size))).sum()),
                                  "min_ms": round(min(ms), 4)}), flush=True)
            finally:
                for k, old in saved.items():
                    if old is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = old


if __name__ == "__main__":
    main()
