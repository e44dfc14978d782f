"""Scan-kernel experiments on one GPU: time ks_count on config workloads under
environment overrides (stride, chunk length, fast/generic kernel).

    python tools/exp_scan.py --config 3 --n 268435456 --reps 5
"""

import argparse
import json
import os
import statistics
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

from paper_1509_01506_b200 import _native, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--variants", default="default")
    args = ap.parse_args()
    w = workloads.make(args.config, args.n)
    variants = {
        "default": {},
        "generic": {"KS_DISABLE_FAST": "1"},
        "chunk2k": {"KS_CHUNK_LEN": "2048"},
        "chunk16k": {"KS_CHUNK_LEN": "16384"},
        "generic_k1": {"KS_DISABLE_FAST": "1", "KS_FORCE_STRIDE": "1"},
        "chunk64": {"KS_CHUNK_LEN": "64"},
        "chunk128": {"KS_CHUNK_LEN": "128"},
        "chunk256": {"KS_CHUNK_LEN": "256"},
        "chunk512": {"KS_CHUNK_LEN": "512"},
    }
    names = [v for v in args.variants.split(",") if v]
    out = {}
    want = None
    for name in names:
        env = variants[name]
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            ctx = _native.DeviceContext(0)
            dh = _native.DfaHandle(ctx, w.dfa)
            sh = ctx.upload_ascii(w.ascii.tobytes())
            counts = ctx.count(dh, sh)
            if want is None:
                want = counts
            assert (counts == want).all(), name
            ms = []
            for _ in range(args.reps):
                ctx.count(dh, sh)
                ms.append(ctx.stats()["scan_ms"])
            st = ctx.stats()
            out[name] = {"scan_ms": statistics.median(ms), "gbases_per_s": w.n / statistics.median(ms) / 1e6,
                         "chunks": st["chunks"], "chunk_len": st["chunk_len"], "info": dh.info}
            print(name, json.dumps(out[name]), flush=True)
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v


if __name__ == "__main__":
    main()
