"""Randomised stress of the visit-class count, the row flags and the plain-item
loops (run on the GPU box):

    python tools/stress_class.py SECONDS [SEED]

Random K = 2 automata (1100-4000 states, row copies), random K = 3 / K = 4
automata, sequences of 1 .. 48 Mi symbols with OTHER as single symbols, runs
across block / unit / tile borders, whole tiles and ragged ends, random unit
sizes (KS_TILE_LB); every trial checks the fused count (device-packed,
host-packed and device-encoded uploads), the ring kernel (KS_NO_CLS=1) and
ranges with random entry states against the oracle.
"""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_01506_b200 as ks  # noqa: E402
from paper_1509_01506_b200 import _native  # noqa: E402
from oracle import oracle as O  # noqa: E402


def dfa_of(text):
    return ks.build_dfa(ks.expand_to_literals(ks.parse_expressions(text)))


def random_dfa(rng):
    kind = rng.choice(["k2", "k2", "k3", "k4"])
    while True:
        nlit = {"k2": (150, 420), "k3": (20, 110), "k4": (2, 24)}[kind]
        lits = set()
        for _ in range(int(rng.integers(*nlit))):
            n = int(rng.choice([1, 2, 3, 4, 6, 8, 10, 12], p=[.02, .06, .1, .12, .2, .2, .15, .15]))
            lits.add("".join("acgt"[x] for x in rng.integers(0, 4, n)))
        lits = sorted(lits)
        rng.shuffle(lits)
        lines, i = [], 0
        while i < len(lits):
            k = int(rng.integers(1, 4))
            lines.append("|".join(lits[i:i + k]))
            i += k
        dfa = dfa_of("\n".join(lines))
        lo, hi = {"k2": (1100, 4000), "k3": (257, 1024), "k4": (2, 256)}[kind]
        if lo <= dfa.state_count <= hi:
            return kind, dfa


def random_codes(rng, n, unit):
    codes = rng.integers(0, 4, n).astype(np.uint8)
    tile = 32 * unit
    if n and rng.random() < 0.7:
        codes[rng.random(n) < float(rng.choice([1e-6, 1e-4, 2e-3]))] = 4
    for _ in range(int(rng.integers(0, 9))):
        if n < 4:
            break
        kind = rng.integers(0, 5)
        if kind == 0:      # a run across block borders
            a = int(rng.integers(0, n)); ln = int(rng.integers(1, 5000))
        elif kind == 1:    # a whole unit
            a = int(rng.integers(0, max(1, n // unit))) * unit; ln = unit
        elif kind == 2:    # a whole tile (or several)
            a = int(rng.integers(0, max(1, n // tile))) * tile; ln = tile * int(rng.integers(1, 3))
        elif kind == 3:    # the first / last base of a unit
            a = int(rng.integers(0, max(1, n // unit))) * unit - int(rng.integers(0, 2)); ln = 1
        else:              # a long run
            a = int(rng.integers(0, n)); ln = int(rng.integers(5000, 300000))
        a = max(0, a)
        codes[a:a + ln] = 4
    return codes


def main():
    seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 60
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    t_end = time.time() + seconds
    trials = fails = 0
    while time.time() < t_end or (trials == 0 and os.environ.get("ONE")):
        s = seed + trials
        trials += 1
        rng = np.random.default_rng(s)
        lb = int(rng.choice([1, 2, 3, 4, 4, 5, 6]))
        if os.environ.get("FORCE_LB"):
            lb = int(os.environ["FORCE_LB"])
        os.environ["KS_TILE_LB"] = str(lb)
        unit = 64 << lb
        kind, dfa = random_dfa(rng)
        n = int(rng.choice([int(rng.integers(0, 5000)), int(rng.integers(5000, 3 << 20)),
                            int(rng.integers(3 << 20, 48 << 20))]))
        codes = random_codes(rng, n, unit)
        if os.environ.get("NO_N"):
            codes[codes == 4] = 0
        if os.environ.get("PREFIX"):
            codes = codes[:int(os.environ["PREFIX"])].copy()
            n = codes.size
        if os.environ.get("DEBUG"):
            print("n", n, "OTHER", int((codes == 4).sum()), "states", dfa.state_count, flush=True)
        want = O.ref_sequential_count(dfa, codes)[0]
        c = _native.DeviceContext(0)
        dh = c.dfa(dfa)
        ascii_bytes = np.frombuffer(b"ACGTN", dtype=np.uint8)[codes].tobytes()
        ok = True
        try:
            for name, sh in (("codes", c.upload_codes(codes)), ("ascii", c.upload_ascii(ascii_bytes))):
                if os.environ.get("DEBUG"):
                    print("upload", name, "done; info", dh.info, flush=True)
                got = c.count(dh, sh)
                if os.environ.get("DEBUG"):
                    print("count done", flush=True)
                if got.tolist() != want.tolist():
                    ok = False
                    print(f"FAIL seed {s} {kind} lb {lb} n {n} upload {name}: count", flush=True)
                os.environ["KS_NO_CLS"] = "1"
                got = c.count(dh, sh)
                del os.environ["KS_NO_CLS"]
                if got.tolist() != want.tolist():
                    ok = False
                    print(f"FAIL seed {s} {kind} lb {lb} n {n} upload {name}: ring count", flush=True)
                for _ in range(3):
                    if n < 2:
                        break
                    b = int(rng.integers(0, n - 1))
                    e = int(rng.integers(b + 1, n + 1))
                    st = int(rng.integers(0, dfa.state_count))
                    g, last, _ = c.scan_range(dh, sh, b, e, st)
                    r, rl = O.ref_sequential_count(dfa, codes, b, e, st)
                    if g.tolist() != r.tolist() or last != rl:
                        ok = False
                        print(f"FAIL seed {s} {kind} lb {lb} n {n} upload {name}: range {b} {e} {st}", flush=True)
        except Exception as exc:  # noqa: BLE001
            ok = False
            print(f"FAIL seed {s} {kind} lb {lb} n {n}: {exc!r}", flush=True)
        fails += not ok
    print(f"stress_class: {trials} trials, {fails} failures (seeds {seed}..{seed + trials - 1})")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
