"""Randomised GPU-vs-oracle stress (run on the GPU box):

    python tools/stress_parity.py SECONDS [SEED]

Random pattern sets (classes, 1-40 literals of 1-70 bases), random hand-built
automata (generic / permutation columns), random sequences with N, lowercase,
whitespace and FASTA headers; every trial checks run() count+locate, the
streamed host-bytes count (raw and FASTA), scan_range with a random entry
state, all three strategies where they apply.  Prints failures with seeds.
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_01506_b200 as ks  # noqa: E402
from paper_1509_01506_b200 import _native  # noqa: E402
from paper_1509_01506_b200.ingest import strip_fasta_headers  # noqa: E402
from oracle import oracle as O  # noqa: E402


def random_text(rng):
    lines = []
    for _ in range(int(rng.integers(1, 12))):
        branches = []
        for _ in range(int(rng.integers(1, 3))):
            atoms = []
            left = 3   # classes per branch (the expansion cap is 4096 literals)
            for _ in range(int(rng.integers(1, 71 if rng.random() < 0.1 else 13))):
                if left and rng.random() < 0.1:
                    left -= 1
                    k = int(rng.integers(2, 5))
                    atoms.append("(" + "|".join(rng.permutation(list("acgt"))[:k]) + ")")
                else:
                    atoms.append("acgt"[int(rng.integers(4))])
            branches.append("".join(atoms))
        lines.append("|".join(branches))
    return "\n".join(lines) + "\n"


def random_dfa(rng):
    nq = int(rng.integers(1, 300))
    trans = rng.integers(0, nq, (nq, 5)).astype(np.int32)
    for c in range(5):
        if rng.random() < 0.4:
            trans[:, c] = rng.permutation(nq)
    if rng.random() < 0.5:
        trans[:, 4] = 0
    outs = [sorted(rng.integers(0, 3, int(rng.integers(0, 3))).tolist()) if rng.random() < 0.3 else []
            for _ in range(nq)]
    off = np.zeros(nq + 1, dtype=np.int32)
    off[1:] = np.cumsum([len(o) for o in outs])
    ids = np.array([e for o in outs for e in o], dtype=np.int32)
    return ks.Dfa(trans, off, ids, tuple("abc"), 3)


def random_bytes(rng, n):
    pool = np.frombuffer(b"acgtACGTnN \n\r>xacgt", dtype=np.uint8)
    p = np.ones(pool.size)
    p[8:14] = [0.02, 0.02, 0.01, 0.01, 0.005, 0.005]
    p[:8] = 1
    p = p / p.sum()
    return bytes(pool[rng.choice(pool.size, size=n, p=p)])


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60
    seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    ctx = _native.context(0)
    t_end = time.time() + budget
    trials = fails = 0
    seed = seed0
    while time.time() < t_end:
        rng = np.random.default_rng([seed, 1509])
        seed += 1
        try:
            dfa = random_dfa(rng) if rng.random() < 0.25 else ks.build_dfa(ks.expand_to_literals(
                ks.parse_expressions(random_text(rng))))
        except (ks.PatternSyntaxError, ks.ExpansionLimitError):
            continue   # the generator drew an invalid set (duplicate literal, too many expansions)
        n = int(rng.integers(0, 400_000 if rng.random() < 0.3 else 5000))
        data = random_bytes(rng, n)
        sym = ks.encode_bytes(data)
        fsym = ks.encode_bytes(strip_fasta_headers(data))
        want, rows = O.ref_run(dfa, sym, 1, 10, True)[:2]
        want_f = O.ref_sequential_count(dfa, fsym)[0]
        strategies = [0, 3] + ([2] if dfa.state_count <= 64 else [])
        for strat in strategies:
            try:
                dh = ctx.dfa(dfa, strategy=strat)
            except Exception:
                continue   # strategy not applicable to this automaton
            tag = f"seed={seed - 1} n={n} nq={dfa.state_count} strategy={dh.info['strategy_name']}"
            try:
                c, r = ctx.locate(dh, ctx.upload_codes(sym))
                assert c.tolist() == want.tolist(), "locate counts"
                assert np.array_equal(r, rows), "locate rows"
                assert ctx.count_host_ascii(dh, data).tolist() == want.tolist(), "stream raw"
                assert ctx.count_host_ascii(dh, data, fasta=True).tolist() == want_f.tolist(), "stream fasta"
                m = len(sym)
                if m:
                    b = int(rng.integers(0, m))
                    e = int(rng.integers(b, m + 1))
                    q = int(rng.integers(0, dfa.state_count))
                    wc, wl = O.ref_sequential_count(dfa, sym[b:e], state=q)
                    gc, gl, _ = ctx.scan_range(dh, ctx.upload_codes(sym), b, e, q)
                    assert gc.tolist() == wc.tolist() and gl == wl, "scan_range"
                rep = ks.run(dfa, ks.Sequence(sym), ks.EngineConfig(workers=int(rng.integers(1, 9)),
                                                                    mode="locate"))
                assert rep.per_expression_counts.tolist() == want.tolist(), "run counts"
                assert np.array_equal(rep.locations, rows), "run rows"
            except AssertionError as exc:
                fails += 1
                print("FAIL", tag, exc, flush=True)
        trials += 1
    print(f"stress: {trials} trials, {fails} failures, seeds {seed0}..{seed - 1}", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
