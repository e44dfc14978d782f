"""Generate golden fixtures by running the REAL reference implementation.

Run in the build container only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py [/root/reference/pkg/src]

Writes tests/golden/*.npz.  Inputs are stored (random cases) or regenerated
from the committed seeded generators with a sha256 guard (config cases).
The regex-dna built-in pattern set is never written to a fixture.
"""

from __future__ import annotations

import hashlib
import itertools
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))
REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF)

import kmerscan as ref  # noqa: E402

from paper_1509_01506_b200 import workloads  # noqa: E402

SEED = 20260823
POOL = np.frombuffer(b"acgtnACGTN", dtype=np.uint8)
GRID = list(itertools.product((1, 2, 3, 7, 16), (0, 1, 4, 10)))


def random_pattern_text(rng) -> str:
    """1-10 expressions, branches of 1-12 atoms, occasional classes
    (same distribution family as the reference's acceptance criterion 1)."""
    while True:
        lines = []
        for _ in range(int(rng.integers(1, 11))):
            branches = []
            for _ in range(int(rng.integers(1, 3))):
                length = int(rng.integers(1, 13))
                left = 3
                atoms = []
                for _ in range(length):
                    if left and rng.random() < 0.15:
                        left -= 1
                        k = int(rng.integers(2, 5))
                        bases = [str(b) for b in rng.permutation(list("acgt"))[:k]]
                        atoms.append("(" + "|".join(bases) + ")")
                    else:
                        atoms.append("acgt"[int(rng.integers(4))])
                branches.append("".join(atoms))
            lines.append("|".join(branches))
        text = "\n".join(lines)
        try:
            ref.parse_expressions(text)
        except ref.PatternSyntaxError:
            continue
        return text


def meta_json(m: dict) -> str:
    keep = {k: m[k] for k in ("input_length", "workers", "effective_workers", "window", "mode",
                              "pss_sizes", "speculative_runs", "converged_runs", "unconverged_runs")}
    keep["convergence_steps"] = {str(k): v for k, v in m["convergence_steps"].items()}
    return json.dumps(keep, sort_keys=True)


def random_cases(count: int = 300):
    rng = np.random.default_rng(SEED)
    out = {"texts": [], "data": [], "workers": [], "window": [], "counts": [], "locs": [], "meta": [],
           "dfa_t": [], "dfa_off": [], "dfa_ids": []}
    for i in range(count):
        n = i if i < 3 else int(rng.integers(0, 5001))
        data = rng.choice(POOL, size=n).tobytes()
        text = random_pattern_text(rng)
        workers, window = GRID[i % len(GRID)]
        dfa = ref.build_dfa(ref.expand_to_literals(ref.parse_expressions(text)))
        seq = ref.Sequence(ref.encode_bytes(data))
        rep = ref.run(dfa, seq, ref.EngineConfig(workers=workers, window=window, mode="locate"))
        out["texts"].append(text)
        out["data"].append(data)
        out["workers"].append(workers)
        out["window"].append(window)
        out["counts"].append(rep.per_expression_counts.astype(np.int64))
        out["locs"].append(rep.locations.astype(np.int64))
        out["meta"].append(meta_json(rep.metadata))
        out["dfa_t"].append(dfa.transitions.astype(np.int32))
        out["dfa_off"].append(dfa.out_offsets.astype(np.int32))
        out["dfa_ids"].append(dfa.out_ids.astype(np.int32))
    return out


def pack_ragged(arrs):
    offs = np.zeros(len(arrs) + 1, dtype=np.int64)
    np.cumsum([a.shape[0] for a in arrs], out=offs[1:])
    flat = np.concatenate(arrs) if arrs else np.zeros(0)
    return flat, offs


def write_random(path: Path) -> None:
    rc = random_cases()
    data_flat, data_off = pack_ragged([np.frombuffer(d, dtype=np.uint8) for d in rc["data"]])
    cnt_flat, cnt_off = pack_ragged(rc["counts"])
    loc_flat, loc_off = pack_ragged([l.reshape(-1, 2) for l in rc["locs"]])
    t_flat, t_off = pack_ragged([t.reshape(-1, 5) for t in rc["dfa_t"]])
    o_flat, o_off = pack_ragged(rc["dfa_off"])
    i_flat, i_off = pack_ragged(rc["dfa_ids"])
    np.savez_compressed(
        path, texts=np.array(rc["texts"]), data=data_flat, data_off=data_off,
        workers=np.array(rc["workers"]), window=np.array(rc["window"]),
        counts=cnt_flat, counts_off=cnt_off, locs=loc_flat.reshape(-1, 2), locs_off=loc_off,
        meta=np.array(rc["meta"]), dfa_t=t_flat.reshape(-1, 5), dfa_t_off=t_off,
        dfa_off=o_flat, dfa_off_off=o_off, dfa_ids=i_flat, dfa_ids_off=i_off)


CONFIG_CASES = [
    # (config, n, workers, window, mode)
    (1, None, 4, 10, "locate"),
    (2, 4 << 20, 8, 10, "locate"),
    (3, 8 << 20, 8, 10, "count"),
    (3, 1 << 20, 3, 10, "locate"),
    (4, 2 << 20, 8, 10, "locate"),
    (5, 1 << 20, 1, 10, "count"),
    (5, 1 << 16, 4, 10, "count"),
]


def write_configs(path: Path) -> None:
    arrays = {}
    index = []
    for i, (k, n, workers, window, mode) in enumerate(CONFIG_CASES):
        w = workloads.make(k, n)
        digest = hashlib.sha256(w.ascii.tobytes()).hexdigest()
        if k == 5:
            d = w.dfa
            dfa = ref.Dfa(transitions=np.array(d.transitions), out_offsets=np.array(d.out_offsets),
                          out_ids=np.array(d.out_ids), labels=d.labels, n_expressions=1)
        else:
            dfa = ref.build_dfa(ref.expand_to_literals(ref.parse_expressions(w.pattern_text)))
        seq = ref.Sequence(ref.encode_bytes(w.ascii.tobytes()))
        rep = ref.run(dfa, seq, ref.EngineConfig(workers=workers, window=window, mode=mode))
        arrays[f"counts_{i}"] = rep.per_expression_counts.astype(np.int64)
        if mode == "locate":
            arrays[f"locs_{i}"] = rep.locations.astype(np.int64)
        index.append({"config": k, "n": w.n, "workers": workers, "window": window, "mode": mode,
                      "sha256": digest, "states": int(dfa.state_count),
                      "meta": json.loads(meta_json(rep.metadata))})
        print(f"config {k} n={w.n}: states={dfa.state_count} total={rep.total_count}", flush=True)
    np.savez_compressed(path, index=np.array(json.dumps(index)), **arrays)


def write_dfas(path: Path) -> None:
    """DFAs of pattern sets whose text is committed (toy + config sets)."""
    texts = ["acg\ncat\ncta\ntta", "a|aa\na", "aca", "ta\ncta", "aa\na", "a",
             "(a|c|g|t)(a|c|g|t)(a|c|g|t)(a|c|g|t)(a|c|g|t)(a|c|g|t)",
             workloads.make(1).pattern_text, workloads.make(2, 64).pattern_text,
             workloads.make(3, 64).pattern_text, workloads.make(4, 64).pattern_text]
    arrays = {}
    for i, text in enumerate(texts):
        d = ref.build_dfa(ref.expand_to_literals(ref.parse_expressions(text)))
        m = ref.minimize(d)
        arrays[f"t_{i}"] = d.transitions
        arrays[f"off_{i}"] = d.out_offsets
        arrays[f"ids_{i}"] = d.out_ids
        arrays[f"labels_{i}"] = np.array(d.labels)
        arrays[f"min_t_{i}"] = m.transitions
        arrays[f"min_ids_{i}"] = m.out_ids
        arrays[f"dump_{i}"] = np.array(ref.dump_dfa(d))
    np.savez_compressed(path, texts=np.array(texts), **arrays)


def write_builtin_summary(path: Path) -> None:
    """Only counts/checksums of the built-in set (its text is not stored)."""
    dfa = ref.build_dfa(ref.expand_to_literals(ref.builtin_expression_set()))
    seq = ref.synthetic_sequence(64 * 1024 * 1024, seed=SEED)
    rep = ref.run(dfa, seq, ref.EngineConfig(workers=8))
    doc = {"states": int(dfa.state_count), "minimized": int(ref.minimize(dfa).state_count),
           "counts_64MiB_seed20260823": rep.per_expression_counts.tolist(),
           "checksum": ref.counts_checksum(rep.per_expression_counts)}
    path.write_text(json.dumps(doc, indent=1) + "\n")


if __name__ == "__main__":
    write_dfas(HERE / "dfas.npz")
    write_random(HERE / "random_cases.npz")
    write_configs(HERE / "configs.npz")
    write_builtin_summary(HERE / "builtin_summary.json")
    print("done")
