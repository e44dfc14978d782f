"""Multi-device contexts (ks_open_multi): one sequence sharded over several
ranks of one process.  The box has one GPU, so the ranks share device 0 and
exchange by stream-ordered peer copies (the NCCL transport needs distinct
devices); slicing, halos, boundary-map composition, shard counts and row
concatenation are the same code.  Bit-exact against the oracle and the
one-device path.  Reference: engine.py:207-237 (one run() over all workers),
ingest.py:78-94 (contiguous partition)."""

import numpy as np
import pytest

import paper_1509_01506_b200 as ks
from paper_1509_01506_b200 import _native, workloads
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def dfa_of(text):
    return ks.build_dfa(ks.expand_to_literals(ks.parse_expressions(text)))


def random_dfa(rng, nq=23):
    """Hand-built automaton with merging columns (SPECULATE strategy)."""
    t = rng.integers(0, nq, size=(nq, 5)).astype(np.int32)
    t[:, 4] = rng.integers(0, nq)
    outs = [sorted(rng.integers(0, 3, rng.integers(0, 3)).tolist()) for _ in range(nq)]
    off = np.zeros(nq + 1, np.int32)
    off[1:] = np.cumsum([len(o) for o in outs])
    ids = np.array([i for o in outs for i in o] or [0], np.int32)[: off[-1]]
    return ks.Dfa(transitions=t, out_offsets=off, out_ids=ids, labels=("0", "1", "2"), n_expressions=3)


@pytest.fixture(scope="module")
def ctx():
    return _native.context(0)


@pytest.mark.parametrize("ranks", [2, 3, 5])
@pytest.mark.parametrize("config", [2, 3, 4, 5])
def test_multi_codes_vs_oracle(ctx, config, ranks):
    w = workloads.make(config, 3_000_001 if config != 5 else 1_000_003)
    codes = ks.encode_bytes(w.ascii.tobytes())
    m = _native.MultiContext([0] * ranks)
    assert not m.uses_nccl   # one device repeated: peer-copy transport
    dh = m.dfa(w.dfa)
    sh = m.upload_codes(codes)
    assert sh.length == codes.size
    want, want_rows, _ = O.ref_run(w.dfa, codes, 1 if config == 5 else 8, 10, True)
    assert m.count(dh, sh).tolist() == want.tolist()
    c, rows = m.locate(dh, sh)
    assert c.tolist() == want.tolist()
    assert np.array_equal(rows, want_rows)
    # the one-device result
    assert ctx.count(ctx.dfa(w.dfa), ctx.upload_codes(codes)).tolist() == want.tolist()


@pytest.mark.parametrize("fasta", [False, True])
def test_multi_ascii_pieces(fasta):
    rng = np.random.default_rng(7)
    w = workloads.make(3, 400_000)
    raw = w.ascii.tobytes()
    if fasta:   # 61-column lines, CRLF and LF, headers inside and across cut points
        lines, i, k = [], 0, 0
        while i < len(raw):
            if k % 97 == 0:
                lines.append(b">chr" + str(k).encode() + b" some header text")
            step = int(rng.integers(20, 80))
            lines.append(raw[i:i + step])
            i += step
            k += 1
        data = b"".join(ln + (b"\r\n" if j % 3 == 0 else b"\n") for j, ln in enumerate(lines))
    else:       # raw bytes with scattered whitespace
        arr = np.frombuffer(raw, np.uint8).copy()
        idx = rng.choice(arr.size, 5000, replace=False)
        arr[idx] = np.frombuffer(b" \t\r\n", np.uint8)[rng.integers(0, 4, idx.size)]
        data = arr.tobytes()
    from paper_1509_01506_b200.ingest import strip_fasta_headers
    codes = ks.encode_bytes(strip_fasta_headers(data) if fasta else data)
    want, want_rows, _ = O.ref_run(w.dfa, codes, 4, 10, True)
    for ranks in (2, 4, 7):
        m = _native.MultiContext([0] * ranks)
        sh = m.upload_ascii(data, fasta=fasta)
        assert sh.length == codes.size
        dh = m.dfa(w.dfa)
        assert m.count(dh, sh).tolist() == want.tolist(), ranks
        c, rows = m.locate(dh, sh)
        assert np.array_equal(rows, want_rows), ranks


@pytest.mark.parametrize("seed", range(3))
def test_multi_generic_automaton(seed):
    rng = np.random.default_rng(seed)
    dfa = random_dfa(rng)
    codes = rng.integers(0, 5, 200_003).astype(np.uint8)
    want, want_rows, _ = O.ref_run(dfa, codes, 1, 10, True)
    m = _native.MultiContext([0, 0, 0])
    dh, sh = m.dfa(dfa), m.upload_codes(codes)
    assert m.count(dh, sh).tolist() == want.tolist()
    c, rows = m.locate(dh, sh)
    assert np.array_equal(rows, want_rows)


def test_multi_small_and_empty():
    dfa = dfa_of("acg\ncat\ncta\ntta")
    m = _native.MultiContext([0, 0, 0, 0])
    dh = m.dfa(dfa)
    for text in ("", "a", "ctancat", "acgt" * 10, "cattacg" * 300):
        codes = ks.encode(text)
        want, want_rows, _ = O.ref_run(dfa, codes, 1, 10, True)
        sh = m.upload_codes(codes)
        assert m.count(dh, sh).tolist() == want.tolist(), text
        c, rows = m.locate(dh, sh)
        assert np.array_equal(rows, want_rows), text


def test_run_with_devices_matches_single_device():
    w = workloads.make(4, 2_000_000)
    seq = ks.Sequence(ks.encode_bytes(w.ascii.tobytes()))
    one = ks.run(w.dfa, seq, ks.EngineConfig(workers=5, mode="locate"))
    many = ks.run(w.dfa, seq, ks.EngineConfig(workers=5, mode="locate", devices=(0, 0, 0)))
    assert many.per_expression_counts.tolist() == one.per_expression_counts.tolist()
    assert np.array_equal(many.locations, one.locations)
    for key in ("pss_sizes", "speculative_runs", "converged_runs", "unconverged_runs", "convergence_steps",
                "effective_workers", "input_length"):
        assert many.metadata[key] == one.metadata[key], key
    assert many.device_stats["devices"] == [0, 0, 0]
