"""GPU parity: the device scan (through the C ABI) against the pinned oracle
and the reference's golden fixtures.  Bit-exact counts and rows."""

import hashlib

import numpy as np
import pytest
import torch

import paper_1509_01506_b200 as ks
from paper_1509_01506_b200 import _native, workloads
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return _native.context(0)


def dfa_of(text):
    return ks.build_dfa(ks.expand_to_literals(ks.parse_expressions(text)))


# ---------------------------------------------------------------- known answers
# (reference tests/test_engine.py, test_oracle_bench.py, test_automaton.py)

def test_known_answers(toy_dfa):
    rep = ks.run(toy_dfa, ks.sequence_from_text("ctancat"), ks.EngineConfig(workers=2))
    assert rep.per_expression_counts.tolist() == [0, 1, 1, 0]
    dfa = dfa_of("aca")
    rep = ks.run(dfa, ks.sequence_from_text("acaca"), ks.EngineConfig(mode="locate"))
    assert rep.per_expression_counts.tolist() == [2]
    assert rep.locations.tolist() == [[3, 0], [5, 0]]
    assert ks.sequential_count(dfa_of("a|aa"), ks.sequence_from_text("aa")).tolist() == [3]
    rep = ks.run(dfa_of("ta\ncta"), ks.sequence_from_text("cta"), ks.EngineConfig(mode="locate"))
    assert rep.locations.tolist() == [[3, 0], [3, 1]]
    rep = ks.run(toy_dfa, ks.sequence_from_text("ctacatacg"), ks.EngineConfig(workers=2))
    assert rep.per_expression_counts.tolist() == [1, 1, 1, 0]
    rep = ks.run(dfa_of("a|aa\na"), ks.sequence_from_text("aaNaa"), ks.EngineConfig(mode="locate"))
    assert rep.locations.tolist() == [[1, 0], [1, 1], [2, 0], [2, 0], [2, 1], [4, 0], [4, 1],
                                      [5, 0], [5, 0], [5, 1]]


def test_global_exclusive_offsets(toy_dfa):
    res = ks.match_chunk(toy_dfa, ks.encode("ttta"), 100, np.array([0]), ks.EngineConfig(mode="locate"))
    assert res[0].locations.tolist() == [[104, 3]]


def test_empty_input(toy_dfa):
    rep = ks.run(toy_dfa, ks.sequence_from_text(""), ks.EngineConfig(workers=8, mode="locate"))
    assert rep.total_count == 0
    assert rep.per_expression_counts.tolist() == [0, 0, 0, 0]
    assert rep.locations.shape == (0, 2)
    assert rep.metadata["effective_workers"] == 1


# ---------------------------------------------------------------- golden fixtures

def test_random_cases_vs_reference(random_cases):
    for i, c in enumerate(random_cases):
        dfa = dfa_of(c["text"])
        seq = ks.Sequence(ks.encode_bytes(c["data"]))
        rep = ks.run(dfa, seq, ks.EngineConfig(workers=c["workers"], window=c["window"], mode="locate"))
        assert rep.per_expression_counts.tolist() == c["counts"].tolist(), i
        assert rep.locations.tolist() == c["locs"].tolist(), i
        for key, val in c["meta"].items():
            got = rep.metadata[key]
            if key == "convergence_steps":
                got = {str(k): v for k, v in got.items()}
            assert got == val, (i, key)


def test_config_cases_vs_reference(config_cases):
    for c in config_cases:
        w = workloads.make(c["config"], c["n"])
        assert hashlib.sha256(w.ascii.tobytes()).hexdigest() == c["sha256"]
        seq = ks.Sequence(ks.encode_bytes(w.ascii.tobytes()))
        rep = ks.run(w.dfa, seq, ks.EngineConfig(workers=c["workers"], window=c["window"], mode=c["mode"]))
        assert rep.per_expression_counts.tolist() == c["counts"].tolist(), c["config"]
        if c["locs"] is not None:
            assert np.array_equal(rep.locations, c["locs"]), c["config"]
        for key, val in c["meta"].items():
            got = rep.metadata[key]
            if key == "convergence_steps":
                got = {str(k): v for k, v in got.items()}
            assert got == val, (c["config"], key)


# ---------------------------------------------------------------- oracle differential

@pytest.mark.parametrize("seed", range(6))
def test_random_vs_oracle(ctx, seed):
    rng = np.random.default_rng(seed)
    lits = sorted({"".join("acgt"[x] for x in rng.integers(0, 4, rng.integers(1, 13)))
                   for _ in range(int(rng.integers(1, 60)))})
    dfa = dfa_of("\n".join(lits))
    for n in (0, 1, 63, 64, 65, 127, 1000, 4097, 200_003):
        codes = rng.integers(0, 4, n).astype(np.uint8)
        codes[rng.random(n) < 0.02] = 4
        if n > 500:  # an N run across block borders
            codes[300:431] = 4
        seq = ks.Sequence(codes)
        want, rows = O.ref_run(dfa, codes, 1, 10, True)[:2]
        rep = ks.run(dfa, seq, ks.EngineConfig(mode="locate"))
        assert rep.per_expression_counts.tolist() == want.tolist(), (seed, n)
        assert np.array_equal(rep.locations, rows), (seed, n)


@pytest.mark.parametrize("stride", ["1", "2", "3", "4"])
def test_forced_strides(monkeypatch, stride):
    monkeypatch.setenv("KS_FORCE_STRIDE", stride)
    monkeypatch.setenv("KS_DISABLE_FAST", "1")   # the generic kernel at each stride
    ctx = _native.DeviceContext(0)
    w = workloads.make(2, 1 << 20)
    codes = ks.encode_bytes(w.ascii.tobytes())
    codes[5000:9000] = 4
    dh = ctx.dfa(w.dfa)
    assert dh.info["stride"] == int(stride)
    want, rows = O.ref_run(w.dfa, codes, 1, 10, True)[:2]
    sh = ctx.upload_codes(codes)
    got, grows = ctx.locate(dh, sh)
    assert got.tolist() == want.tolist()
    assert np.array_equal(grows, rows)


def test_global_tables(monkeypatch):
    monkeypatch.setenv("KS_FORCE_GLOBAL_TABLES", "1")
    ctx = _native.DeviceContext(0)
    w = workloads.make(3, 1 << 20)
    codes = ks.encode_bytes(w.ascii.tobytes())
    dh = ctx.dfa(w.dfa)
    assert dh.info["tables_in_smem"] == 0
    want = O.ref_sequential_count(w.dfa, codes)[0]
    assert ctx.count(dh, ctx.upload_codes(codes)).tolist() == want.tolist()


@pytest.mark.parametrize("chunk", ["64", "128", "1024"])
def test_small_chunks(monkeypatch, chunk):
    """Many lane chunks: every chunk derives its entry state by lookback."""
    monkeypatch.setenv("KS_CHUNK_LEN", chunk)
    ctx = _native.DeviceContext(0)
    w = workloads.make(3, 1 << 19)
    codes = ks.encode_bytes(w.ascii.tobytes())
    want, rows = O.ref_run(w.dfa, codes, 1, 10, True)[:2]
    dh = ctx.dfa(w.dfa)
    got, grows = ctx.locate(dh, ctx.upload_codes(codes))
    assert got.tolist() == want.tolist()
    assert np.array_equal(grows, rows)


# ---------------------------------------------------------------- non-converging DFA (C5)

def test_permutation_dfa_mapscan(ctx, monkeypatch):
    monkeypatch.setenv("KS_CHUNK_LEN", "256")
    c2 = _native.DeviceContext(0)
    dfa = workloads.permutation_dfa()
    dh = c2.dfa(dfa)
    assert dh.info["strategy_name"] == "mapscan"
    assert dh.info["monoid_size"] == 2048
    rng = np.random.default_rng(5)
    codes = rng.integers(0, 4, 300_001).astype(np.uint8)
    codes[rng.random(codes.size) < 0.001] = 4
    want, rows = O.ref_run(dfa, codes, 1, 10, True)[:2]
    got, grows = c2.locate(dh, c2.upload_codes(codes))
    assert got.tolist() == want.tolist()
    assert np.array_equal(grows, rows)


def test_small_random_dfas_mapscan(ctx):
    rng = np.random.default_rng(11)
    for trial in range(20):
        nq = int(rng.integers(1, 5))
        trans = rng.integers(0, nq, (nq, 5)).astype(np.int32)
        outs = [sorted(rng.integers(0, 3, rng.integers(0, 3)).tolist()) for _ in range(nq)]
        off = np.zeros(nq + 1, dtype=np.int32)
        off[1:] = np.cumsum([len(o) for o in outs])
        ids = np.array([e for o in outs for e in o], dtype=np.int32)
        dfa = ks.Dfa(trans, off, ids, tuple(str(i) for i in range(nq)), 3)
        codes = rng.integers(0, 5, int(rng.integers(0, 20000))).astype(np.uint8)
        want, rows = O.ref_run(dfa, codes, 1, 10, True)[:2]
        rep = ks.run(dfa, ks.Sequence(codes), ks.EngineConfig(mode="locate"))
        assert rep.per_expression_counts.tolist() == want.tolist(), trial
        assert np.array_equal(rep.locations, rows), trial


# ---------------------------------------------------------------- ranges / maps

def test_scan_range_and_segment_map(ctx):
    w = workloads.make(2, 1 << 18)
    codes = ks.encode_bytes(w.ascii.tobytes())
    dh = ctx.dfa(w.dfa)
    sh = ctx.upload_codes(codes)
    rng = np.random.default_rng(3)
    for _ in range(20):
        b, e = sorted(rng.integers(0, codes.size, 2).tolist())
        entry = int(rng.integers(0, w.dfa.state_count))
        want, last = O.ref_sequential_count(w.dfa, codes, b, e, entry)
        got, ex, _ = ctx.scan_range(dh, sh, b, e, entry)
        assert got.tolist() == want.tolist()
        assert ex == last
        # true-state entry (-1) == entry from the sequential state at b
        _, sb = O.ref_sequential_count(w.dfa, codes, 0, b, 0)
        want2, last2 = O.ref_sequential_count(w.dfa, codes, b, e, sb)
        got2, ex2, _ = ctx.scan_range(dh, sh, b, e, -1)
        assert got2.tolist() == want2.tolist() and ex2 == last2
        m = ctx.segment_map(dh, sh, b, e)
        for q in rng.integers(0, w.dfa.state_count, 5):
            assert m[q] == O.ref_sequential_count(w.dfa, codes, b, e, int(q))[1]


def test_segment_map_permutation(ctx):
    dfa = workloads.permutation_dfa()
    dh = ctx.dfa(dfa)
    codes = np.random.default_rng(9).integers(0, 4, 70_000).astype(np.uint8)
    sh = ctx.upload_codes(codes)
    m = ctx.segment_map(dh, sh, 1000, 65_000)
    g = int((codes[1000:65_000] == 2).sum())
    assert m.tolist() == [(q + g) % 1024 for q in range(1024)]


# ---------------------------------------------------------------- encode (K1)

def test_device_encode_matches_host():
    ctx = _native.context(0)
    rng = np.random.default_rng(7)
    for n in (0, 1, 63, 64, 65, 1000, 100_003):
        raw = rng.integers(0, 256, n).astype(np.uint8)
        mask = rng.random(n) < 0.6
        raw[mask] = rng.choice(np.frombuffer(b"acgtACGTNn \n\r\t", np.uint8), int(mask.sum()))
        sh = ctx.upload_ascii(raw.tobytes())
        want = ks.encode_bytes(raw.tobytes())
        assert sh.length == want.size
        assert np.array_equal(sh.codes(), want)
    # whitespace-free fast path + soft-mask bitmap
    text = b"ACGTacgtNnxX" * 1000
    sh = ctx.upload_ascii(text)
    assert np.array_equal(sh.codes(), ks.encode_bytes(text))
    soft = sh.softmask()
    assert np.array_equal(soft, np.frombuffer(text, np.uint8) >= ord("a"))


def test_device_encode_every_byte():
    ctx = _native.context(0)
    raw = bytes(range(256)) * 3
    sh = ctx.upload_ascii(raw)
    assert np.array_equal(sh.codes(), ks.encode_bytes(raw))


def test_bad_codes_rejected(ctx):
    with pytest.raises(ValueError):
        ctx.upload_codes(np.array([0, 1, 7], dtype=np.uint8))


# ---------------------------------------------------------------- match_chunk

def test_match_chunk_vs_oracle(toy_dfa):
    sym = ks.encode("acgtacgctacattta" * 3)
    pss = ks.possible_starting_states(toy_dfa, 0, 1)
    res = ks.match_chunk(toy_dfa, sym, 0, pss, ks.EngineConfig(mode="locate"))
    for r in res:
        c, last = O.ref_sequential_count(toy_dfa, sym, 0, None, r.init_state)
        assert r.counts.tolist() == c.tolist()
        assert r.last_state == last
    for window in (0, 1, 4):
        res = ks.match_chunk(toy_dfa, sym, 7, pss, ks.EngineConfig(window=window, mode="locate"))
        for r in res:
            c, last = O.ref_sequential_count(toy_dfa, sym, 0, None, r.init_state)
            assert r.counts.tolist() == c.tolist() and r.last_state == last
            if window == 0:
                assert r.converged_at is None


def test_match_chunk_reduce_roundtrip(toy_dfa):
    seq = ks.sequence_from_text("ttacatctacgtttacta" * 7)
    cfg = ks.EngineConfig(workers=4, mode="locate")
    plan = ks.plan_chunks(seq, 4)
    per = []
    for i, (lo, hi) in enumerate(plan.bounds):
        pss = np.array([0]) if i == 0 else ks.possible_starting_states(toy_dfa, *plan.boundary_symbols[i])
        per.append(ks.match_chunk(toy_dfa, seq.symbols[lo:hi], lo, pss, cfg))
    red = ks.reduce(toy_dfa, plan, per, cfg)
    rep = ks.run(toy_dfa, seq, cfg)
    assert red.per_expression_counts.tolist() == rep.per_expression_counts.tolist()
    assert red.locations.tolist() == rep.locations.tolist()
    for key in ("pss_sizes", "speculative_runs", "converged_runs", "convergence_steps"):
        assert red.metadata[key] == rep.metadata[key]


# ---------------------------------------------------------------- streaming host input

@pytest.mark.parametrize("encode", ["host", "device"])
@pytest.mark.parametrize("config,n", [(3, (1 << 20) + 12345), (2, 300_001), (5, 200_003), (1, 0), (1, 1)])
def test_count_host_ascii_matches(config, n, encode, monkeypatch):
    if encode == "device":
        monkeypatch.setenv("KS_DEVICE_ENCODE", "1")
    w = workloads.make(config, max(n, 1))
    data = w.ascii.tobytes()[:n]
    ctx = _native.context(0)
    dh = ctx.dfa(w.dfa)
    want = O.ref_sequential_count(w.dfa, ks.encode_bytes(data))[0]
    assert ctx.count_host_ascii(dh, data).tolist() == want.tolist()
    counts, rows = ks.scan_bytes(w.dfa, data)
    assert counts.tolist() == want.tolist() and rows is None


def test_count_host_ascii_small_pieces_and_whitespace():
    """Many pieces (entry state carried across pieces) and the whitespace
    fallback."""
    w = workloads.make(3, 1 << 22)
    data = w.ascii.tobytes()
    ctx = _native.context(0)
    dh = ctx.dfa(w.dfa)
    want = O.ref_sequential_count(w.dfa, ks.encode_bytes(data))[0]
    assert ctx.count_host_ascii(dh, data).tolist() == want.tolist()
    text = b"\n".join(data[i:i + 61] for i in range(0, 200_000, 61))
    want = O.ref_sequential_count(w.dfa, ks.encode_bytes(text))[0]
    assert ctx.count_host_ascii(dh, text).tolist() == want.tolist()


@pytest.mark.parametrize("encode", ["host", "device"])
def test_count_host_ascii_many_pieces(encode, monkeypatch):
    """Five 64 MiB pieces: the 3-slot pinned staging ring wraps, the device
    double buffer alternates, the entry state crosses every piece boundary
    (cuts fall inside units), and OTHER appears in some pieces only (nmask
    copied vs zero-filled)."""
    if encode == "device":
        monkeypatch.setenv("KS_DEVICE_ENCODE", "1")
    piece = 64 << 20
    w = workloads.make(3, 4 * piece + 777_777)
    buf = bytearray(w.ascii.tobytes())
    rng = np.random.default_rng(5)
    for p in rng.integers(piece, 2 * piece, size=1000).tolist() + [3 * piece - 1, 3 * piece, 4 * piece + 5]:
        buf[p] = ord("N")
    data = bytes(buf)
    want = O.ref_sequential_count(w.dfa, ks.encode_bytes(data))[0]
    ctx = _native.context(0)
    dh = ctx.dfa(w.dfa)
    pinned = torch.empty(len(data), dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = np.frombuffer(data, dtype=np.uint8)
    assert ctx.count_host_ascii(dh, pinned.numpy()).tolist() == want.tolist()
    assert ctx.count_host_ascii(dh, data).tolist() == want.tolist()   # pageable input too
    # whitespace only inside a piece that travels raw (pinned input, piece 2):
    # detected on the device, the call redoes the input on the compacting path
    pinned.numpy()[2 * piece + 12345] = ord("\n")
    text = pinned.numpy().tobytes()
    want_ws = O.ref_sequential_count(w.dfa, ks.encode_bytes(text))[0]
    assert ctx.count_host_ascii(dh, pinned.numpy()).tolist() == want_ws.tolist()


# ---------------------------------------------------------------- multi-GPU building blocks (on one GPU)

@pytest.mark.parametrize("config,n,world", [(3, 1 << 20, 3), (4, 1 << 19, 2), (5, 300_000, 4), (1, 5000, 3)])
def test_sharded_async_matches_sequential(config, n, world):
    """The NCCL path's device pieces, emulated rank by rank on one GPU: each
    shard's boundary map (ks_segment_map_async), the entry composed on the
    device from the 'gathered' maps, the shard scan (ks_count_shard_async);
    the summed counts equal one sequential pass."""
    import torch
    from paper_1509_01506_b200.distributed import shard_bounds

    w = workloads.make(config, n)
    codes = ks.encode_bytes(w.ascii.tobytes())
    ctx = _native.DeviceContext(0)
    dh = ctx.dfa(w.dfa)
    bounds = shard_bounds(codes.size, world)
    shards = [ctx.upload_codes(codes[b:e]) for b, e in bounds]
    nq, ne = w.dfa.state_count, w.dfa.n_expressions
    maps = torch.empty((world, nq), dtype=torch.int32, device="cuda")
    for r, sh in enumerate(shards):
        ctx.segment_map_async(dh, sh, 0, sh.length, maps[r].data_ptr())
    ctx.synchronize()
    total = np.zeros(ne, dtype=np.int64)
    for r, sh in enumerate(shards):
        c = torch.zeros(max(ne, 1), dtype=torch.int64, device="cuda")
        ctx.count_shard_async(dh, sh, 0, sh.length, maps.data_ptr(), r, c.data_ptr())
        ctx.synchronize()
        total += c.cpu().numpy()[:ne]
        # the gathered map of shard r is the host map
        b, e = bounds[r]
        want_map = ctx.segment_map(dh, sh, 0, sh.length)
        assert maps[r].cpu().numpy().tolist() == want_map.tolist()
    want = O.ref_sequential_count(w.dfa, codes)[0]
    assert total.tolist() == want.tolist()


@pytest.mark.parametrize("config,n,world", [(3, 1 << 20, 3), (4, 1 << 19, 4), (2, 300_000, 2)])
def test_sharded_halo_matches_sequential(config, n, world):
    """Halo mode of the multi-GPU step (definite automata): each shard is
    loaded with the previous shard's last bases in front, scanned from
    `halo` without any map exchange; the summed counts equal one pass."""
    import torch
    from paper_1509_01506_b200.distributed import shard_bounds

    w = workloads.make(config, n)
    codes = ks.encode_bytes(w.ascii.tobytes())
    ctx = _native.DeviceContext(0)
    dh = ctx.dfa(w.dfa)
    depth = dh.info["sync_depth"]
    halo = -(-max(depth, 1) // 64) * 64
    total = np.zeros(w.dfa.n_expressions, dtype=np.int64)
    for r, (b, e) in enumerate(shard_bounds(codes.size, world)):
        h = min(halo, b)
        sh = ctx.upload_codes(codes[b - h:e])
        c = torch.zeros(max(w.dfa.n_expressions, 1), dtype=torch.int64, device="cuda")
        ctx.count_shard_async(dh, sh, h, h + (e - b), 0, r, c.data_ptr())
        ctx.synchronize()
        total += c.cpu().numpy()[: w.dfa.n_expressions]
    assert total.tolist() == O.ref_sequential_count(w.dfa, codes)[0].tolist()
    with pytest.raises(ValueError):   # a halo shorter than the synchronisation depth is refused
        ctx.count_shard_async(dh, ctx.upload_codes(codes[:4096]), depth - 1, 4096, 0, 1,
                              torch.zeros(64, dtype=torch.int64, device="cuda").data_ptr())


# ---------------------------------------------------------------- device ingest (FASTA / whitespace)

FASTA_CASES = [
    b">s1 demo\nctacat\n",
    b">h\r\nACGT\r\nacgN\r\n>h2\r\nTTTT",
    b">h\rAC\rGT\r>x\r\rnn",
    b"acgt\n>not a header at file start? yes it is\nggg\n",
    b"ac>gt\n>hdr\n>hdr2\nA C\tG T\n\n\n",
    b">only header without newline",
    b"",
    b"\n\n\r\n",
    b"no header at all\nACGTTT\n",
    b">" + b"x" * 300 + b"\n" + b"acgt" * 70 + b"\n>" + b"y" * 130 + b"\r\n" + b"TTGCA" * 40,
]


def _fasta_expected(data: bytes) -> np.ndarray:
    from paper_1509_01506_b200.ingest import strip_fasta_headers
    return ks.encode_bytes(strip_fasta_headers(data))


def _random_fasta(rng, n_records: int, line: int) -> bytes:
    parts = []
    for r in range(n_records):
        parts.append(b">" + bytes(rng.choice(list(b"abc xyz>"), size=int(rng.integers(0, 150)))) +
                     rng.choice([b"\n", b"\r\n", b"\r"]))
        body = bytes(rng.choice(list(b"acgtACGTnN-"), size=int(rng.integers(0, 3000))))
        for i in range(0, len(body), line):
            parts.append(body[i:i + line] + rng.choice([b"\n", b"\r\n", b"\r", b" \n"]))
    return b"".join(parts)


@pytest.mark.parametrize("k", range(len(FASTA_CASES)))
def test_device_fasta_ingest_cases(k):
    data = FASTA_CASES[k]
    ctx = _native.context(0)
    sh = ctx.upload_ascii(data, fasta=True)
    assert sh.codes().tolist() == _fasta_expected(data).tolist()
    raw = ctx.upload_ascii(data, fasta=False)
    assert raw.codes().tolist() == ks.encode_bytes(data).tolist()


@pytest.mark.parametrize("seed,line", [(1, 60), (2, 80), (3, 61), (4, 200), (5, 7)])
def test_device_fasta_ingest_random(seed, line):
    rng = np.random.default_rng(seed)
    data = _random_fasta(rng, 40, line)
    ctx = _native.context(0)
    assert ctx.upload_ascii(data, fasta=True).codes().tolist() == _fasta_expected(data).tolist()


@pytest.mark.parametrize("piece_kb", [1, 3, 64])
@pytest.mark.parametrize("fmt", ["fasta", "raw"])
def test_count_host_bytes_streams_fasta_and_whitespace(piece_kb, fmt, monkeypatch):
    """Many small pieces: the header-line state and the DFA state cross every
    piece boundary (cuts fall inside headers, CRLF pairs and sequence lines)."""
    monkeypatch.setenv("KS_PIECE_KB", str(piece_kb))
    rng = np.random.default_rng(piece_kb)
    data = _random_fasta(rng, 60, 61)
    w = workloads.make(3, 4096)
    ctx = _native.context(0)
    dh = ctx.dfa(w.dfa)
    sym = _fasta_expected(data) if fmt == "fasta" else ks.encode_bytes(data)
    want = O.ref_sequential_count(w.dfa, sym)[0]
    assert ctx.count_host_ascii(dh, data, fasta=fmt == "fasta").tolist() == want.tolist()
    counts, rows = ks.scan_bytes(w.dfa, data, "locate", fmt=fmt)
    assert counts.tolist() == want.tolist()
    ref = O.ref_scan_rows(w.dfa, sym, 0, len(sym), w.dfa.start)[2]
    assert np.array_equal(rows, ref)


@pytest.mark.parametrize("task_blocks,piece_kb", [(1, 7), (2, 64), (3, 1), (4096, 64 * 1024)])
@pytest.mark.parametrize("encode", ["host", "device"])
def test_fasta_stream_tasks_and_pieces(task_blocks, piece_kb, encode, monkeypatch):
    """Host wire packing of FASTA: tiny tasks so that header lines, CRLF pairs
    and sequence lines straddle task and piece boundaries; a header line
    longer than a task; a file that does not end with a newline."""
    monkeypatch.setenv("KS_WIRE_TASK_BLOCKS", str(task_blocks))
    monkeypatch.setenv("KS_PIECE_KB", str(piece_kb))
    if encode == "device":
        monkeypatch.setenv("KS_DEVICE_ENCODE", "1")
    rng = np.random.default_rng(task_blocks * 7 + piece_kb)
    data = (_random_fasta(rng, 25, 61) + b">" + b"h" * 700 + b"\r\n" + _random_fasta(rng, 10, 200) +
            b"acgt\r>not a header\racgtNN>x\n\n>last header, no newline")
    w = workloads.make(3, 4096)
    ctx = _native.context(0)
    dh = ctx.dfa(w.dfa)
    want = O.ref_sequential_count(w.dfa, _fasta_expected(data))[0]
    assert ctx.count_host_ascii(dh, data, fasta=True).tolist() == want.tolist()
    want_raw = O.ref_sequential_count(w.dfa, ks.encode_bytes(data))[0]
    assert ctx.count_host_ascii(dh, data).tolist() == want_raw.tolist()


def test_load_sequence_device_matches_host(tmp_path):
    rng = np.random.default_rng(7)
    for name, fmt in (("a.fa", "fasta"), ("b.txt", "raw")):
        path = tmp_path / name
        path.write_bytes(_random_fasta(rng, 20, 70))
        dev = ks.load_sequence_device(path, fmt)
        host = ks.load_sequence(path, fmt)
        assert dev.symbols.tolist() == host.symbols.tolist() and dev.length == host.length
        w = workloads.make(2, 4096)
        assert ks.run(w.dfa, dev).per_expression_counts.tolist() == \
            ks.run(w.dfa, host).per_expression_counts.tolist()


# ---------------------------------------------------------------- long literals (lookback > 64 bases)

@pytest.mark.parametrize("lengths", [(70, 90), (150, 300), (1000, 1500)])
def test_long_literals_lookback(lengths):
    """Literals longer than a 64-base block: the synchronisation depth is the
    longest literal and the lookback spans several blocks (and, for the last
    case, the whole previous unit)."""
    rng = np.random.default_rng(lengths[0])
    lits = ["".join(rng.choice(list("acgt"), size=int(rng.integers(*lengths)))) for _ in range(6)]
    text = "\n".join(lits[:3] + [f"{lits[3]}|{lits[4]}", lits[5][:40]]) + "\n"
    dfa = ks.build_dfa(ks.expand_to_literals(ks.parse_expressions(text)))
    n = 1 << 20
    sym = rng.integers(0, 4, size=n).astype(np.uint8)
    for k in range(300):   # plant occurrences, some overlapping unit boundaries
        lit = lits[k % len(lits)]
        p = int(rng.integers(0, n - len(lit)))
        sym[p:p + len(lit)] = [("acgt".index(c)) for c in lit]
    sym[rng.integers(0, n, size=50)] = 4
    seq = ks.Sequence(sym)
    ctx = _native.context(0)
    dh = ctx.dfa(dfa)
    info = dh.info
    assert info["strategy_name"] == "lookback" and info["sync_depth"] >= lengths[0]
    want = O.ref_sequential_count(dfa, sym)[0]
    assert ctx.count(dh, ctx.seq(seq)).tolist() == want.tolist()
    assert want.sum() >= 150   # planted (some overwritten by later plants or N)
    rep = ks.run(dfa, seq, ks.EngineConfig(workers=7, mode="locate"))
    ref = O.ref_scan_rows(dfa, sym, 0, n, dfa.start)[2]
    assert np.array_equal(rep.locations, ref)


# ---------------------------------------------------------------- SPECULATE strategy (generic automata)

def _wild_dfa(nq=200, seed=3):
    """Three permutation columns (the generated group is huge, so no small
    monoid), one merging column, OTHER -> 0: neither definite nor MAPSCAN."""
    rng = np.random.default_rng(seed)
    trans = np.empty((nq, 5), dtype=np.int32)
    for c in range(3):
        trans[:, c] = rng.permutation(nq)
    trans[:, 3] = rng.integers(0, nq, nq)
    trans[:, 4] = 0
    outs = [sorted(rng.integers(0, 4, int(rng.integers(0, 3))).tolist()) if rng.random() < 0.2 else []
            for _ in range(nq)]
    off = np.zeros(nq + 1, dtype=np.int32)
    off[1:] = np.cumsum([len(o) for o in outs])
    ids = np.array([e for o in outs for e in o], dtype=np.int32)
    return ks.Dfa(trans, off, ids, tuple(str(i) for i in range(4)), 4)


@pytest.mark.parametrize("n", [1, 1000, 300_001])
def test_speculate_generic_automaton(n):
    dfa = _wild_dfa()
    ctx = _native.context(0)
    dh = ctx.dfa(dfa)
    assert dh.info["strategy_name"] == "speculate"
    rng = np.random.default_rng(n)
    codes = rng.integers(0, 4, n).astype(np.uint8)
    codes[rng.random(n) < 0.0005] = 4
    want, rows = O.ref_run(dfa, codes, 1, 10, True)[:2]
    got, grows = ctx.locate(dh, ctx.upload_codes(codes))
    assert got.tolist() == want.tolist()
    assert np.array_equal(grows, rows)
    rep = ks.run(dfa, ks.Sequence(codes), ks.EngineConfig(workers=5, mode="locate"))
    assert rep.per_expression_counts.tolist() == want.tolist()
    assert np.array_equal(rep.locations, rows)
    # ranges entering in given states and the exit state
    sh = ctx.upload_codes(codes)
    for b, e, q in ((0, n, 7), (n // 3, n, -1), (n // 2, n // 2 + 5000, 11)):
        e = min(e, n)
        q0 = q if q >= 0 else (int(O.ref_sequential_count(dfa, codes[:b])[1]) if b else 0)
        wc, wl = O.ref_sequential_count(dfa, codes[b:e], state=q0)
        c, last, _ = ctx.scan_range(dh, sh, b, e, q)
        assert c.tolist() == wc.tolist() and last == wl


@pytest.mark.parametrize("config", [1, 2, 3, 5])
def test_speculate_forced_on_config_automata(config):
    """The generic strategy forced onto the config automata (definite and
    MAPSCAN ones) must give their results too."""
    w = workloads.make(config, 200_003)
    ctx = _native.context(0)
    dh = ctx.dfa(w.dfa, strategy=_native.STRATEGY_SPECULATE)
    assert dh.info["strategy_name"] == "speculate"
    sym = ks.encode_bytes(w.ascii.tobytes())
    want = O.ref_sequential_count(w.dfa, sym)[0]
    assert ctx.count(dh, ctx.seq(ks.Sequence(sym))).tolist() == want.tolist()
    assert ctx.count_host_ascii(dh, w.ascii.tobytes()).tolist() == want.tolist()


def test_speculate_streamed_and_sharded(monkeypatch):
    monkeypatch.setenv("KS_PIECE_KB", "16")
    dfa = _wild_dfa(97, seed=9)
    rng = np.random.default_rng(2)
    data = bytes(np.frombuffer(b"acgtN", dtype=np.uint8)[rng.choice(5, 100_000, p=[.25, .25, .25, .2499, .0001])])
    sym = ks.encode_bytes(data)
    want = O.ref_sequential_count(dfa, sym)[0]
    ctx = _native.context(0)
    dh = ctx.dfa(dfa)
    assert dh.info["strategy_name"] == "speculate"
    assert ctx.count_host_ascii(dh, data).tolist() == want.tolist()
    assert ctx.count_host_ascii(dh, data, fasta=True).tolist() == want.tolist()
    # segment maps (every state walks the shard) composed like the NCCL path
    sh = ctx.upload_codes(sym)
    cuts = [0, 30_001, 64_000, len(sym)]
    state, total = 0, np.zeros_like(want)
    for b, e in zip(cuts[:-1], cuts[1:]):
        m = ctx.segment_map(dh, sh, b, e)
        c, last, _ = ctx.scan_range(dh, sh, b, e, state)
        assert last == m[state]
        total += c
        state = int(m[state])
    assert total.tolist() == want.tolist()


@pytest.mark.parametrize("lean", ["", "1"])
@pytest.mark.parametrize("n", [200_000, 6_000_000])
def test_locate_log_and_overflow_fallback(monkeypatch, n, lean):
    """Single-pass locate logs every accepting visit; a hit-dense scan whose
    visits overflow the log (C3's automaton on 6 M bases: > 64 Ki visits)
    takes the two-pass path.  Both give the reference's sorted rows (also
    with lean blocks forced: their re-runs in the rows and emit passes)."""
    if lean:
        monkeypatch.setenv("KS_LEAN", lean)
    w = workloads.make(3, n)
    sym = ks.encode_bytes(w.ascii.tobytes())
    ctx = _native.DeviceContext(0)
    dh = ctx.dfa(w.dfa)
    counts, rows = ctx.locate(dh, ctx.upload_codes(sym))
    ref_counts, _, ref_rows = O.ref_scan_rows(w.dfa, sym, 0, n, w.dfa.start)
    assert counts.tolist() == ref_counts.tolist()
    assert np.array_equal(rows, ref_rows)


# ---------------------------------------------------------------- full-size properties (C3, 1 GiB)

def test_full_size_c3_properties(monkeypatch):
    """At the benchmark's own size, size-independent properties (no oracle):
    resident count == streamed count (host-packed wire, raw pieces) ==
    streamed count with device encoding; additivity over 7 ranges whose
    entry states come from composed segment maps; locate rows == counts."""
    w = workloads.make(3)
    ctx = _native.context(0)
    dh = ctx.dfa(w.dfa)
    pinned = torch.empty(w.n, dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = w.ascii
    sh = ctx.upload_ascii(pinned.numpy())
    whole = ctx.count(dh, sh)
    assert ctx.count_host_ascii(dh, pinned.numpy()).tolist() == whole.tolist()
    monkeypatch.setenv("KS_DEVICE_ENCODE", "1")
    assert ctx.count_host_ascii(dh, pinned.numpy()).tolist() == whole.tolist()
    monkeypatch.delenv("KS_DEVICE_ENCODE")
    cuts = sorted(set([0, w.n] + [int(x) for x in np.random.default_rng(3).integers(1, w.n, 6)]))
    state, total = 0, np.zeros_like(whole)
    for b, e in zip(cuts[:-1], cuts[1:]):
        m = ctx.segment_map(dh, sh, b, e)
        c, last, _ = ctx.scan_range(dh, sh, b, e, state)
        assert last == m[state]
        total += c
        state = int(m[state])
    assert total.tolist() == whole.tolist()
    counts, rows = ctx.locate(dh, sh)
    assert counts.tolist() == whole.tolist() and rows.shape[0] == int(whole.sum())
    assert np.all(np.diff(rows[:, 0]) >= 0)


@pytest.mark.parametrize("data", [b"\n" * 1000, b" \t\r\n" * 5000, b">only a header\n", b">h\n" * 3000,
                                  b"N" * 100_000, b"acgt", b"x", b"a" * 64, b"a" * 65, b"\n" + b"acgt" * 40000])
@pytest.mark.parametrize("fasta", [False, True])
def test_degenerate_inputs(data, fasta):
    """Inputs that compact to nothing or to a handful of symbols, through the
    streamed count, the device ingest and run()."""
    from paper_1509_01506_b200.ingest import strip_fasta_headers
    w = workloads.make(2, 4096)
    ctx = _native.context(0)
    dh = ctx.dfa(w.dfa)
    sym = ks.encode_bytes(strip_fasta_headers(data) if fasta else data)
    want = O.ref_sequential_count(w.dfa, sym)[0]
    assert ctx.count_host_ascii(dh, data, fasta=fasta).tolist() == want.tolist()
    sh = ctx.upload_ascii(data, fasta=fasta)
    assert sh.length == sym.size
    assert ctx.count(dh, sh).tolist() == want.tolist()
    rep = ks.run(w.dfa, ks.Sequence(sym), ks.EngineConfig(workers=3, mode="locate"))
    assert rep.per_expression_counts.tolist() == want.tolist()


# ---------------------------------------------------------------- wide automata (> 32767 states)

@pytest.fixture(scope="module")
def wide_dfa():
    rng = np.random.default_rng(5)
    lits = set()
    while len(lits) < 4600:
        lits.add("".join(rng.choice(list("acgt"), size=int(rng.integers(12, 17)))))
    text = "\n".join(sorted(lits)[:2300]) + "\n" + "|".join(sorted(lits)[2300:2400]) + "\n" + \
        "\n".join(sorted(lits)[2400:]) + "\n"
    dfa = ks.build_dfa(ks.expand_to_literals(ks.parse_expressions(text)))
    assert dfa.state_count > 32767
    return dfa, sorted(lits)


@pytest.mark.parametrize("hot", ["default", "64", "chunks", "off"])
def test_wide_automaton(wide_dfa, hot, monkeypatch):
    """Automata above the 16-bit state range: 32-bit ids, LOOKBACK, the wide
    scan kernels (hot table in shared memory + cold transitions from L2; a
    64-state hot set; the L2-only kernel) -- counts, sorted rows, ranges,
    run() with metadata, the streamed call (which falls back to one upload)
    and the halo shard."""
    import torch

    if hot == "off":
        monkeypatch.setenv("KS_WIDE_HOT", "0")
    elif hot == "chunks":
        monkeypatch.setenv("KS_WIDE_TASKS", "0")
    elif hot != "default":
        monkeypatch.setenv("KS_WIDE_HOT_STATES", hot)
    dfa, lits = wide_dfa
    dfa = ks.Dfa(dfa.transitions, dfa.out_offsets, dfa.out_ids, dfa.labels, dfa.n_expressions)  # fresh upload
    rng = np.random.default_rng(9)
    n = 1 << 20
    sym = rng.integers(0, 4, n).astype(np.uint8)
    for k in range(400):
        lit = lits[int(rng.integers(0, len(lits)))]
        p = int(rng.integers(0, n - len(lit)))
        sym[p:p + len(lit)] = ["acgt".index(c) for c in lit]
    sym[rng.integers(0, n, 40)] = 4
    ctx = _native.DeviceContext(0)
    dh = ctx.dfa(dfa)
    assert dh.info["strategy_name"] == "lookback"
    want, rows, meta = O.ref_run(dfa, sym, 6, 10, True)
    sh = ctx.upload_codes(sym)
    got, grows = ctx.locate(dh, sh)
    assert got.tolist() == want.tolist() and np.array_equal(grows, rows) and want.sum() >= 300
    assert ctx.count(dh, sh).tolist() == want.tolist()
    rep = ks.run(dfa, ks.Sequence(sym), ks.EngineConfig(workers=6, mode="locate"))
    assert rep.per_expression_counts.tolist() == want.tolist() and np.array_equal(rep.locations, rows)
    for key in ("pss_sizes", "speculative_runs", "converged_runs", "convergence_steps"):
        assert rep.metadata[key] == meta[key], key
    q = dfa.state_count - 3
    wc, wl = O.ref_sequential_count(dfa, sym[1000:900_000], state=q)
    c, last, _ = ctx.scan_range(dh, sh, 1000, 900_000, q)
    assert c.tolist() == wc.tolist() and last == wl
    ascii_ = np.frombuffer(b"acgtN", dtype=np.uint8)[sym].tobytes()
    assert ctx.count_host_ascii(dh, ascii_).tolist() == want.tolist()
    m = ctx.segment_map(dh, sh, 0, 5000)
    assert int(m[0]) == int(O.ref_sequential_count(dfa, sym[:5000])[1])
    half = n // 2
    counts = np.zeros_like(want)
    depth = dh.info["sync_depth"]
    for r, (b, e, h) in enumerate(((0, half, 0), (half, n, 64 * (-(-depth // 64))))):
        sub = ctx.upload_codes(sym[b - h:e])
        t = torch.zeros(max(dfa.n_expressions, 1), dtype=torch.int64, device="cuda")
        ctx.count_shard_async(dh, sub, h, h + (e - b), 0, r, t.data_ptr())
        ctx.synchronize()
        counts += t.cpu().numpy()[: dfa.n_expressions]
    assert counts.tolist() == want.tolist()


# ---------------------------------------------------------------- MAPSCAN over the OTHER-free submonoid

def _monoid_dfas():
    """Non-definite automata with small transition monoids: a shift group
    (OTHER -> 0), mixed ones resetting to a non-start state (monoids of 156
    and 3152 maps), and one whose OTHER column is not constant (full-monoid
    map pass, 582 maps)."""
    out = [("shift64", workloads.permutation_dfa(64))]
    outs_all = [[0], [], [1, 1], [], [], [0, 2], [], [], [2], [], [], [1]]
    mixed = lambda nq, x: [(x + 1) % nq, (x + 3) % nq, x ^ 1 if (x ^ 1) < nq else x, (x // 2) * 2]
    cycmin = lambda nq, x: [(x + 1) % nq, x, (x + 2) % nq, min(x, 3)]
    for name, nq, cols, other in (("mixed_reset5", 12, mixed, lambda x: 5),
                                  ("cycmin_reset5", 8, cycmin, lambda x: 5),
                                  ("mixed_noreset", 6, mixed, lambda x: x // 3)):
        trans = np.array([cols(nq, x) + [other(x)] for x in range(nq)], dtype=np.int32)
        outs = outs_all[:nq]
        off = np.zeros(nq + 1, dtype=np.int32)
        off[1:] = np.cumsum([len(o) for o in outs])
        ids = np.array([e for o in outs for e in o], dtype=np.int32)
        out.append((name, ks.Dfa(trans, off, ids, ("a", "b", "c"), 3)))
    return out


def _codes_with_n_runs(n, seed):
    rng = np.random.default_rng(seed)
    codes = rng.integers(0, 4, n).astype(np.uint8)
    for _ in range(40):   # N runs of every length class, and lone Ns
        p = int(rng.integers(0, n))
        codes[p:p + int(rng.choice([1, 2, 63, 64, 65, 300, 1500]))] = 4
    codes[rng.random(n) < 0.0005] = 4
    return codes


@pytest.mark.parametrize("mono_full", ["0", "1"])
@pytest.mark.parametrize("global_tables", ["0", "1"])
def test_mapscan_submonoid_parity(monkeypatch, mono_full, global_tables):
    monkeypatch.setenv("KS_MONO_FULL", mono_full)
    monkeypatch.setenv("KS_FORCE_GLOBAL_TABLES", global_tables)
    c2 = _native.DeviceContext(0)
    for name, dfa in _monoid_dfas():
        dh = c2.dfa(dfa, strategy=_native.STRATEGY_MAPSCAN)
        assert dh.info["strategy_name"] == "mapscan", name
        for n, seed in ((1, 1), (777, 2), (200_003, 3)):
            codes = _codes_with_n_runs(n, seed)
            want, rows = O.ref_run(dfa, codes, 1, 10, True)[:2]
            sh = c2.upload_codes(codes)
            assert c2.count(dh, sh).tolist() == want.tolist(), (name, n)
            got, grows = c2.locate(dh, sh)
            assert got.tolist() == want.tolist() and np.array_equal(grows, rows), (name, n)
            if n > 1000:
                rng = np.random.default_rng(seed)
                for _ in range(4):
                    b, e = sorted(rng.integers(0, n, 2).tolist())
                    entry = int(rng.integers(0, dfa.state_count))
                    w2, last = O.ref_sequential_count(dfa, codes, b, e, entry)
                    g2, ex, _ = c2.scan_range(dh, sh, b, e, entry)
                    assert g2.tolist() == w2.tolist() and ex == last, (name, b, e)
                    m = c2.segment_map(dh, sh, b, e)
                    for q in range(dfa.state_count):
                        assert m[q] == O.ref_sequential_count(dfa, codes, b, e, q)[1], (name, b, e, q)
                text = bytes(np.frombuffer(b"ACGTN", dtype=np.uint8)[codes])
                assert c2.count_host_ascii(dh, text).tolist() == want.tolist(), name


def test_concurrent_calls_on_one_context():
    """The C ABI serialises calls on one context: threads that call ks_count /
    ks_locate directly (no Python-side lock; ctypes releases the GIL) all get
    the reference's results."""
    import ctypes as C
    import threading

    w = workloads.make(2, 300_001)
    codes = ks.encode_bytes(w.ascii.tobytes())
    want, rows = O.ref_run(w.dfa, codes, 1, 10, True)[:2]
    c2 = _native.DeviceContext(0)
    dh = c2.dfa(w.dfa)
    sh = c2.upload_codes(codes)
    lib = _native.library()
    errors = []

    def worker(k):
        try:
            for i in range(12):
                counts = np.zeros(max(w.dfa.n_expressions, 1), dtype=np.int64)
                if (i + k) % 3:
                    rc = lib.ks_count(c2.handle, dh.handle, sh.handle, _native._ptr(counts, C.c_int64))
                    assert rc == 0 and counts.tolist() == want.tolist()
                else:
                    rp, nr = C.POINTER(C.c_int64)(), C.c_int64()
                    rc = lib.ks_locate(c2.handle, dh.handle, sh.handle, _native._ptr(counts, C.c_int64),
                                       C.byref(rp), C.byref(nr))
                    assert rc == 0 and counts.tolist() == want.tolist() and nr.value == rows.shape[0]
                    got = np.ctypeslib.as_array(rp, shape=(nr.value * 2,)).reshape(-1, 2).copy()
                    lib.ks_free(rp)
                    assert np.array_equal(got, rows)
        except Exception as exc:   # surfaced below
            errors.append(repr(exc))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors[:3]


@pytest.mark.parametrize("lean", ["0", "1"])
@pytest.mark.parametrize("config", [1, 2, 3, 4])
def test_lean_blocks_forced(monkeypatch, config, lean):
    """Blocks scanned without hit bookkeeping and re-run when a lane hit
    (the default for rare-hit automata such as C4's) forced on and off for
    every config automaton: counts, rows, ranges, streamed input."""
    monkeypatch.setenv("KS_LEAN", lean)
    w = workloads.make(config, 300_007)
    codes = ks.encode_bytes(w.ascii.tobytes())
    want, rows = O.ref_run(w.dfa, codes, 1, 10, True)[:2]
    c2 = _native.DeviceContext(0)
    dh = c2.dfa(w.dfa)
    sh = c2.upload_codes(codes)
    assert c2.count(dh, sh).tolist() == want.tolist()
    got, grows = c2.locate(dh, sh)
    assert got.tolist() == want.tolist() and np.array_equal(grows, rows)
    assert c2.count_host_ascii(dh, w.ascii.tobytes()).tolist() == want.tolist()
    rng = np.random.default_rng(config)
    for _ in range(4):
        b, e = sorted(rng.integers(0, codes.size, 2).tolist())
        entry = int(rng.integers(0, w.dfa.state_count))
        w2, last = O.ref_sequential_count(w.dfa, codes, b, e, entry)
        g2, ex, _ = c2.scan_range(dh, sh, b, e, entry)
        assert g2.tolist() == w2.tolist() and ex == last


def test_async_back_to_back_mixed():
    """Back-to-back ks_count_async calls (no host sync, no events between the
    kernels, programmatic dependent launch) alternating automata, sequences
    and result buffers: every call's counts are the oracle's."""
    ctx = _native.DeviceContext(0)
    work = []
    for cfg, n in ((2, 200_003), (4, 300_001), (5, 150_007), (3, 250_009)):
        w = workloads.make(cfg, n)
        codes = ks.encode_bytes(w.ascii.tobytes())
        work.append((ctx.dfa(w.dfa), ctx.upload_codes(codes), O.ref_sequential_count(w.dfa, codes)[0]))
    outs = []
    for rep in range(3):
        for dh, sh, want in work:
            buf = torch.zeros(max(dh.n_expressions, 1), dtype=torch.int64).pin_memory()
            ctx.count_async(dh, sh, buf.numpy())
            outs.append((buf, want))
    waited = ctx.async_wait()
    assert waited["kernel_launches"] >= len(outs)
    for buf, want in outs:
        assert buf.numpy()[: want.size].tolist() == want.tolist()


def test_kernels_scan_from_dropin(toy_dfa):
    """paper_1509_01506_b200._kernels.scan_from: the reference's raw-array
    kernel signature (_kernels.py:18-29) on the device, counts added in place."""
    from paper_1509_01506_b200 import _kernels

    rng = np.random.default_rng(3)
    sym = rng.integers(0, 5, 5000).astype(np.uint8)
    for start, end, state in ((0, 5000, 0), (17, 4000, 3), (100, 100, 2), (4999, 5000, 1)):
        counts = np.full(toy_dfa.n_expressions, 7, dtype=np.int64)
        last = _kernels.scan_from(toy_dfa.transitions, toy_dfa.out_offsets, toy_dfa.out_ids, sym, start, end,
                                  state, counts)
        want, wl = O.ref_sequential_count(toy_dfa, sym, start, end, state)
        assert counts.tolist() == (want + 7).tolist() and last == wl


def test_mid_automaton_takes_the_wide_path():
    """A definite automaton of ~27K states: its 16-bit 1-base table does not
    fit shared memory, so it is compiled to the wide form (hot table in
    shared memory, cold transitions from L2) -- counts, rows and ranges
    against the oracle."""
    rng = np.random.default_rng(11)
    lits = set()
    while len(lits) < 3000:
        lits.add("".join(rng.choice(list("acgt"), size=14)))
    lits = sorted(lits)
    dfa = dfa_of("\n".join(lits))
    assert 16384 < dfa.state_count <= 32767
    n = 1 << 20
    sym = rng.integers(0, 4, n).astype(np.uint8)
    for k in range(300):
        lit = lits[int(rng.integers(0, len(lits)))]
        p = int(rng.integers(0, n - len(lit)))
        sym[p:p + len(lit)] = ["acgt".index(c) for c in lit]
    sym[rng.integers(0, n, 50)] = 4
    ctx = _native.DeviceContext(0)
    dh = ctx.dfa(dfa)
    assert dh.info["strategy_name"] == "lookback" and dh.info["tables_in_smem"] == 0
    want, rows, _ = O.ref_run(dfa, sym, 4, 10, True)
    sh = ctx.upload_codes(sym)
    assert ctx.count(dh, sh).tolist() == want.tolist() and want.sum() >= 300
    got, grows = ctx.locate(dh, sh)
    assert got.tolist() == want.tolist() and np.array_equal(grows, rows)
    wc, wl = O.ref_sequential_count(dfa, sym[777:600_001], state=5)
    c, last, _ = ctx.scan_range(dh, sh, 777, 600_001, 5)
    assert c.tolist() == wc.tolist() and last == wl


@pytest.mark.parametrize("config", [3, 4])
def test_dynamic_tiles_and_split_tails(monkeypatch, config):
    """Count-mode work items beyond two rounds come from a device counter and
    the last round is cut into block ranges entered by lookback mid-chunk
    (scan_fast.cu): every split (1, 2 parts) and the static round-robin
    give the oracle's counts, whole sequence and unaligned ranges from an
    explicit entry state."""
    monkeypatch.setenv("KS_TILE_LB", "1")   # 128-base units: > 6 rounds of tiles at this size
    w = workloads.make(config, 150_000_037)
    codes = ks.encode_bytes(w.ascii.tobytes())
    want = O.ref_run(w.dfa, codes, 16, 10, False)[0]
    rng = np.random.default_rng(config)
    ranges = []
    for _ in range(3):
        b, e = sorted(rng.integers(0, codes.size, 2).tolist())
        entry = int(rng.integers(0, w.dfa.state_count))
        ranges.append((b, e, entry, *O.ref_sequential_count(w.dfa, codes, b, e, entry)))
    c2 = _native.DeviceContext(0)
    dh = c2.dfa(w.dfa)
    sh = c2.upload_codes(codes)
    for env in ({"KS_STATIC_TILES": "1"}, {"KS_SPLIT_PARTS": "1"}, {"KS_SPLIT_PARTS": "2"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        assert c2.count(dh, sh).tolist() == want.tolist(), env
        for b, e, entry, w2, last in ranges:
            g2, ex, _ = c2.scan_range(dh, sh, b, e, entry)
            assert g2.tolist() == w2.tolist() and ex == last, (env, b, e)
        for k in env:
            monkeypatch.delenv(k)


def test_pipelined_allreduce_single_rank_nccl():
    """bench.py's overlapped per-step all-reduce (PipelinedAllReduce: the scan
    kernel raises a device flag, a side stream waits on it with
    ks_stream_wait_value32 and runs the NCCL collective) on a one-rank NCCL
    group with the scan grid leaving SMs free (ks_set_reserved_sms): every
    step's counts reach their buffer and the last one the pinned buffer."""
    import socket

    import torch.distributed as dist

    import bench as B

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=dev)
    prev = torch.cuda.current_stream()
    try:
        c2 = _native.DeviceContext(0)
        stream = torch.cuda.Stream(dev)
        torch.cuda.set_stream(stream)
        c2.set_stream(stream.cuda_stream)
        with pytest.raises(ValueError):
            c2.set_reserved_sms(10_000)
        c2.set_reserved_sms(B.PipelinedAllReduce.RESERVED_SMS)
        w = workloads.make(3, 3_000_017)
        codes = ks.encode_bytes(w.ascii.tobytes())
        want = O.ref_sequential_count(w.dfa, codes)[0]
        dh = c2.dfa(w.dfa)
        sh = c2.upload_codes(codes)
        ne = w.dfa.n_expressions
        pin = torch.zeros(max(ne, 1), dtype=torch.int64).pin_memory()
        pipe = B.PipelinedAllReduce(ne, dev, pin)
        for _ in range(7):
            pipe.step(lambda cp, fp, v: c2.count_shard_async_signal(dh, sh, 0, codes.size, 0, 0, cp, fp, v))
        pipe.finish()
        c2.async_wait()
        torch.cuda.synchronize()
        assert pin.numpy()[:ne].tolist() == want.tolist()
        assert pipe.last().cpu().numpy()[:ne].tolist() == want.tolist()
        assert int(pipe.flag.item()) == pipe.seq == 7
        # every step's buffer holds that step's (identical) counts
        assert all(pipe.bufs[k].cpu().numpy()[:ne].tolist() == want.tolist() for k in range(7))
        c2.set_reserved_sms(0)
        assert c2.count(dh, sh).tolist() == want.tolist()
    finally:
        torch.cuda.set_stream(prev)
        dist.destroy_process_group()


@pytest.mark.parametrize("generic", [False, True])
def test_count_shard_signal_raises_flag(monkeypatch, generic):
    """ks_count_shard_async_signal: the fused kernel's finalizing CTA (or, on
    the multi-launch generic path, a stream write after the finalize) sets
    the flag once the counts are final; a side stream gated by
    ks_stream_wait_value32 reads the final counts."""
    if generic:
        monkeypatch.setenv("KS_DISABLE_FAST", "1")
    w = workloads.make(2, 2_000_003)
    codes = ks.encode_bytes(w.ascii.tobytes())
    want = O.ref_sequential_count(w.dfa, codes)[0]
    c2 = _native.DeviceContext(0)
    dh = c2.dfa(w.dfa)
    sh = c2.upload_codes(codes)
    ne = w.dfa.n_expressions
    dev = torch.device("cuda", 0)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    counts = torch.zeros(max(ne, 1), dtype=torch.int64, device=dev)
    side = torch.cuda.Stream(dev)
    got = torch.zeros_like(counts)
    for v in (3, 4):
        c2.count_shard_async_signal(dh, sh, 0, codes.size, 0, 0, counts.data_ptr(), flag.data_ptr(), v)
        with torch.cuda.stream(side):
            _native.DeviceContext.stream_wait_value32(side.cuda_stream, flag.data_ptr(), v)
            got.copy_(counts)
        side.synchronize()
        assert got.cpu().numpy()[:ne].tolist() == want.tolist()
        assert int(flag.item()) == v
    c2.async_wait()


def test_back_to_back_dynamic_and_deferred_wait(monkeypatch):
    """Back-to-back async counts (deferred griddepcontrol.wait: each scan
    starts while the previous call drains) alternating automata, sequences
    and the static / dynamic item paths (> 6 rounds of tiles at 64-base
    units), interleaved with signalled shard counts and a MAPSCAN call: every
    call's counts are the oracle's."""
    monkeypatch.setenv("KS_TILE_LB", "0")
    ctx = _native.DeviceContext(0)
    work = []
    for cfg, n in ((3, 60_000_013), (4, 60_000_011), (2, 3_000_017), (5, 1_000_003)):
        w = workloads.make(cfg, n)
        codes = ks.encode_bytes(w.ascii.tobytes())
        want = O.ref_run(w.dfa, codes, 16 if cfg != 5 else 1, 10, False)[0]
        work.append((ctx.dfa(w.dfa), ctx.upload_codes(codes), want, codes.size))
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    outs = []
    v = 0
    for rep in range(3):
        for dh, sh, want, n in work:
            buf = torch.zeros(max(dh.n_expressions, 1), dtype=torch.int64).pin_memory()
            ctx.count_async(dh, sh, buf.numpy())
            outs.append((buf, want))
            if dh.info["strategy_name"] == "lookback":
                v += 1
                dbuf = torch.zeros(max(dh.n_expressions, 1), dtype=torch.int64, device="cuda")
                ctx.count_shard_async_signal(dh, sh, 0, n, 0, 0, dbuf.data_ptr(), flag.data_ptr(), v)
                outs.append((dbuf, want))
    ctx.async_wait()
    torch.cuda.synchronize()
    assert int(flag.item()) == v
    for buf, want in outs:
        assert buf.cpu().numpy()[: want.size].tolist() == want.tolist()


def test_upload_codes_host_packed(monkeypatch):
    """ks_seq_upload_codes of >= 8 Mi symbols packs on the host (worker pool,
    pinned staging ring, pieces copied while the next is packed): the
    sequence equals the device-packed one (counts, locate rows, ranges) and a
    code above 4 is rejected."""
    w = workloads.make(4, 20_000_003)
    codes = ks.encode_bytes(w.ascii.tobytes())
    want, want_rows = O.ref_run(w.dfa, codes, 16, 10, True)[:2]
    c2 = _native.DeviceContext(0)
    dh = c2.dfa(w.dfa)
    sh = c2.upload_codes(codes)
    monkeypatch.setenv("KS_DEVICE_PACK_CODES", "1")
    sd = c2.upload_codes(codes)
    monkeypatch.delenv("KS_DEVICE_PACK_CODES")
    for h in (sh, sd):
        got, rows = c2.locate(dh, h)
        assert got.tolist() == want.tolist() and np.array_equal(rows, want_rows)
    b, e = 1_234_567, 17_654_321
    assert c2.scan_range(dh, sh, b, e, 5)[0].tolist() == c2.scan_range(dh, sd, b, e, 5)[0].tolist()
    bad = codes.copy()
    bad[9_999_999] = 7
    with pytest.raises(ValueError, match="out of range"):
        c2.upload_codes(bad)


# ---------------------------------------------------------------- visit-class table (K = 2 fused count)

def _k2_dfa(rng):
    """A 1025..4095-state automaton (K = 2 fast table) with many short
    literals, so many accepting states enter the same state: rows copied
    for a 4th, 5th, ... intermediate multiset."""
    while True:
        lits = set()
        for _ in range(int(rng.integers(150, 420))):
            n = int(rng.choice([1, 2, 3, 4, 6, 8, 10, 12], p=[.02, .06, .1, .12, .2, .2, .15, .15]))
            lits.add("".join("acgt"[x] for x in rng.integers(0, 4, n)))
        lits = sorted(lits)
        rng.shuffle(lits)
        # 1-3 literals per expression: output multisets with repeated ids
        lines, i = [], 0
        while i < len(lits):
            k = int(rng.integers(1, 4))
            lines.append("|".join(lits[i:i + k]))
            i += k
        dfa = dfa_of("\n".join(lines))
        if 1100 <= dfa.state_count <= 4000:
            return dfa


@pytest.mark.gpu
def test_dense_hits_k3_ring_never_overflows():
    """A 3-base-stride automaton with 2-mers among its literals accepts in
    most steps: the hit ring's fill check must also run after the last of a
    block's 21 steps (13 pushes could pass between two checks and a lane at
    the threshold wrote past its ring into the histogram: wrong counts at
    1000 bases, an illegal access at 100000 -- found by tools/stress_class.py,
    seed 20261036)."""
    rng = np.random.default_rng(5)
    lits = ["ta", "ga", "cc", "act", "ggc"]
    lits += ["".join("acgt"[x] for x in rng.integers(0, 4, int(rng.integers(8, 13)))) for _ in range(60)]
    dfa = dfa_of("\n".join(lits))
    c = _native.DeviceContext(0)
    dh = c.dfa(dfa)
    assert dh.info["stride"] == 3, dh.info
    for n in (1000, 20_000, 100_000, 400_000, 3_000_001):
        codes = rng.integers(0, 4, n).astype(np.uint8)
        want = O.ref_sequential_count(dfa, codes)[0]
        sh = c.upload_codes(codes)
        for _ in range(2):
            assert c.count(dh, sh).tolist() == want.tolist(), n
        counts, rows = c.locate(dh, sh)
        assert counts.tolist() == want.tolist() and rows.shape[0] == int(want.sum()), n


@pytest.mark.gpu
@pytest.mark.parametrize("tile_lb", [None, "2", "5"])
def test_row_flags_and_plain_items(monkeypatch, tile_lb):
    """Per-tile row flags (SeqView::rowmask, computed when an upload ends) and
    the class count's plain-item loop: OTHER placed so that whole tiles are
    clean, single rows of a tile are dirty (one N in one lane's block), whole
    units and whole tiles are N, and the sequence ends inside a tile -- through
    the device encode, the device-packed and the host-packed codes uploads,
    every count equal to the oracle and to the ring kernel."""
    if tile_lb is not None:
        monkeypatch.setenv("KS_TILE_LB", tile_lb)
    rng = np.random.default_rng(77)
    dfa = _k2_dfa(rng)
    c = _native.DeviceContext(0)
    dh = c.dfa(dfa)
    assert dh.info["stride"] == 2, dh.info
    lb = int(tile_lb) if tile_lb is not None else 4
    unit = 64 << lb
    tile = 32 * unit
    for n in (6 * tile + 12345, (9 << 20) + 77):      # the second takes the host-packed codes upload
        codes = rng.integers(0, 4, n).astype(np.uint8)
        codes[tile + 5 * unit + 64 * 1 + 7] = 4                    # one N: row 1 of tile 1 dirty, the rest clean
        codes[2 * tile + 3 * unit: 2 * tile + 4 * unit] = 4          # a whole unit of N (all rows of tile 2)
        codes[3 * tile: 4 * tile] = 4                                # a whole tile of N
        codes[4 * tile + unit - 1] = 4                               # last base of a unit
        codes[4 * tile + 2 * unit] = 4                               # first base of a unit
        codes[n - 3:] = 4                                            # the ragged end
        want = O.ref_sequential_count(dfa, codes)[0]
        ascii_bytes = np.frombuffer(b"ACGTN", dtype=np.uint8)[codes].tobytes()
        for sh in (c.upload_codes(codes), c.upload_ascii(ascii_bytes)):
            assert c.count(dh, sh).tolist() == want.tolist(), (tile_lb, n)
            monkeypatch.setenv("KS_NO_CLS", "1")
            assert c.count(dh, sh).tolist() == want.tolist(), (tile_lb, n)
            monkeypatch.delenv("KS_NO_CLS")
            # ranges (per-chunk entry states, partial first and last blocks) on the same sequence
            for (b, e) in ((0, n), (tile + 17, 5 * tile + 4001), (n - 5000, n)):
                st = int(rng.integers(0, dfa.state_count))
                got, last, _ = c.scan_range(dh, sh, b, e, st)
                ref, ref_last = O.ref_sequential_count(dfa, codes, b, e, st)
                assert got.tolist() == ref.tolist() and last == ref_last, (tile_lb, n, b, e)


@pytest.mark.parametrize("seed", range(4))
def test_class_table_counts_vs_oracle(monkeypatch, seed):
    """The fused K = 2 count on the visit-class table (scan_fast CLS kernel)
    equals the oracle and the ring kernel (KS_NO_CLS=1) on automata with
    row copies, across N runs, OTHER symbols, tiny and block-ragged inputs."""
    rng = np.random.default_rng(1000 + seed)
    dfa = _k2_dfa(rng)
    c = _native.DeviceContext(0)
    dh = c.dfa(dfa)
    assert dh.info["stride"] == 2, dh.info
    for n in (0, 1, 2, 63, 64, 65, 4097, 200_003, 3_000_017):
        codes = rng.integers(0, 4, n).astype(np.uint8)
        codes[rng.random(n) < 0.002] = 4
        if n > 5000:
            codes[1000:1377] = 4          # an N run across block borders
            codes[4000:4064] = 4          # exactly one block
        sh = c.upload_codes(codes)
        want = O.ref_sequential_count(dfa, codes)[0]
        got = c.count(dh, sh)
        assert got.tolist() == want.tolist(), (seed, n)
        monkeypatch.setenv("KS_NO_CLS", "1")
        assert c.count(dh, sh).tolist() == want.tolist(), (seed, n)
        monkeypatch.delenv("KS_NO_CLS")
        # back to back on the persistent class counters (kept zero by the kernel)
        assert c.count(dh, sh).tolist() == want.tolist(), (seed, n)
