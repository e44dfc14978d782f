"""Full-size parity: every BASELINE config (C1..C5) at its BASELINE size,
scanned by the device path through the C ABI and by the oracle (the C
restatement of the reference's run(), oracle/ref_scan.c) on the same seeded
input.  Bit-exact counts for all five, sorted (offset, id) rows for the
configs that locate (C1, C2, C4 -- C4's offsets run past 2^31).

Reference: /root/reference/pkg/tests/test_acceptance.py:77-106 (four-way
equality including locations), engine.py:176-179 (sorted rows, len == total).
C5 runs the oracle with one worker: with more, every chunk speculates all
1024 states (|Q|x the work).
"""

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_1509_01506_b200 as ks
from paper_1509_01506_b200 import _native, workloads
from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

LOCATE = {1: True, 2: True, 3: False, 4: True, 5: False}


def host_codes(ascii_: np.ndarray) -> np.ndarray:
    """ks.encode_bytes for whitespace-free input, in parallel 64 MiB pieces
    (the oracle's input; the device encodes the same bytes on its own)."""
    lut = ks.alphabet.BYTE_CODES
    assert not np.any(lut[np.frombuffer(b" \t\r\n", np.uint8)] != ks.alphabet.DROP)
    out = np.empty(ascii_.size, dtype=np.uint8)
    step = 64 << 20

    def piece(lo):
        np.take(lut, ascii_[lo:lo + step], out=out[lo:lo + step])

    with ThreadPoolExecutor(os.cpu_count() or 4) as ex:
        list(ex.map(piece, range(0, ascii_.size, step)))
    assert not np.any(out == ks.alphabet.DROP)
    return out


@pytest.fixture(scope="module")
def ctx():
    return _native.context(0)


@pytest.mark.parametrize("config", [1, 2, 3, 4, 5])
def test_full_size_configs_vs_oracle(ctx, config):
    w = workloads.make(config)
    assert w.n == workloads.FULL_SIZES[config]
    codes = host_codes(w.ascii)
    workers = 1 if config == 5 else 4 if config == 1 else (os.cpu_count() or 1)
    want, want_rows, _ = O.ref_run(w.dfa, codes, workers, 10, LOCATE[config])

    sh = ctx.upload_ascii(w.ascii)          # device encode of the raw bytes
    dh = ctx.dfa(w.dfa)
    if LOCATE[config]:
        counts, rows = ctx.locate(dh, sh)
        assert rows.shape == want_rows.shape, (config, rows.shape, want_rows.shape)
        assert np.array_equal(rows, want_rows), config
        assert rows.shape[0] == int(want.sum())
        if config == 4:
            assert int(rows[-1, 0]) > 2**31     # offsets beyond int32
    else:
        counts = ctx.count(dh, sh)
    assert counts.tolist() == want.tolist(), config
    assert int(want.sum()) > 0

    # the drop-in API on the reference's own input form (Sequence of codes)
    seq = ks.Sequence(codes)
    rep = ks.run(w.dfa, seq, ks.EngineConfig(workers=workers, mode="locate" if LOCATE[config] else "count"))
    assert rep.per_expression_counts.tolist() == want.tolist(), config
    if LOCATE[config]:
        assert np.array_equal(rep.locations, want_rows), config
    # the end-to-end call from host bytes
    assert ctx.count_host_ascii(dh, w.ascii).tolist() == want.tolist(), config
