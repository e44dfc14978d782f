"""The C-ABI library: it loads, exports every symbol include/kmerscan_b200.h
declares, reports CUDA absence as an error (no crash, no CPU fallback), and the
product package never touches the oracle.  No GPU needed."""

import ctypes
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1509_01506_b200 import _native

REPO = Path(__file__).resolve().parents[1]
HEADER = REPO / "include" / "kmerscan_b200.h"


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^KS_API\s+[\w\s\*]+?\b(ks_\w+)\(", text, flags=re.M)))


def test_header_declares_api():
    syms = header_symbols()
    assert "ks_count" in syms and "ks_locate" in syms and "ks_dfa_upload" in syms
    assert len(syms) >= 20


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert set(header_symbols()) == set(_native.EXPORTED)


def test_version_and_errors_without_device():
    lib = _native.library()
    assert b"sm_100a" in lib.ks_version()
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    rc = lib.ks_open(0, ctypes.byref(h))
    assert rc != 0
    assert lib.ks_last_error()


def test_product_fails_loudly_without_library():
    code = ("import paper_1509_01506_b200 as ks\n"
            "try:\n"
            "    ks.run(ks.build_dfa(ks.expand_to_literals(ks.parse_expressions('acg'))), "
            "ks.sequence_from_text('acgt'))\n"
            "except RuntimeError as e:\n"
            "    print('RAISED', e)\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=REPO, capture_output=True, text=True,
                         env={"KMERSCAN_B200_LIB": "/nonexistent/libkmerscan_b200.so", "PATH": "/usr/bin"})
    assert "RAISED" in out.stdout, out.stderr
    assert "native library not found" in out.stdout


def test_product_never_imports_oracle():
    for path in (REPO / "paper_1509_01506_b200").rglob("*.py"):
        text = path.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", text, flags=re.M), path


def _blk_slot(g, lb):
    u = g >> lb
    return ((u >> 5) << (5 + lb)) | ((g & ((1 << lb) - 1)) << 5) | (u & 31)


def _pack_reference(data: bytes, lb: int):
    """Straight restatement of the wire format (encode.cu header) in numpy."""
    x = np.frombuffer(data, dtype=np.uint8).astype(np.int64)
    lx = x | 0x20
    base = np.isin(lx, [ord(c) for c in "acgt"])
    ws = np.isin(x, [9, 10, 13, 32])
    code = np.where(base, ((x >> 1) ^ (x >> 2)) & 3, 0)
    other = ~base & ~ws
    nblk = (x.size + 63) // 64
    tile = 32 << lb
    slots = max(-(-nblk // tile) * tile, 1)
    bases = np.zeros(2 * slots, dtype=np.uint64)
    nmask = np.zeros(slots, dtype=np.uint64)
    for g in range(nblk):
        s = _blk_slot(g, lb)
        c = code[64 * g: 64 * g + 64]
        o = other[64 * g: 64 * g + 64]
        for i in range(c.size):
            bases[2 * s + (i >> 5)] |= np.uint64(int(c[i]) << (2 * (i & 31)))
            nmask[s] |= np.uint64(int(o[i]) << i)
    return bases, nmask, int(ws.any()) | (int(other.any()) << 1)


@pytest.mark.parametrize("n,lb,alphabet", [
    (0, 0, b"acgt"), (1, 0, b"acgt"), (63, 1, b"ACGTacgt"), (64, 0, b"acgtN"), (4097, 2, b"acgtACGTnNx-"),
    (70_000, 4, b"acgt"), (70_001, 3, b"acgt \n"), (9000, 1, b"\x00\xffacgt\t\r"),
])
@pytest.mark.parametrize("scalar", [False, True])
def test_host_packer_matches_wire_format(n, lb, alphabet, scalar, monkeypatch):
    """ks_pack_host_ascii (AVX-512 and scalar paths, run in a subprocess for
    the scalar switch) reproduces the documented wire format bit for bit."""
    rng = np.random.default_rng(n * 7 + lb)
    data = bytes(np.frombuffer(alphabet, dtype=np.uint8)[rng.integers(0, len(alphabet), size=n)])
    want = _pack_reference(data, lb)
    if scalar:
        code = ("import sys, numpy as np; from paper_1509_01506_b200 import _native;"
                f"b, m, f = _native.pack_host_ascii(open(sys.argv[1], 'rb').read(), {lb});"
                "np.save(sys.argv[2], np.concatenate([b, m, np.array([f], dtype=np.uint64)]))")
        import tempfile
        with tempfile.TemporaryDirectory() as d:
            Path(d, "in").write_bytes(data)
            env = dict(__import__("os").environ, KS_HOST_SCALAR="1")
            subprocess.run([sys.executable, "-c", code, str(Path(d, "in")), str(Path(d, "out.npy"))],
                           check=True, env=env, cwd=REPO)
            out = np.load(Path(d, "out.npy"))
        k = want[0].size
        got = (out[:k], out[k:-1], int(out[-1]))
    else:
        got = _native.pack_host_ascii(data, lb)
    assert got[2] == want[2]
    nblk = (n + 63) // 64
    slots = [_blk_slot(g, lb) for g in range(nblk)]
    assert np.array_equal(got[1][slots], want[1][slots])
    assert np.array_equal(got[0].reshape(-1, 2)[slots], want[0].reshape(-1, 2)[slots])


def _wire_decode(bases, special, n_bytes):
    """Retained symbol codes (0..4) of a wire buffer, by the documented rules."""
    out = []
    for g in range((n_bytes + 63) // 64):
        for i in range(64):
            code = (int(bases[2 * g + (i >> 5)]) >> (2 * (i & 31))) & 3
            if (int(special[g]) >> i) & 1:
                if code == 1:
                    continue        # dropped
                out.append(4)       # OTHER
            else:
                out.append(code)
    return np.array(out, dtype=np.uint8)


WIRE_CASES = [
    b">s1 demo\nctacat\n", b">h\r\nACGT\r\nacgN\r\n>h2\r\nTTTT", b">h\rAC\rGT\r>x\r\rnn",
    b"ac>gt\n>hdr\n>hdr2\nA C\tG T\n\n\n", b"", b">" + b"x" * 300 + b"\n" + b"acgt" * 70 + b"\n>y\r\n" + b"TTGCA" * 40,
]


@pytest.mark.parametrize("k", range(len(WIRE_CASES)))
@pytest.mark.parametrize("fasta", [True, False])
def test_host_wire_packer(k, fasta):
    """ks_pack_host_wire against ingest's own host normalisation (the
    reference's load_sequence rules), AVX-512 and scalar paths."""
    from paper_1509_01506_b200.ingest import strip_fasta_headers
    import paper_1509_01506_b200 as ks
    data = WIRE_CASES[k]
    rng = np.random.default_rng(k)
    data += bytes(rng.choice(list(b"acgtN \n\r>"), size=int(rng.integers(0, 3000))))
    want = ks.encode_bytes(strip_fasta_headers(data) if fasta else data)
    bases, special, kept = _native.pack_host_wire(data, fasta)
    assert kept == want.size
    assert _wire_decode(bases, special, len(data)).tolist() == want.tolist()
    code = ("import sys, numpy as np; from paper_1509_01506_b200 import _native;"
            f"b, s, k = _native.pack_host_wire(open(sys.argv[1], 'rb').read(), {fasta});"
            "np.save(sys.argv[2], np.concatenate([b, s, np.array([k], dtype=np.uint64)]))")
    import os
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        Path(d, "in").write_bytes(data)
        subprocess.run([sys.executable, "-c", code, str(Path(d, "in")), str(Path(d, "out.npy"))], check=True,
                       env=dict(os.environ, KS_HOST_SCALAR="1"), cwd=REPO)
        out = np.load(Path(d, "out.npy"))
    assert int(out[-1]) == want.size
    nb = special.size
    assert _wire_decode(out[:2 * nb], out[2 * nb:3 * nb], len(data)).tolist() == want.tolist()


@pytest.mark.parametrize("n,lb", [(0, 0), (1, 0), (63, 1), (64, 2), (200_003, 3), (70_001, 4)])
@pytest.mark.parametrize("scalar", [False, True])
def test_host_codes_packer_matches_ascii_packer(n, lb, scalar):
    """ks_pack_host_codes (the packed codes upload's host side; AVX-512 and
    scalar paths) gives the ASCII packer's tile-slot output for the same
    sequence spelled ACGTN, padding included; a code above 4 is rejected."""
    rng = np.random.default_rng(n + 17 * lb)
    codes = rng.choice(np.array([0, 1, 2, 3, 4], dtype=np.uint8), size=n, p=[0.24, 0.24, 0.24, 0.24, 0.04])
    ascii_ = np.frombuffer(b"ACGTN", dtype=np.uint8)[codes].tobytes()
    want_b, want_m, _ = _native.pack_host_ascii(ascii_, lb)
    if scalar:
        code = ("import sys, numpy as np; from paper_1509_01506_b200 import _native;"
                f"b, m = _native.pack_host_codes(np.load(sys.argv[1]), {lb});"
                "np.save(sys.argv[2], np.concatenate([b, m]))")
        import tempfile
        with tempfile.TemporaryDirectory() as d:
            np.save(Path(d, "in.npy"), codes)
            env = dict(__import__("os").environ, KS_HOST_SCALAR="1")
            subprocess.run([sys.executable, "-c", code, str(Path(d, "in.npy")), str(Path(d, "out.npy"))],
                           check=True, env=env, cwd=REPO)
            out = np.load(Path(d, "out.npy"))
        got_b, got_m = out[:want_b.size], out[want_b.size:]
    else:
        got_b, got_m = _native.pack_host_codes(codes, lb)
    assert np.array_equal(got_b, want_b) and np.array_equal(got_m, want_m)
    if n:
        bad = codes.copy()
        bad[n // 2] = 5
        with pytest.raises(ValueError, match="out of range"):
            _native.pack_host_codes(bad, lb)
