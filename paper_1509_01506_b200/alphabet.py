"""Five-class symbol alphabet (host side).

Mirrors the reference's byte normalisation (`kmerscan/alphabet.py:13-47`):

* ``a/A -> 0, c/C -> 1, g/G -> 2, t/T -> 3`` (case folded, so soft-masked
  lowercase bases match exactly like uppercase ones);
* the four ASCII whitespace bytes (space, TAB, CR, LF) are *dropped*
  (``DROP``), so match offsets count post-drop symbols;
* every other byte value is ``OTHER`` (4): ``N``, IUPAC ambiguity codes,
  digits, ``\\v``, ``\\f``, bytes >= 0x80 and ``>`` when a FASTA file is read
  raw.

The device encoder (``ks_seq_upload_ascii``, csrc/encode.cu) implements the
same classification on the GPU; this module is the host-side table used for
in-memory text and for the parity tests.
"""

from __future__ import annotations

import numpy as np

A, C, G, T, OTHER = 0, 1, 2, 3, 4
N_SYMBOLS = 5
DROP = 5

BASES = "acgt"
BASE_CODES = {ch: code for code, ch in enumerate(BASES)}
CODE_CHARS = "acgt?"

WHITESPACE_BYTES = b" \t\r\n"


def _byte_code_table() -> np.ndarray:
    lut = np.full(256, OTHER, dtype=np.uint8)
    for code, ch in enumerate(BASES):
        lut[ord(ch)] = code
        lut[ord(ch.upper())] = code
    lut[np.frombuffer(WHITESPACE_BYTES, dtype=np.uint8)] = DROP
    lut.setflags(write=False)
    return lut


BYTE_CODES = _byte_code_table()


def encode_bytes(data: bytes) -> np.ndarray:
    """Bytes -> contiguous uint8 symbol codes with whitespace removed."""
    codes = BYTE_CODES[np.frombuffer(data, dtype=np.uint8)]
    keep = codes != DROP
    if keep.all():
        return np.ascontiguousarray(codes)
    return np.ascontiguousarray(codes[keep])


def encode(text: str) -> np.ndarray:
    """str -> codes; each non-ASCII character becomes exactly one OTHER.

    ``errors="replace"`` turns every unencodable character into one ``?``
    byte, which classifies as OTHER (reference `alphabet.py:40-42`).
    """
    return encode_bytes(text.encode("ascii", errors="replace"))


def decode(codes) -> str:
    """Codes -> diagnostic text ('?' renders OTHER)."""
    return "".join(CODE_CHARS[int(c)] for c in codes)
