"""Drop-in for the reference's compiled kernel module (`kmerscan/_kernels.py`).

The reference exposes its numba kernels with raw-array signatures; callers
(its tests' ground truth, `tests/test_engine.py:6-15`) use ``scan_from``
directly.  Here the same signature runs on the GPU through the C ABI
(``ks_scan_range`` from an explicit entry state) -- no CPU loop.

``scan_from(trans, out_off, out_ids, sym, start, end, state, counts) -> last``
(`_kernels.py:18-29`): scan ``sym[start:end]`` from ``state``; ``counts`` is
incremented in place (the reference adds into the caller's array) and the
final state is returned.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .automaton import Dfa

__all__ = ["scan_from"]


def _dfa_of(trans, out_off, out_ids, ne: int) -> Dfa:
    return Dfa(transitions=np.ascontiguousarray(trans, dtype=np.int32).copy(),
               out_offsets=np.ascontiguousarray(out_off, dtype=np.int32).copy(),
               out_ids=np.ascontiguousarray(out_ids, dtype=np.int32).copy(),
               labels=tuple(str(i) for i in range(ne)), n_expressions=int(ne))


def scan_from(trans, out_off, out_ids, sym, start, end, state, counts):
    """One run over sym[start:end] from `state` on the device; adds the
    per-expression counts into `counts` and returns the final state."""
    counts = np.asarray(counts)
    start, end, state = int(start), int(end), int(state)
    ne = int(counts.shape[0])
    ctx = _native.context(0)
    dh = ctx.dfa(_dfa_of(trans, out_off, out_ids, ne))
    seg = np.ascontiguousarray(np.asarray(sym)[start:end], dtype=np.uint8)
    sh = ctx.upload_codes(seg)
    try:
        got, last, _ = ctx.scan_range(dh, sh, 0, seg.size, state)
    finally:
        sh.free()
        dh.free()
    if seg.size == 0:
        return state
    counts += got.astype(counts.dtype)
    return last
