"""Multi-rank sharded scan logic (paper_1509_01506_b200.distributed) on CPU:
world_size 2 over gloo, with an oracle-backed shard scanner standing in for
the device one (the exchange, composition and reduction are what is tested;
the per-rank device scan is covered by the GPU tests)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_1509_01506_b200 as ks
from paper_1509_01506_b200 import distributed as D
from paper_1509_01506_b200 import workloads


class OracleShardScanner:
    """Shard scanner over local codes with global row offsets (test only)."""

    def __init__(self, dfa, codes, row_base):
        self.dfa = dfa
        self.codes = codes
        self.row_base = row_base
        self.n_states = dfa.state_count
        self.n_expressions = dfa.n_expressions

    def segment_map(self, begin, end):
        from oracle import oracle as O
        return np.array([O.ref_sequential_count(self.dfa, self.codes, begin, end, q)[1]
                         for q in range(self.n_states)], dtype=np.int32)

    def scan(self, begin, end, entry, locate):
        from oracle import oracle as O
        counts, _, rows = O.ref_scan_rows(self.dfa, self.codes, begin, end, entry, self.row_base)
        return counts, rows if locate else None


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dfa, codes = case()
        b, e = D.shard_bounds(codes.size, world)[rank]
        scanner = OracleShardScanner(dfa, codes[b:e], b)
        counts, rows = D.run_sharded(scanner, 0, e - b, locate=True)
        out[rank] = (counts.tolist(), rows.tolist())
    finally:
        dist.destroy_process_group()


def toy_case():
    dfa = ks.build_dfa(ks.expand_to_literals(ks.parse_expressions("acg\ncat\ncta\ntta\nta")))
    codes = np.random.default_rng(3).integers(0, 5, 5003).astype(np.uint8)
    return dfa, codes


def perm_case():
    dfa = workloads.permutation_dfa(64)
    codes = np.random.default_rng(4).integers(0, 4, 3001).astype(np.uint8)
    return dfa, codes


@pytest.mark.parametrize("case", [toy_case, perm_case])
@pytest.mark.parametrize("world", [2])
def test_sharded_equals_sequential(case, world):
    from oracle import oracle as O
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, case, out), nprocs=world, join=True)
    dfa, codes = case()
    want, _, want_rows = O.ref_scan_rows(dfa, codes, 0, codes.size, 0, 0)
    for r in range(world):
        assert out[r][0] == want.tolist()
    rows = [row for r in range(world) for row in out[r][1]]
    assert rows == want_rows.tolist()


def test_shard_bounds():
    for n in (0, 1, 63, 64, 1000, 123457):
        for world in (1, 2, 3, 8):
            b = D.shard_bounds(n, world)
            assert b[0][0] == 0 and b[-1][1] == n and len(b) == world
            for (a0, a1), (b0, _) in zip(b, b[1:]):
                assert a1 == b0 and a0 <= a1 and (a1 % 64 == 0 or a1 == n)


def test_compose_entry():
    maps = np.array([[1, 2, 0], [2, 2, 1], [0, 1, 2]])
    assert D.compose_entry(maps, 0) == 0
    assert D.compose_entry(maps, 1) == 1
    assert D.compose_entry(maps, 2) == 2
