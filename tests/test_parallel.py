"""Sharded matching: shard bounds, the map all-gather across 2 processes (gloo,
CPU) and the GPU map/combine kernels against the oracle.

Theorem 3: any division of the text gives the same result;
Lemma 1: the state of a concatenation composes the parts'."""
import os
import socket

import numpy as np
import pytest

import oracle as O
import paper_1405_0562_b200 as P
from paper_1405_0562_b200 import parallel as PL
import workloads as W

CFG2 = ("([0-4]{5}[5-9]{5})*", b"0123456789")


def test_shard_bounds_cover_text():
    for n in (0, 1, 7, 10, 1000, 268_435_450):
        for world in (1, 2, 3, 8):
            b = [PL.shard_bounds(n, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            sizes = [y - x for x, y in b]
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)


def _oracle_map(d: O.OracleDFA, text: np.ndarray) -> np.ndarray:
    """f_text(q) for every DFA state q, by the oracle's Alg. 2 from each q."""
    table = d.table.astype(np.int64)
    q = np.arange(d.n, dtype=np.int64)
    for b in text.tolist():
        q = table[q, b]
    return q


def _worker(rank, world, port, text, rx, alpha, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = O.OracleDFA(rx, alpha)
    a, b = PL.shard_bounds(text.size, world, rank)
    local = torch.from_numpy(_oracle_map(d, text[a:b]).astype(np.int32))
    maps = PL.gather_maps(local)
    q = 0
    for r in range(world):          # the reduction sfa_combine_maps runs on the device
        q = int(maps[r, q])
    out[rank] = q
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_gather_maps_two_ranks_gloo(world):
    """World-size-2 gloo run of the N>1 host logic: shard bounds, the map
    all-gather in rank order and the in-order reduction give the oracle's
    whole-text state (shards cut mid-block and mid-word)."""
    import torch.multiprocessing as mp
    rx, alpha = CFG2
    d = O.OracleDFA(rx, alpha)
    for text in (W.cfg2_accepted(3_001)[:30_007], W.cfg2_rejected(text=W.cfg2_accepted(2_000))):
        mgr = mp.Manager()
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), text, rx, alpha, out), nprocs=world, join=True)
        q_exp, _ = d.run(text)
        assert [out[r] for r in range(world)] == [q_exp] * world


@pytest.mark.gpu
def test_match_map_and_combine_on_gpu(cuda_ok):
    """sfa_match_map per shard + sfa_combine_maps = the oracle's result, for
    shards on both scan kernels (direct < 4 MiB <= TMA) and every compose mode."""
    import torch
    for rx, alpha, text in [(*CFG2, W.cfg2_accepted(1_300_000)), ("(ab|ba)*c", b"abc", W.cfg1_accepted(3_000_000)),
                            (".*a[ab]{8}", b"ab", W.cfg4_text(9_000_001)), (W.cfg3_regex(), None, W.cfg3_text(9 << 20, plant=True))]:
        d = O.OracleDFA(rx, alpha)
        sfa = P.SFA(rx, alpha)
        nD = sfa.info()["dfa_states"]
        dt = torch.from_numpy(text).cuda()
        exp = d.run(text)
        for world in (1, 2, 3, 7):
            maps = torch.empty((world, nD), dtype=torch.int32, device="cuda")
            for r in range(world):
                a, b = PL.shard_bounds(text.size, world, r)
                sfa.match_map(dt[a:b], maps[r])
            res = torch.zeros(2, dtype=torch.int32, device="cuda")
            sfa.combine_maps(maps, world, res)
            torch.cuda.synchronize()
            q, acc = res.cpu().tolist()
            assert (q, bool(acc)) == exp, (rx, world)
        # the mapping itself, bit-exact against the oracle's Alg. 2 from every q
        small = text[:20_011]
        m = torch.empty(nD, dtype=torch.int32, device="cuda")
        sfa.match_map(dt[:small.size], m)
        torch.cuda.synchronize()
        assert (m.cpu().numpy() == _oracle_map(d, small)).all(), rx


def _sharded_worker(rank, world, port, text, rx, alpha, out):
    """One rank of parallel.match_sharded: its shard on the GPU (sfa_match_map),
    the maps all-gathered over gloo (staged through the host), the in-order
    reduction on the device (sfa_combine_maps)."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    sfa = P.SFA(rx, alpha)
    a, b = PL.shard_bounds(text.size, world, rank)
    out[rank] = PL.match_sharded(sfa, torch.from_numpy(text[a:b]).cuda())
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_match_sharded_end_to_end(cuda_ok, world):
    """The product's parallel.match_sharded with world ranks (processes) on one
    GPU over gloo: every rank returns the oracle's whole-text result; shards
    are cut mid-block (cfg2) and mid-word (cfg3), and span both scan kernels."""
    import torch.multiprocessing as mp
    for rx, alpha, text in [(*CFG2, W.cfg2_accepted(1_300_011)), (*CFG2, W.cfg2_rejected(text=W.cfg2_accepted(700_000))),
                            (W.cfg3_regex(), None, W.cfg3_text(9 << 20, plant=True))]:
        d = O.OracleDFA(rx, alpha)
        mgr = mp.Manager()
        out = mgr.dict()
        mp.spawn(_sharded_worker, args=(world, _free_port(), text, rx, alpha, out), nprocs=world, join=True)
        assert [out[r] for r in range(world)] == [d.run(text)] * world
