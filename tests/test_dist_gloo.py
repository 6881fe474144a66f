"""Multi-rank host logic on CPU: world_size 2 over gloo (127.0.0.1).

Covers the N>1 data-parallel path without a GPU: batch sharding and the per-shard
verdict all-gather that is the only collective of the protected forward."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2003_12203_b200 import dist as D
from paper_2003_12203_b200.ftconv import LayerReport


def test_shard_range_partitions_the_batch():
    for N in (1, 7, 64, 128, 256):
        for G in (1, 2, 4, 8):
            if G > N:
                continue
            spans = [D.shard_range(N, G, g) for g in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == N
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    assert D.shard_range(64, 8, 3) == (24, 32)
    with pytest.raises(ValueError):
        D.shard_range(8, 2, 2)


def _rep(rank, layer):
    r = LayerReport(detected=bool((rank + layer) % 2), stage="coc" if (rank + layer) % 2 else "none",
                    corrected_blocks=[(rank, layer)] if (rank + layer) % 2 else [],
                    stages_attempted=["coc"] if (rank + layer) % 2 else [], max_rel_dev=1e-3 * (layer + 1),
                    n_flagged=rank + layer, n_blocks=1 if (rank + layer) % 2 else 0)
    return r


def test_pack_roundtrip():
    reps = [_rep(1, l) for l in range(5)]
    back = D.unpack_reports(D.pack_reports(reps, lo=32))
    for r, b in zip(reps, back):
        assert b["detected"] == r.detected and b["stage"] == r.stage
        assert b["stages_attempted"] == r.stages_attempted
        assert b["max_rel_dev"] == r.max_rel_dev
        assert b["corrected_blocks"] == list(r.corrected_blocks)
        assert b["image_offset"] == 32 and not b["blocks_truncated"]


def test_pack_keeps_every_block_up_to_capacity():
    """A row correction lists one block per kernel: the record carries the full list up
    to BLOCK_CAP plus the true count (and flags truncation beyond it)."""
    many = [(3, j) for j in range(D.BLOCK_CAP + 10)]
    r = LayerReport(detected=True, stage="rc", corrected_blocks=many, stages_attempted=["coc", "rc"],
                    n_blocks=len(many))
    few = LayerReport(detected=True, stage="rc", corrected_blocks=many[:40], stages_attempted=["coc", "rc"],
                      n_blocks=40)
    b_many, b_few = D.unpack_reports(D.pack_reports([r, few], lo=8))
    assert b_few["corrected_blocks"] == many[:40] and not b_few["blocks_truncated"]
    assert b_many["n_blocks"] == len(many) and b_many["blocks_truncated"]
    assert b_many["corrected_blocks"] == many[:D.BLOCK_CAP]
    glob = D.global_blocks([[D.unpack_reports(D.pack_reports([few], lo=8))[0]]])
    assert glob[0] == [(11, j) for j in range(40)]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    reps = [_rep(rank, l) for l in range(4)]
    table = D.gather_verdicts(reps)
    q.put((rank, [[rec["stage"] for rec in shard] for shard in table], D.summarize(table)))
    dist.barrier()
    dist.destroy_process_group()


def _shard_worker(rank, world, port, q):
    """The bench's sharded harness minus the device: shard the global batch, report
    shard-local blocks, all-gather the packed records, map them to global images."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = D.shard_range(64, world, rank)
    reps = [LayerReport(detected=True, stage="coc", corrected_blocks=[(hi - lo - 1, 5 + rank)],
                        stages_attempted=["coc"], n_blocks=1),
            LayerReport()]
    table = D.gather_verdicts(reps, lo=lo)
    q.put((rank, D.global_blocks(table), D.summarize(table)))
    dist.barrier()
    dist.destroy_process_group()


def _det_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rec = torch.zeros((3, 2), dtype=torch.int64)
    rec[:, 1] = torch.tensor([1e-6, 2e-6, 3e-6], dtype=torch.float64).view(torch.int64)
    if rank == 1:
        rec[2, 0] = 5  # shard 1 flagged 5 positions of layer 2
    g = D.gather_detect_records(rec)
    q.put((rank, tuple(g.shape), D.any_flagged(g), int(g[1, 2, 0]), float(g[0, 1, 1].view(torch.float64))))
    dist.barrier()
    dist.destroy_process_group()


def test_detect_records_allgather_world2_gloo():
    """The clean path's per-layer CoC-D records are all-gathered as one tensor; a flag
    on any shard is visible on every rank (which then gathers the full reports)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_det_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, shape, flagged, n, mrd in got:
        assert shape == (2, 3, 2) and flagged and n == 5 and mrd == 2e-6


def test_sharded_verdicts_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, glob, summ in got:
        # shard 0 owns images 0..31, shard 1 32..63; each corrected its last local image
        assert glob == {0: [(31, 5), (63, 6)]}
        assert summ["shards"] == 2 and summ["detected"] == 2 and summ["corrected_blocks"] == 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_verdict_allgather_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = [[("coc" if (r + l) % 2 else "none") for l in range(4)] for r in range(2)]
    for rank, stages, summ in got:
        assert stages == expect
        assert summ["shards"] == 2 and summ["detected"] == 4
