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
    back = D.unpack_reports(D.pack_reports(reps))
    for r, b in zip(reps, back):
        assert b["detected"] == r.detected and b["stage"] == r.stage
        assert b["stages_attempted"] == r.stages_attempted
        assert b["max_rel_dev"] == r.max_rel_dev


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
