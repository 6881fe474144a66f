"""Data-parallel plumbing for multi-GPU protected inference.

The path shards by batch with no data exchange: shard g of G owns images
[g*N/G, (g+1)*N/G) and runs its own ABFT (local Cd1/Cd2, local block indices,
local So*).  The only collective is one all-gather per forward of fixed-size
per-layer verdict records (~100 B/layer/shard), so every rank ends with the whole
job's verdict table.  Works with NCCL (CUDA tensors) and gloo (CPU tensors; used by
the world-size-2 CPU tests).
"""
from __future__ import annotations

import numpy as np

STAGES = ["none", "reload", "coc", "rc", "clc", "fc", "discard", "recompute"]
REC_INTS = 16  # detected, stage, reloaded, recomputed, n_blocks, b0i, b0j, n_stages, stages[6], n_flagged, repaired
REC_LEN = REC_INTS + 1  # + max_rel_dev as float64 bits


def shard_range(global_batch: int, world: int, rank: int):
    """Contiguous, balanced batch shard [lo, hi) of `rank` (the first N % G shards
    get one extra image)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(global_batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def pack_reports(reports) -> np.ndarray:
    """LayerReports (in layer order) -> int64 array [L, REC_LEN]."""
    out = np.zeros((len(reports), REC_LEN), np.int64)
    for li, r in enumerate(reports):
        st = [STAGES.index(s) for s in r.stages_attempted][:6]
        b0 = r.corrected_blocks[0] if r.corrected_blocks else (-1, -1)
        row = [int(r.detected), STAGES.index(r.stage), int(r.weights_reloaded), int(r.recomputed),
               int(r.n_blocks), int(b0[0]), int(b0[1]), len(st)] + st + [0] * (6 - len(st)) + \
              [int(r.n_flagged), int(r.repaired_planes)]
        out[li, :REC_INTS] = row
        out[li, REC_INTS] = np.array([r.max_rel_dev], np.float64).view(np.int64)[0]
    return out


def unpack_reports(arr: np.ndarray):
    recs = []
    for row in np.asarray(arr, np.int64):
        ns = int(row[7])
        recs.append({
            "detected": bool(row[0]), "stage": STAGES[int(row[1])], "weights_reloaded": bool(row[2]),
            "recomputed": bool(row[3]), "n_blocks": int(row[4]),
            "first_block": (int(row[5]), int(row[6])) if row[5] >= 0 else None,
            "stages_attempted": [STAGES[int(s)] for s in row[8:8 + ns]],
            "n_flagged": int(row[14]), "repaired_planes": int(row[15]),
            "max_rel_dev": float(np.array([row[16]], np.int64).view(np.float64)[0]),
        })
    return recs


def gather_verdicts(reports, device=None):
    """All-gather every rank's packed per-layer records; returns [rank][layer] dicts.
    The only cross-GPU traffic of the ABFT path."""
    import torch
    import torch.distributed as dist
    local = torch.from_numpy(pack_reports(reports))
    if device is not None:
        local = local.to(device)
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [unpack_reports(local.cpu().numpy())]
    bufs = [torch.empty_like(local) for _ in range(dist.get_world_size())]
    dist.all_gather(bufs, local)
    return [unpack_reports(b.cpu().numpy()) for b in bufs]


def summarize(table) -> dict:
    """Job-wide verdict summary from gather_verdicts' table."""
    out = {"shards": len(table), "layers": len(table[0]) if table else 0, "detected": 0, "by_stage": {}}
    for shard in table:
        for rec in shard:
            out["detected"] += int(rec["detected"])
            out["by_stage"][rec["stage"]] = out["by_stage"].get(rec["stage"], 0) + 1
    return out
