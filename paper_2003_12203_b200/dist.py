"""Data-parallel plumbing for multi-GPU protected inference.

The path shards by batch with no data exchange: shard g of G owns images
[g*N/G, (g+1)*N/G) of the global batch and runs its own ABFT (local Cd1/Cd2, local
block indices, local So*, a tau_L calibrated on its own shard).  The only collective
is one all-gather per forward of fixed-size per-layer verdict records, so every rank
ends with the whole job's verdict table.  Two levels: the clean path's CoC-D records
(16 B per layer, gather_detect_records) are all-gathered on the device, stream-ordered
after the last layer, with no host round trip; only when some shard flagged a layer are
the full LayerReports of its error path all-gathered (gather_verdicts).  Works with NCCL
(CUDA tensors) and gloo (CPU tensors; used by the world-size-2 CPU tests).

Wire record (int64 words, one row per protected layer):
    [0] detected  [1] stage  [2] weights_reloaded  [3] recomputed
    [4] n_blocks (true count)  [5] n_stages  [6:12] stages_attempted
    [12] n_flagged  [13] repaired_planes  [14] max_rel_dev (float64 bits)
    [15] shard image offset lo (local block i + lo = global image index)
    [16 : 16 + 2*BLOCK_CAP] corrected_blocks (i, j), the first BLOCK_CAP of n_blocks
"""
from __future__ import annotations

import numpy as np

STAGES = ["none", "reload", "coc", "rc", "clc", "fc", "discard", "recompute"]
BLOCK_CAP = 64
HEAD = 16
REC_LEN = HEAD + 2 * BLOCK_CAP


def shard_range(global_batch: int, world: int, rank: int):
    """Contiguous, balanced batch shard [lo, hi) of `rank` (the first N % G shards
    get one extra image)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if global_batch < world:
        raise ValueError("fewer images than shards")
    base, extra = divmod(global_batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def pack_reports(reports, lo: int = 0) -> np.ndarray:
    """LayerReports (in layer order) -> int64 array [L, REC_LEN]."""
    out = np.zeros((len(reports), REC_LEN), np.int64)
    for li, r in enumerate(reports):
        st = [STAGES.index(s) for s in r.stages_attempted][:6]
        row = out[li]
        row[0] = int(r.detected)
        row[1] = STAGES.index(r.stage)
        row[2] = int(r.weights_reloaded)
        row[3] = int(r.recomputed)
        row[4] = max(int(r.n_blocks), len(r.corrected_blocks))
        row[5] = len(st)
        row[6:6 + len(st)] = st
        row[12] = int(r.n_flagged)
        row[13] = int(r.repaired_planes)
        row[14] = np.array([r.max_rel_dev], np.float64).view(np.int64)[0]
        row[15] = int(lo)
        blocks = list(r.corrected_blocks)[:BLOCK_CAP]
        for b, (i, j) in enumerate(blocks):
            row[HEAD + 2 * b] = int(i)
            row[HEAD + 2 * b + 1] = int(j)
    return out


def unpack_reports(arr: np.ndarray):
    recs = []
    for row in np.asarray(arr, np.int64):
        ns, nb = int(row[5]), int(row[4])
        listed = min(nb, BLOCK_CAP)
        recs.append({
            "detected": bool(row[0]), "stage": STAGES[int(row[1])], "weights_reloaded": bool(row[2]),
            "recomputed": bool(row[3]), "n_blocks": nb,
            "corrected_blocks": [(int(row[HEAD + 2 * b]), int(row[HEAD + 2 * b + 1])) for b in range(listed)],
            "blocks_truncated": nb > BLOCK_CAP,
            "stages_attempted": [STAGES[int(s)] for s in row[6:6 + ns]],
            "n_flagged": int(row[12]), "repaired_planes": int(row[13]),
            "max_rel_dev": float(np.array([row[14]], np.int64).view(np.float64)[0]),
            "image_offset": int(row[15]),
        })
    return recs


def gather_packed(local, device=None):
    """All-gather a packed [L, REC_LEN] int64 array (torch tensor or numpy) from every
    rank; returns the list of per-rank numpy arrays."""
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(local)
    if device is not None:
        t = t.to(device, non_blocking=True)
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [t.cpu().numpy()]
    bufs = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(bufs, t)
    return [b.cpu().numpy() for b in bufs]


def gather_detect_records(records):
    """On-device all-gather of every shard's per-layer clean-path CoC-D records (a
    [L, 2] int64 CUDA tensor from ProtectedNet.detect_records): enqueued on the current
    stream, no host synchronisation -- the collective of the clean (common) path.
    Returns the [world, L, 2] tensor (the local records alone on one rank)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return records.unsqueeze(0)
    out = torch.empty((dist.get_world_size(),) + tuple(records.shape), dtype=records.dtype,
                      device=records.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, records.contiguous())
    else:  # gloo (CPU tests) has no all_gather_into_tensor
        dist.all_gather(list(out.unbind(0)), records.contiguous())
    return out


def any_flagged(gathered) -> bool:
    """True if any shard's layer flagged a position (then the full LayerReports are
    gathered with gather_verdicts after the error paths ran)."""
    return bool((gathered[..., 0].view(-1) & 0xFFFFFFFF).any().item())


def gather_verdicts(reports, device=None, lo: int = 0):
    """All-gather every rank's packed per-layer records; returns [rank][layer] dicts.
    The only cross-GPU traffic of the ABFT path."""
    return [unpack_reports(a) for a in gather_packed(pack_reports(reports, lo), device)]


def global_blocks(table):
    """Corrected (image, kernel) blocks of the whole job in global image indices:
    {layer_index: sorted [(n_global, m)]} from gather_verdicts' table."""
    out = {}
    for shard in table:
        for li, rec in enumerate(shard):
            for (i, j) in rec["corrected_blocks"]:
                out.setdefault(li, []).append((i + rec["image_offset"], j))
    return {k: sorted(v) for k, v in out.items()}


def summarize(table) -> dict:
    """Job-wide verdict summary from gather_verdicts' table."""
    out = {"shards": len(table), "layers": len(table[0]) if table else 0, "detected": 0, "by_stage": {},
           "corrected_blocks": 0, "blocks_truncated": 0}
    for shard in table:
        for rec in shard:
            out["detected"] += int(rec["detected"])
            out["by_stage"][rec["stage"]] = out["by_stage"].get(rec["stage"], 0) + 1
            out["corrected_blocks"] += rec["n_blocks"]
            out["blocks_truncated"] += int(rec["blocks_truncated"])
    return out
