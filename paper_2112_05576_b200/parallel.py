"""Theta-slab sharding of the top-level search across ranks (one process per
GPU, torch.distributed for the plumbing).

The reference partitions the theta-major pose index into contiguous blocks,
one per worker thread (search.cpp:116-120), and merges the per-worker top-k
lists by `better` (search.cpp:130-139).  Snapping the blocks to theta gives
contiguous theta slabs; the merge is associative and commutative, so one
all-gather of every rank's top-k (k x 40 B) followed by the same merge
reproduces the single-process result bit for bit.  That all-gather is the
only collective on the data path.
"""
import numpy as np

from . import abi

ROW = 5  # score, grid_index, ux, uy, theta (float64; grid_index < 2^53)


def theta_slab(nt, rank, world):
    """[it_begin, it_end) of `rank`: the reference's block partition on theta."""
    return nt * rank // world, nt * (rank + 1) // world


def pack(seeds, k):
    rows = np.full((k, ROW), np.nan)
    for i, s in enumerate(seeds[:k]):
        rows[i] = (s.score, float(s.grid_index), s.pose.ux, s.pose.uy, s.pose.theta)
    return rows


def unpack(rows):
    out = []
    for r in np.asarray(rows).reshape(-1, ROW):
        if not np.isnan(r[0]):
            out.append(abi.ScoredPose(r[0], int(r[1]), abi.Pose(r[2], r[3], r[4])))
    return out


def merge(cands, k):
    """search.cpp:130-139: sort by (score desc, index asc), keep k."""
    cands = sorted(cands, key=lambda s: (-s.score, int(s.grid_index)))
    return cands[:k]


def gather_topk(seeds, k, device=None, group=None):
    """All-gather every rank's top-k and merge (identical on every rank)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    local = torch.from_numpy(pack(seeds, k)).to(device if device is not None else "cpu")
    out = torch.empty((world * k, ROW), dtype=torch.float64, device=local.device)
    dist.all_gather_into_tensor(out, local, group=group)
    return merge(unpack(out.cpu().numpy()), k)


def gather_rows_device(local_rows, k, ctx, group=None):
    """Device-resident exchange: all-gather every rank's k x 5 float64 rows
    (a CUDA tensor written by search_top_slab_async) over NCCL and merge them
    on the device (merge_rows_async).  Returns the merged k x 5 CUDA tensor;
    nothing touches the host."""
    import torch
    import torch.distributed as dist

    from . import api

    world = dist.get_world_size(group)
    gathered = torch.empty((world * k, ROW), dtype=torch.float64, device=local_rows.device)
    dist.all_gather_into_tensor(gathered, local_rows, group=group)
    merged = torch.empty((k, ROW), dtype=torch.float64, device=local_rows.device)
    api.merge_rows_async(ctx, gathered.data_ptr(), world * k, k, merged.data_ptr())
    return merged
