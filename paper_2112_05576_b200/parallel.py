"""Theta-slab sharding of the top-level search across ranks (one process per
GPU).

The reference partitions the theta-major pose index into contiguous blocks,
one per worker thread (search.cpp:116-120), and merges the per-worker top-k
lists by `better` (search.cpp:130-139).  Snapping the blocks to theta gives
contiguous theta slabs; the merge is associative and commutative, so one
all-gather of every rank's top-k (k x 40 B) followed by the same merge
reproduces the single-process result bit for bit.  That all-gather is the
only collective on the data path.

The device data path lives in the C++ library (include/edgealign_b200.h,
"multi-GPU"): ea_comm_init joins a context to an NCCL communicator,
ea_gather_rows_async all-gathers and merges device rows, ea_detect_sharded /
ea_search_levels_sharded run a whole sharded detect.  This module only
hands the NCCL id around over torch.distributed (any backend) and keeps the
host-side restatement (pack / unpack / merge, gather_topk over gloo) that
the CPU tests use.
"""
import numpy as np

from . import abi

ROW = 5  # score, grid_index, ux, uy, theta (float64; grid_index < 2^53)


def theta_slab(nt, rank, world):
    """[it_begin, it_end) of `rank`: the reference's block partition on theta
    (the library's ea_theta_slab)."""
    from . import api
    return api.theta_slab(nt, rank, world)


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
    """Host-side exchange: all-gather every rank's top-k over torch.distributed
    and merge (identical on every rank)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    local = torch.from_numpy(pack(seeds, k)).to(device if device is not None else "cpu")
    out = torch.empty((world * k, ROW), dtype=torch.float64, device=local.device)
    dist.all_gather_into_tensor(out, local, group=group)
    return merge(unpack(out.cpu().numpy()), k)


def share_comm_id(group=None):
    """Rank 0's ea_comm_id, broadcast to every rank over torch.distributed."""
    import torch.distributed as dist

    from . import api

    obj = [abi.comm_id_bytes(api.comm_unique_id()) if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return abi.comm_id_from_bytes(obj[0])


def init_comm(ctx, group=None):
    """Join `ctx` to an NCCL communicator spanning the torch.distributed group
    (ea_comm_init; rank and world taken from the group)."""
    import torch.distributed as dist

    cid = share_comm_id(group)
    ctx.comm_init(dist.get_rank(group), dist.get_world_size(group), cid)
    return ctx


def gather_rows_device(local_rows, k, ctx, merged=None):
    """Device-resident exchange through the library: all-gather every rank's
    k x 5 float64 rows (a CUDA tensor written by search_top_slab_async) over
    the context's NCCL communicator and merge them on the device
    (ea_gather_rows_async).  Returns the merged k x 5 CUDA tensor; nothing
    touches the host."""
    import torch

    from . import api

    if merged is None:
        merged = torch.empty((k, ROW), dtype=torch.float64, device=local_rows.device)
    api.gather_rows_async(ctx, local_rows.data_ptr(), k, merged.data_ptr())
    return merged
