"""Cycle-window sharding across GPUs (one process per GPU).

Windows are independent given the replicated design (window-start values come
from zero-delay evaluation, edges past a window end are dropped), so ranks
simulate disjoint contiguous window ranges with no communication, and the only
exchange is one all-reduce of the per-net int64 sums ``[t1 | tc | ig |
filtered, ic_filtered, discarded]`` at the end.  Integer
addition is associative, so the merged statistics -- and the SAIF -- are
byte-identical for any number of ranks (the reference's segmentation
transparency, ``report.py:46-54``).

Shards are balanced by the prefix sum of per-window input toggles (the cost
proxy for uneven activity, GATSPI ``PAPER.md:62``), not by window count.
"""

import numpy as np


def window_weights(stimuli):
    """Per-window input-toggle counts (+1 so idle windows still cost a little)."""
    b = stimuli.boundaries
    if stimuli.is_csr:
        w = np.zeros(stimuli.num_windows, dtype=np.int64)
        for p in range(stimuli.num_pis):
            seg = stimuli.pi_times[stimuli.pi_off[p]:stimuli.pi_off[p + 1]]
            w += np.diff(np.searchsorted(seg, b, side="left"))
        return w + 1
    return stimuli.counts.sum(axis=0) + 1


def shard_windows(num_windows, world, rank, weights=None):
    """Contiguous window range ``[lo, hi)`` of ``rank``: equal shares of the
    cumulative ``weights`` (equal window counts when ``weights`` is None)."""
    if weights is None:
        edges = [num_windows * r // world for r in range(world + 1)]
    else:
        c = np.concatenate(([0], np.cumsum(np.asarray(weights, dtype=np.float64))))
        targets = c[-1] * np.arange(world + 1) / world
        edges = np.searchsorted(c, targets, side="left").tolist()
        edges[0], edges[-1] = 0, num_windows
        for r in range(1, world + 1):  # keep ranges ordered
            edges[r] = max(edges[r], edges[r - 1])
    return int(edges[rank]), int(edges[rank + 1])


def pack(t1, tc, ig, totals):
    """Stats as one int64 vector ``[t1 | tc | ig | 3 totals]`` (the all-reduce buffer)."""
    return np.concatenate([t1, tc, ig, np.asarray(totals, dtype=np.int64)]).astype(np.int64)


def unpack(vec, num_nets):
    N = num_nets
    return vec[:N], vec[N:2 * N], vec[2 * N:3 * N], tuple(int(x) for x in vec[3 * N:3 * N + 3])


def allreduce_sum(vec, group=None, device=None):
    """Sum an int64 vector over all ranks (NCCL when ``device`` is a CUDA device,
    gloo on the CPU); returns a numpy array."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(vec))
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy()


def nccl_comm(group=None, device=None):
    """This rank's NCCL communicator over the process group (ids shared over
    torch.distributed): the one :func:`simulate_sharded` all-reduces the
    device sums with (``gs_allreduce_stats``)."""
    import torch.distributed as dist
    from . import _native
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    box = [_native.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0,
                               group=group)
    return _native.NcclComm(box[0], world, rank, device)


def simulate_sharded(model, stimuli, pct=100, group=None, runner=None, device=None,
                     balance=True, comm=None):
    """Per-net statistics of all windows, computed as this rank's shard plus one
    all-reduce.

    Default (``runner`` None): the GPU engine of this process's device adds
    the shard's sums into a device int64 buffer ``[t1 | tc | ig | 3 totals]``
    (``gs_run_stats_device``), the buffer is all-reduced where it lies -- by
    the library's NCCL all-reduce (``gs_allreduce_stats``) over ``comm`` when
    given (:func:`nccl_comm`), else by the process group's all-reduce -- and
    one device-to-host copy returns the merged result.  A ``runner(w_lo, w_hi) -> (t1, tc, ig,
    totals)`` (host arrays) replaces the engine, e.g. the CPU oracle in the
    gloo tests.  Returns ``((t1, tc, ig, totals), (lo, hi))``.
    """
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    W = stimuli.num_windows
    lo, hi = shard_windows(W, world, rank, window_weights(stimuli) if balance else None)
    N = model.num_nets
    if runner is None:
        import torch
        from . import _native, simcore
        dev = torch.device("cuda", _native.current_device()) if device is None else device
        acc = torch.zeros(3 * N + 3, dtype=torch.int64, device=dev)
        if hi > lo:
            s = simcore._Session.get(model, stimuli)
            # synchronous on the engine's stream: acc is complete on return
            s.engine.run_stats_device(s.stim, lo, hi, int(pct), acc.data_ptr())
        if world > 1:
            if comm is not None:  # the library's own NCCL all-reduce
                torch.cuda.synchronize(dev)
                comm.allreduce_stats(acc.data_ptr(), acc.numel(),
                                     torch.cuda.current_stream(dev).cuda_stream)
            else:
                dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
        return unpack(acc.cpu().numpy(), N), (lo, hi)
    if hi > lo:
        vec = pack(*runner(lo, hi))
    else:
        vec = np.zeros(3 * N + 3, dtype=np.int64)
    if world > 1:
        vec = allreduce_sum(vec, group, device)
    return unpack(vec, N), (lo, hi)
