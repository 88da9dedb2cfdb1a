"""Multi-GPU plumbing (one process per GPU): process group, peer-mapped workspaces, the token /
expert partition, and the max-over-ranks timing reduction used by bench.py.

Only setup and measurement live here: the data path has no collective (legs move by one-sided
NVLink stores into peer-mapped workspaces). Everything except
`peer_workspace` runs on the gloo backend too (tests/test_dist_gloo.py)."""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env():
    """(world_size, rank, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def owners(E: int, G: int):
    """Expert placement: all layers of expert e live on rank e mod G."""
    return [e % G for e in range(E)]


def hosted_experts(E: int, S: int, G: int, rank: int):
    """Routed experts owned by `rank` plus the S shared experts (ids E..E+S-1, on every rank)."""
    return [e for e in range(E) if e % G == rank] + [E + j for j in range(S)]


def token_range(rank: int, T: int):
    """Global token ids homed on `rank` (attention-DP rank binding): [rank*T, rank*T+T)."""
    return range(rank * T, rank * T + T)


def peer_workspace(nbytes: int, device, group=None, method: str | None = None):
    """Peer-mapped workspace: (tensor, [address of every rank's workspace, valid in THIS process]).

    method "ipc" (default): each rank allocates its workspace with torch and publishes a CUDA IPC
    handle through the process group (all_gather_object); every rank opens its peers' handles
    (cudaIpcOpenMemHandle: NVLink peer mappings across GPUs, or same-device mappings when ranks
    share a GPU). method "symm": torch symmetric memory (empty + rendezvous). Setup only."""
    method = method or os.environ.get("AMOE_PEER_METHOD", "ipc")
    if method == "symm":
        import torch.distributed._symmetric_memory as symm_mem
        try:
            symm_mem.set_backend("CUDA")
        except Exception:
            pass
        ws = symm_mem.empty(nbytes, dtype=torch.uint8, device=device)
        hdl = symm_mem.rendezvous(ws, group or dist.group.WORLD)
        ptrs = [int(p) for p in hdl.buffer_ptrs]
        _keep = None
    else:
        from torch.multiprocessing.reductions import reduce_tensor
        ws = torch.zeros(nbytes + 256, dtype=torch.uint8, device=device)
        ws = ws[(-ws.data_ptr()) % 256:][:nbytes]
        rebuild, rargs = reduce_tensor(ws)
        world = dist.get_world_size(group)
        handles = [None] * world
        dist.all_gather_object(handles, (rebuild, rargs), group=group)
        me = dist.get_rank(group)
        _keep = []
        ptrs = []
        for r, (fn, a) in enumerate(handles):
            if r == me:
                ptrs.append(ws.data_ptr())
            else:
                t = fn(*a)
                _keep.append(t)
                ptrs.append(t.data_ptr())
        torch.cuda.synchronize()
    if any(p % 256 for p in ptrs):
        raise RuntimeError("peer workspaces must be 256-byte aligned")
    peer_workspace._keep = getattr(peer_workspace, "_keep", []) + [_keep]
    return ws, ptrs


def reduce_timing(ms: float, counts, device="cpu", group=None):
    """Max of the per-rank elapsed time and sum of per-rank work counters (whole-job throughput
    = Σ work / max time). Identity when not distributed."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(ms), [int(c) for c in counts]
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    c = torch.tensor([float(x) for x in counts], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(c, op=dist.ReduceOp.SUM, group=group)
    return float(t[0]), [int(round(x)) for x in c.tolist()]


def gather_values(vals, device="cpu", group=None):
    """Per-rank float vectors → [rank][i] on every rank (bench's per-GPU stall report)."""
    vals = [float(v) for v in vals]
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return [vals]
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return [o.tolist() for o in out]


def barrier(group=None):
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.barrier(group=group)
