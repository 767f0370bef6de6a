"""Process-group plumbing for the multi-GPU construction (one process per GPU).

Only plumbing lives here (PyTorch is used for process groups, not for compute):
  share_nccl_id  -- rank 0 creates the NCCL unique id, every rank receives the bytes
  max_over_ranks -- the max of a per-rank number (timing: max over ranks)
  share_peer_handles -- every rank's IPC handles of its tile-exchange buffers, in rank order
  comm_from_group -- a gc_comm for this rank (world 1: no NCCL); on GPUs it attaches the peers,
                     so gc_generate_rank runs the pipelined engine with peer stores over NVLink
The construction itself is gc_generate_rank (libgc.so).
"""
from __future__ import annotations

import warnings

import torch
import torch.distributed as dist

from . import _binding as B


def _device_for(group=None):
    backend = dist.get_backend(group)
    return torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")


def share_nccl_id(group=None, make_id=None) -> bytes:
    """Rank 0's fresh NCCL unique id (gc_nccl_unique_id), broadcast to every rank."""
    make_id = make_id or B.gc_nccl_unique_id
    dev = _device_for(group)
    t = torch.zeros(128, dtype=torch.uint8, device=dev)
    if dist.get_rank(group) == 0:
        t.copy_(torch.frombuffer(bytearray(make_id()), dtype=torch.uint8))
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().numpy().tobytes())


def share_peer_handles(group=None, make_handles=None) -> bytes:
    """All ranks' gc_peer_handles blobs, concatenated in rank order (all-gather of bytes)."""
    make_handles = make_handles or B.gc_peer_handles
    dev = _device_for(group)
    mine = make_handles()
    t = torch.frombuffer(bytearray(mine), dtype=torch.uint8).to(dev)
    parts = [torch.zeros_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t, group=group)
    return b"".join(bytes(p.cpu().numpy().tobytes()) for p in parts)


def max_over_ranks(x: float, group=None) -> float:
    dev = _device_for(group)
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def comm_from_group(group=None):
    """gc_comm for this process: NCCL over `world` ranks (world 1: no NCCL)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if world == 1:
        return B.gc_comm_create(None, 0, 1)
    comm = B.gc_comm_create(share_nccl_id(group), rank, world)
    if dist.get_backend(group) == "nccl" and world <= 8:
        handles = share_peer_handles(group)
        ok = True
        try:
            B.gc_comm_attach_peers(comm, handles)
        except B.GCError as e:                      # no peer access: the tile-barrier NCCL path
            ok = False
            warnings.warn(f"gc_comm_attach_peers failed ({e}); using the NCCL all-gather engine")
        # every rank must take the same engine
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=_device_for(group))
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if not int(flag.item()) and ok:
            comm.close()
            comm = B.gc_comm_create(share_nccl_id(group), rank, world)
    return comm
