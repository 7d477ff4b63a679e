"""torch.distributed plumbing for multi-GPU use (one process per GPU).

Only the bootstrap crosses the process group: the NCCL unique id of the
library's own communicator is broadcast, and (All-to-All) every rank's plan
descriptor is all-gathered so that each rank can lay out what it receives (the
census).  The data path never goes through torch.distributed.
"""
from __future__ import annotations

from typing import Optional

import torch.distributed as dist

from . import Context, Plan, PlanSpec, unique_id


def broadcast_unique_id(group=None, src: int = 0) -> bytes:
    obj = [unique_id() if dist.get_rank(group) == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def make_context(device: int, group=None, nccl_max_ctas: int = 0) -> Context:
    uid = broadcast_unique_id(group)
    return Context.create(device, dist.get_rank(group), dist.get_world_size(group), uid, nccl_max_ctas)


def context_from_process_group(device: int, group=None) -> Context:
    """Context on the NCCL communicator torch's process group already holds
    (ProcessGroupNCCL._comm_ptr(); borrowed: the group keeps owning it, so the
    library adds no communicator of its own).  Collective: a one-element
    all_reduce first makes sure the group's communicator exists."""
    import torch
    t = torch.zeros(1, device=torch.device("cuda", device))
    dist.all_reduce(t, group=group)
    pg = group if group is not None else dist.group.WORLD
    comm = pg._get_backend(torch.device("cuda", device))._comm_ptr()
    return Context.from_comm(device, comm, dist.get_rank(group), dist.get_world_size(group))


def _plain(spec: dict) -> dict:
    out = {}
    for k, v in spec.items():
        if hasattr(v, "tolist"):
            v = v.tolist()
        out[k] = v
    return out


def gather_specs(spec: dict, group=None) -> list:
    specs = [None] * dist.get_world_size(group)
    dist.all_gather_object(specs, _plain(spec), group=group)
    return specs


def make_plan(group=None, **spec) -> Plan:
    """Collective: build this rank's plan; for All-to-All the peers' specs are gathered first."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    peers: Optional[list] = gather_specs(spec, group) if spec.get("coll") == "alltoall" else None
    return Plan(rank=rank, world=world, peers=peers, **spec)


__all__ = ["broadcast_unique_id", "make_context", "context_from_process_group", "gather_specs", "make_plan", "PlanSpec"]
