"""Multi-GPU bootstrap: one process per GPU, CUDA IPC between them.

torch.distributed is used only as plumbing here (exchanging 64-byte arena
handles and checking that every rank built the same plan); the all-to-all
itself runs in a2a_exec_kernel with direct NVLink peer stores and
system-scope flags — no collective on the data path.
"""
from __future__ import annotations

import hashlib

import numpy as np

__all__ = ["plan_digest", "check_same_plan", "connect", "disconnect", "local_nodes"]


def plan_digest(plan) -> str:
    """Hash of everything that must agree across ranks: per-GPU buffer sizes,
    schedule bytes, placement and -- once bound -- the device layout (CTA
    count, execution schedule, unit size, recv buffer count, flag region and
    arena sizes, engine, protocol), from which every rank computes the
    offsets it stores to in its peers' arenas."""
    h = hashlib.sha256()
    for g in range(plan.n_gpus):
        h.update(repr(sorted(plan.gpu_info(g).items())).encode())
    h.update(np.ascontiguousarray(plan.link_bytes()).tobytes())
    h.update(plan.placement.tobytes())
    if plan.rank is not None:
        h.update(repr(sorted(plan.layout().items())).encode())
    return h.hexdigest()


def check_same_plan(plan, group=None):
    import torch.distributed as dist
    mine = plan_digest(plan)
    alld = [None] * dist.get_world_size(group)
    dist.all_gather_object(alld, mine, group=group)
    if any(d != mine for d in alld):
        raise RuntimeError("ranks built different plans (schedule/placement/m differ)")


def connect(plan, group=None, check: bool = True):
    """Exchange arena IPC handles so every rank can store into its peers."""
    import torch.distributed as dist
    if check:
        check_same_plan(plan, group)
    hs = [None] * plan.n_gpus
    dist.all_gather_object(hs, plan.export_handle(), group=group)
    plan.import_handles(hs)


def disconnect(plan, group=None):
    """Two-phase multi-GPU teardown: unmap the peers' arenas, wait until every
    rank has, then free this rank's own arena (a peer may map it until then)."""
    import torch.distributed as dist
    plan.close_peers()
    dist.barrier(group=group)
    plan.close()


def local_nodes(plan, rank: int) -> list:
    """Virtual nodes placed on GPU `rank`, ascending (row order of its buffers)."""
    return [v for v in range(plan.n) if int(plan.placement[v]) == rank]
