"""Host-side logic of the multi-GPU path (one process per GPU).

* Placement: GPU ``rank`` holds the paper nodes ``rank*L .. rank*L+L-1``
  (global node ids; R21 sums node contributions in that global order, so the
  selection does not depend on how nodes are placed on GPUs).
* Consistency: every rank must pass identical parameters (SPMD).  The library
  checks a hash over NCCL inside ``arc_topk_create``; ``check_consistent`` is
  the same check over any torch process group (e.g. gloo), done before any
  device memory is touched.
"""
from __future__ import annotations

import hashlib
import struct
from typing import Sequence


def node_ids(rank: int, nodes_local: int) -> list[int]:
    return list(range(rank * nodes_local, (rank + 1) * nodes_local))


def params_digest(d: int, blocks: Sequence, N: int, nodes_local: int, r: int, eta: float, seed: int,
                  reduce: str, method: str = "arc", wire: str = "f32") -> str:
    h = hashlib.sha256()
    h.update(struct.pack("<qiiifQ", int(d), int(N), int(nodes_local), int(r), float(eta), int(seed) & (2**64 - 1)))
    h.update(reduce.encode())
    h.update(method.encode())
    h.update(wire.encode())
    for b in blocks:
        h.update(struct.pack("<qqqqqi", int(b.offset), int(b.len), int(b.m), int(b.n), int(b.K), int(b.kind)))
    return h.hexdigest()


def check_consistent(pg, digest: str) -> None:
    """Raises ValueError on every rank if any rank's digest differs."""
    import torch.distributed as dist
    world = dist.get_world_size(pg)
    got = [None] * world
    dist.all_gather_object(got, digest, group=pg)
    bad = [i for i, x in enumerate(got) if x != got[0]]
    if bad:
        raise ValueError(f"ARC-Top-K parameters differ across ranks (ranks {bad} vs rank 0)")


def private_nccl_group(pg, device):
    """A new NCCL process group over the ranks of `pg`, used only by the library
    (its communicator is split from / created next to torch's).  Collective:
    every rank of `pg` calls it in the same order."""
    import torch
    import torch.distributed as dist
    ranks = dist.get_process_group_ranks(pg)
    new = dist.new_group(ranks=ranks, backend="nccl", device_id=device, use_local_synchronization=True)
    backend = new._get_backend(device)
    if int(backend._comm_ptr()) == 0:        # lazily created: one tiny collective creates it
        t = torch.zeros(1, device=device)
        dist.all_reduce(t, group=new)
        torch.cuda.synchronize(device)
    return new
