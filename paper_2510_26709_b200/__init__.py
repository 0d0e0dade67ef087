"""B200-native EF21M + ARC-Top-K compression step (arXiv 2510.26709).

Public surface:

* :class:`ArcTopK` — one compression context (a C-ABI ``arc_topk_ctx``);
  ``step()`` runs one EF21M + ARC-Top-K iteration on CUDA tensors.
* :func:`apply_update` — the SGD (eq:ef21m-3) or Adam update of x from gbar.
* :class:`Block`, :func:`flat_layout` — the m x n block views of the flat
  gradient (per-tensor blocks P:130).

Everything runs in ``libarctopk.so`` (hand-written sm_100a CUDA + NCCL).
PyTorch supplies device memory, streams and the process group only.
"""
from __future__ import annotations

from .api import (ArcTopK, Block, LoopbackGroup, apply_update, flat_layout, nccl_comm_ptr,  # noqa: F401
                  per_tensor_layout)
from .ledger import comm_entries  # noqa: F401

__all__ = ["ArcTopK", "Block", "LoopbackGroup", "apply_update", "flat_layout", "per_tensor_layout", "nccl_comm_ptr", "comm_entries"]
