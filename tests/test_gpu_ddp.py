"""The DDP communication hook (paper_2510_26709_b200/ddp.py) on one GPU: per-bucket
EF21M + ARC-Top-K with per-tensor blocks in bucket order, the dense warm-up and
the switch initialisation, checked bit for bit against the oracle run on the
same bucket gradients."""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("warmup,graphs", [(0, False), (1, False), (0, True), (1, True)])
def test_ddp_hook_matches_oracle(orc, warmup, graphs):
    """warmup = 0: the EF21M state is initialised at each context's first compressed
    iteration, including the contexts DDP's bucket rebuild (after iteration 0)
    creates; warmup = 1: dense average first, then the same."""
    import torch.distributed as dist
    import torch.nn as nn
    from torch.nn.parallel import DistributedDataParallel as DDP

    import __graft_entry__
    __graft_entry__.build()
    from paper_2510_26709_b200.ddp import ArcTopKHookState, arc_topk_hook, bucket_layout

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(29531 + warmup + 2 * graphs)
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    torch.manual_seed(0)
    model = nn.Sequential(nn.Linear(96, 80), nn.ReLU(), nn.Linear(80, 64), nn.ReLU(), nn.Linear(64, 10)).to(dev)
    ddp = DDP(model, device_ids=[0], bucket_cap_mb=0.02)
    state = ArcTopKHookState(mu_bp=1000, eta=0.2, r=4, seed=11, warmup_steps=warmup, cuda_graphs=graphs)
    seen = []

    def recording_hook(st, bucket):
        seen.append((st.iteration, bucket.index(), [tuple(p.shape) for p in bucket.parameters()],
                     bucket.buffer().detach().clone()))
        return arc_topk_hook(st, bucket)

    ddp.register_comm_hook(state, recording_hook)
    oracles = {}
    max_buckets = 0
    for step in range(5):
        seen.clear()
        x = torch.randn(32, 96, device=dev)
        ddp.zero_grad(set_to_none=False)
        ddp(x).square().sum().backward()
        torch.cuda.synchronize()
        max_buckets = max(max_buckets, len(seen))
        for (t, idx, shapes, raw) in seen:
            d, blocks = bucket_layout(shapes, 1000)
            buf = raw.cpu().numpy()
            if t < warmup:
                expect = buf                                   # dense warm-up (one rank)
            elif idx not in oracles or oracles[idx][0] != shapes:
                # a context's first compressed iteration: h = g = gbar = the gradient
                oracles[idx] = (shapes, orc.OracleEF21M(d, blocks, N=1, eta=0.2, r=4, seed=11 + 7919 * idx,
                                                        h0=[buf], g0=[buf], gbar0=buf))
                expect = buf
            else:
                oracles[idx][1].step(t, [buf])
                expect = oracles[idx][1].gbar
            # the parameters' gradients now hold the hook's output, in bucket order
            got = torch.cat([p.grad.reshape(-1) for p in _in_bucket_order(model, shapes)]).cpu().numpy()
            assert got.tobytes() == np.asarray(expect, np.float32).tobytes(), f"step {step} bucket {idx}"
    assert max_buckets >= 2, "expected several buckets after DDP's rebuild"
    assert len(oracles) >= 2
    dist.destroy_process_group()


def _in_bucket_order(model, shapes):
    """The model's parameters matching a bucket's shape list, in that order (shapes
    are unique per bucket in this model)."""
    by_shape = {}
    for p in model.parameters():
        by_shape.setdefault(tuple(p.shape), []).append(p)
    out = []
    for s in shapes:
        out.append(by_shape[s].pop(0))
    return out
