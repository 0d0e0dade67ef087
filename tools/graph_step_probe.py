"""Device time of a step with the host out of the loop: S consecutive steps (one per
gradient set of the pool, device iteration counter) captured in ONE CUDA graph and
replayed R times; ms per step = elapsed / (R * S).  Usage: graph_step_probe.py CONFIG [R]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2510_26709_b200 import ArcTopK
from synth import GradientSource, config_blocks, CONFIGS


def graph_ms(config, R=50, S=8, L=None):
    d, blocks = config_blocks(config)
    L = L or 1
    dev = torch.device("cuda", 0)
    src = GradientSource(d, blocks, L, seed=20251030, device=dev)
    pool = [src.grads(t) for t in range(S)]
    h = [torch.zeros(d, device=dev) for _ in range(L)]
    g = [torch.zeros(d, device=dev) for _ in range(L)]
    gbar = torch.zeros(d, device=dev)
    ctx = ArcTopK(d, blocks, N=L, eta=0.1, seed=20251030, nodes_local=L, device_t=True)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for j in range(S):   # warm-up (and lazy init) outside the capture
            ctx.step(0, pool[j], h, g, gbar, stream=s)
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s, capture_error_mode="relaxed"):
        for j in range(S):
            ctx.step(0, pool[j], h, g, gbar, stream=s)
    ctx.set_iteration(S)
    torch.cuda.synchronize()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(R):
        graph.replay()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / (R * S)
    ctx.close()
    return ms


if __name__ == "__main__":
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C5_1e6"
    L = CONFIGS[cfg].get("N", 1) if cfg == "C1" else 1
    print(cfg, "ARC_TAIL=" + os.environ.get("ARC_TAIL", "1"), f"{graph_ms(cfg, L=L) * 1e3:.2f} us/step (graph-replayed)")
