"""Per-phase device times of one method (arc / topk_allgather / randk) on a config."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_26709_b200 import ArcTopK
from paper_2510_26709_b200 import _lib as L
from synth import GradientSource, config_blocks
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
method = sys.argv[2] if len(sys.argv) > 2 else "topk_allgather"
d, blocks = config_blocks(cfg)
dev = torch.device("cuda", 0)
src = GradientSource(d, blocks, 1, seed=3, device=dev)
pool = [src.grads(t) for t in range(4)]
h, g, gbar = [torch.zeros(d, device=dev)], [torch.zeros(d, device=dev)], torch.zeros(d, device=dev)
ctx = ArcTopK(d, blocks, N=1, eta=0.1, seed=3, method=method)
for t in range(10):
    ctx.step(t, pool[t % 4], h, g, gbar)
ctx.set_timing(True)
for t in range(10, 60):
    ctx.step(t, pool[t % 4], h, g, gbar)
torch.cuda.synchronize()
ph, steps = ctx.read_timing()
print(cfg, method, {k: round(v / steps * 1000, 1) for k, v in ph.items() if v / steps > 0.003})
