"""Print the selection's boundary-bin candidate count per step (C3 bench workload)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2510_26709_b200 import ArcTopK
from paper_2510_26709_b200 import _lib as L
from synth import GradientSource, config_blocks
d, blocks = config_blocks(sys.argv[1] if len(sys.argv) > 1 else "C3")
dev = torch.device("cuda", 0)
src = GradientSource(d, blocks, 1, seed=20251030, device=dev)
pool = [src.grads(t) for t in range(8)]
h, g, gbar = [torch.zeros(d, device=dev)], [torch.zeros(d, device=dev)], torch.zeros(d, device=dev)
ctx = ArcTopK(d, blocks, N=1, eta=0.1, seed=20251030)
for t in range(400):
    ctx.step(t, pool[t % 8], h, g, gbar)
    if t % 25 == 0 or t < 5:
        c = ctx.query(L.Q_CANDIDATES).cpu()
        sig = ctx.query(L.Q_SIGMA).cpu()
        print(t, "candidates", int(c.max()), "sigma==0:", int((sig == 0).sum()), flush=True)
