"""Phase durations of the fused small-problem tail from %globaltimer stamps (tools; one B200)."""
import ctypes, os, sys
os.environ["ARC_DEBUG_STAMPS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2510_26709_b200 import ArcTopK
from synth import GradientSource, config_blocks
d, blocks = config_blocks(sys.argv[1] if len(sys.argv) > 1 else "C5_1e6")
dev = torch.device("cuda", 0)
src = GradientSource(d, blocks, 1, seed=20251030, device=dev)
pool = [src.grads(t) for t in range(4)]
h, g, gbar = [torch.zeros(d, device=dev)], [torch.zeros(d, device=dev)], torch.zeros(d, device=dev)
ctx = ArcTopK(d, blocks, N=1, eta=0.1, seed=20251030)
names = ["sketch (CTA 0 start -> last CTA arrives)", "keys + hist", "digits", "ordered pass", "update"]
for t in range(60):
    ctx.step(t, pool[t % 4], h, g, gbar)
    if t in (10, 30, 59):
        buf = np.zeros(8, np.uint64)
        gr = ctypes.c_int32()
        ctx.lib.arc_topk_debug_stamps(ctx.ctx, buf.ctypes.data, buf.size, ctypes.byref(gr))
        st = buf.astype(np.int64)
        print(f"step {t}: " + "  ".join(f"{names[k]} {(st[k+1]-st[k])/1e3:.2f} us" for k in range(5)))
