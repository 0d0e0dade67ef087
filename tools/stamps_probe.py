"""Per-phase durations of the select/gather kernel from %globaltimer stamps (C3)."""
import ctypes, os, sys
os.environ["ARC_DEBUG_STAMPS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2510_26709_b200 import ArcTopK
from synth import GradientSource, config_blocks
d, blocks = config_blocks(sys.argv[1] if len(sys.argv) > 1 else "C3", int(sys.argv[2]) if len(sys.argv) > 2 else None)
dev = torch.device("cuda", 0)
src = GradientSource(d, blocks, 1, seed=20251030, device=dev)
pool = [src.grads(t) for t in range(4)]
h, g, gbar = [torch.zeros(d, device=dev)], [torch.zeros(d, device=dev)], torch.zeros(d, device=dev)
ctx = ArcTopK(d, blocks, N=1, eta=0.1, seed=20251030, force_exchange=os.environ.get("ARC_PROBE_FX") == "1")
names = ["A: keys, hist1, digit 1, candidates", "barrier 1", "post-barrier loads", "resolve + before",
         "compaction", "segment prefetch + barrier 2", "gather"]
for t in range(60):
    ctx.step(t, pool[t % 4], h, g, gbar)
    if t in (10, 30, 59):
        buf = np.zeros(8 * 4096, np.uint64)
        gr = ctypes.c_int32()
        ctx.lib.arc_topk_debug_stamps(ctx.ctx, buf.ctypes.data, buf.size, ctypes.byref(gr))
        st = buf[: gr.value * 8].reshape(gr.value, 8).astype(np.int64)
        t0 = st[:, 0].min()
        print(f"step {t}: grid {gr.value}; kernel span {(st[:, 7].max() - t0)/1e3:.1f} us; first CTA start->last start {(st[:,0].max()-t0)/1e3:.1f} us")
        for k in range(1, 8):
            dur = st[:, k] - st[:, k - 1]
            print(f"  {names[k-1] if k>0 else ''}: mean {dur.mean()/1e3:6.2f} us  max {dur.max()/1e3:6.2f} us   end(max) {(st[:, k].max()-t0)/1e3:6.1f}")
