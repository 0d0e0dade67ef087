"""Bucketed C4 (DDP-style buckets, one context each) vs its single call, with the
fused tail on or off (ARC_TAIL): python tools/bucket_probe.py [graphs]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__
__graft_entry__.build()
import bench

args = argparse.Namespace(nodes_per_gpu=1, reduce="nccl", wire="f32", force_exchange=False)
run = bench.Runner(args)
graphs = len(sys.argv) > 1 and sys.argv[1] == "graphs"
out = bench.measure_bucketed(run, args, "C4", 30, 5, graphs=graphs)
print(json.dumps({"ARC_TAIL": os.environ.get("ARC_TAIL", "1"), "graphs": graphs,
                  "ms_per_step": out["ms_per_step"], "buckets": out.get("buckets"),
                  "kernels_per_step": out.get("kernels_per_step")}))
