"""Summarise ncu captures into tracked files under profiles/.

    python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep [--launches gpurun_out/launches.csv]
                                --out profiles/r01 [--workload C3]

Writes <out>_kernels.json (per captured kernel: duration, DRAM bytes, DRAM and
SM throughput, occupancy, registers) and, with --launches, <out>_launches.csv
(one row per launch of our kernels: name, device ns; cold-cache and serialised,
so compare SHARES of the step, not absolutes) plus the share table in the JSON.
If a k_ef_sketch launch is present its per-launch DRAM bytes are also written
to profiles/ncu_ef_sketch.json, which bench.py reports as roofline.traffic.
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_of_peak",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "lts__t_bytes.sum": "l2_bytes",
}
SCALE = {"us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def short(name):
    for k in ["k_ef_sketch_tma", "k_ef_sketch", "k_select_gather", "k_vgen", "k_sigma_slice", "k_scatter", "k_gather_ef",
              "k_select", "k_sel_scan", "k_sel_write"]:
        if k in name:
            return k
    return name.split("(")[0][-60:]


def kernels_from_rep(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for m, key in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if key in ("duration",):
                    v *= SCALE.get(u, 1.0)
                elif key in ("dram_read", "dram_write", "l2_bytes"):
                    v *= SCALE.get(u, 1.0)
                d[key] = v
        if "dram_read" in d and "dram_write" in d:
            d["dram_bytes"] = d["dram_read"] + d["dram_write"]
            if d.get("duration"):
                d["dram_GBps"] = d["dram_bytes"] / d["duration"] / 1e9
        out.append(d)
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    res = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                unit = d.get("Metric Unit", "nsecond")
                ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
                res.append((short(d["Kernel Name"]), ns))
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--nodes-per-gpu", type=int, default=1)
    a = ap.parse_args()
    summary = {"workload": a.workload, "kernels": []}
    for rep in a.rep:
        summary["kernels"] += [dict(k, report=os.path.basename(rep)) for k in kernels_from_rep(rep)]
    if a.launches:
        ls = [x for x in launches(a.launches) if x[0].startswith("k_")]
        with open(a.out + "_launches.csv", "w") as f:
            f.write("kernel,device_ns\n")
            for k, ns in ls:
                f.write(f"{k},{ns:.0f}\n")
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for k, ns in ls:
            tot[k] += ns
            cnt[k] += 1
        allns = sum(tot.values())
        summary["launch_share"] = {k: {"launches": cnt[k], "mean_us": tot[k] / cnt[k] / 1e3,
                                       "share_of_our_kernels": tot[k] / allns} for k in tot}
    with open(a.out + "_kernels.json", "w") as f:
        json.dump(summary, f, indent=1)
    sk = [k for k in summary["kernels"] if k["kernel"] == "k_ef_sketch" and "dram_bytes" in k]
    if sk:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        json.dump({"workload": a.workload, "nodes_per_gpu": a.nodes_per_gpu,
                   "dram_bytes_per_launch": sk[-1]["dram_bytes"], "duration_s_under_ncu": sk[-1].get("duration"),
                   "source": a.out + "_kernels.json"},
                  open(os.path.join(root, "profiles", "ncu_ef_sketch.json"), "w"), indent=1)
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()
