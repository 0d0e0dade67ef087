"""Communication ledger: scalar entries per node per iteration (Table I
table:communication_cmp), in the paper's convention (R18):

    Dense      2 m n            All-Reduce
    Top-K      (N-1)(n K + K)   All-Gather of values and indices
    Rand-K     2 K n            All-Reduce
    ARC-Top-K  2 K n + 2 m r    All-Reduce (sketch + values)

and the NCCL bus bytes this build actually moves per GPU for one step.
"""
from __future__ import annotations


def comm_entries(method: str, m: int, n: int, N: int, K: int, r: int = 4) -> int:
    """Entries per node per iteration for one m x n block (Table I)."""
    if N <= 1:
        return 0
    if method == "dense":
        return 2 * m * n
    if method == "topk":
        return (N - 1) * (n * K + K)
    if method == "randk":
        return 2 * K * n
    if method == "arc":
        return 2 * K * n + 2 * m * r
    raise ValueError(method)


def arc_bus_bytes(sum_m: int, sum_Kn: int, r: int, G: int, nodes_local: int = 1,
                  reduce: str = "nccl") -> dict:
    """Bytes each GPU sends over NVLink per step in this build's schedule:
    exchange #1 = all-to-all of row slices of the per-node sketches
    ((G-1) slices of ceil(sum_m/G) rows x nodes_local x r fp32) plus an
    all-gather of the Sigma slices ((G-1) x ceil(sum_m/G) fp32 received, one
    slice sent per peer); exchange #2 = ncclAllReduce of the K rows (ring bus
    bytes 2(G-1)/G) or, in ordered mode, an all-gather of the per-node rows;
    in lsa mode every rank loads the (G-1) peers' per-node rows over NVLink
    (the same bytes as the ordered all-gather, read instead of pushed)."""
    if G <= 1:
        return {"sketch": 0, "values": 0, "total": 0}
    Ms = -(-sum_m // G)
    sk = (G - 1) * Ms * nodes_local * r * 4 + (G - 1) * Ms * 4
    if reduce == "nccl":
        vals = int(2 * (G - 1) / G * sum_Kn * 4)
    else:
        vals = (G - 1) * sum_Kn * nodes_local * 4
    return {"sketch": sk, "values": vals, "total": sk + vals}
