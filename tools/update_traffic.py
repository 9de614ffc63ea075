"""profiles/traffic.json entries (the `roofline.traffic` bench.py reports) from ncu --set full summaries.

  python tools/update_traffic.py <summary.json> <config:model:prec:materialization> [--note "..."]

Per phase, the DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of one launch of each kernel
that phase runs, summed over the phase's kernels: gemm_fwd = k_gemm_fwd_tc, aggregate =
k_aggregate_narrow + k_aggregate (or k_aggregate_ring), bwd_fused = k_bwd_fused_tc.
"""
import json
import os
import sys

PHASES = {"gemm_fwd": ("k_gemm_fwd_tc",), "aggregate": ("k_aggregate_narrow", "k_aggregate<", "k_aggregate_ring"),
          "bwd_fused": ("k_bwd_fused_tc",), "bwd_tm": ("k_bwd_rgat_tm",), "dst_term": ("k_dst_term",)}


def main(summary, key, note=None):
    rows = json.load(open(summary))
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    tj = json.load(open(path))
    for phase, prefixes in PHASES.items():
        seen, tot = set(), 0
        for r in rows:
            name = r["kernel"]
            pre = next((p for p in prefixes if name.startswith(p)), None)
            if pre is None or pre in seen:
                continue  # one launch per kernel of the phase
            seen.add(pre)
            tot += int(r["dram_bytes"])
        if tot:
            tj[f"{key}:{phase}"] = tot
    if note:
        tj["_about"] = tj.get("_about", "") + " | " + note
    json.dump(tj, open(path, "w"), indent=1)
    print(json.dumps({k: v for k, v in tj.items() if k.startswith(key)}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[4] if len(sys.argv) > 4 and sys.argv[3] == "--note" else None)
