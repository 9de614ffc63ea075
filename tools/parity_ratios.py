"""Summarise an RGNN_PARITY_LOG file (tests/parity.py): worst error / bound ratio of every parity
assertion under SURVEY O19's global-rms atol and under the per-slice rms (per relation for
dW / dA, per row for Y) -- the evidence behind DESIGN.md reading O19.

  python tools/parity_ratios.py gpurun_out/<run>/parity_ratios.jsonl [> profiles/r02/parity_ratios.md]
"""
import json
import math
import sys


def main(path):
    rows = [json.loads(line) for line in open(path)]

    def ok(v):
        return v is not None and not (math.isnan(v) or math.isinf(v))

    groups = {}
    for r in rows:
        if "unrounded" in r["what"]:
            key = "bf16 vs unrounded W (diagnostic)"
        elif "full-size" in r["what"]:
            key = "full size (" + r["what"].split()[1] + ")"
        else:
            key = f"{r['prec']} {'dW/dA [R,.,.]' if len(r['shape']) == 3 else 'Y / dX / other'}"
        groups.setdefault(key, []).append(r)
    print("| assertions | n | worst ratio, global rms | worst ratio, per-slice rms | #global > 1 | worst rel. Frobenius |")
    print("|---|---|---|---|---|---|")
    for k in sorted(groups):
        g = groups[k]
        gl = [r["ratio_global"] for r in g if ok(r["ratio_global"])]
        ps = [r["ratio_per_slice"] for r in g if ok(r.get("ratio_per_slice"))]
        print(f"| {k} | {len(g)} | {max(gl):.3f} | {max(ps):.3f} | {sum(x > 1 for x in gl)} | "
              f"{max(r['fro'] for r in g):.2e} |" if ps else
              f"| {k} | {len(g)} | {max(gl):.3f} | - | {sum(x > 1 for x in gl)} | {max(r['fro'] for r in g):.2e} |")
    print()
    print("Full-size assertions:")
    for r in rows:
        if "full-size" in r["what"] or "unrounded" in r["what"]:
            ps = r.get("ratio_per_slice")
            print(f"* {r['what']}: global {r['ratio_global']:.3f}, per-slice "
                  f"{(f'{ps:.3f}' if ok(ps) else '-')}, rel. Frobenius {r['fro']:.2e}")


if __name__ == "__main__":
    main(sys.argv[1])
