"""Warp-stall samples of one kernel aggregated by CUDA source line (ncu cuda,sass view).
  python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur, agg, ins, fname = None, {}, {}, ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 5 or r[0] == "Line No":
        continue
    if r[0] != "":
        cur = (fname, r[0], r[1].strip()[:80])
        continue
    try:
        agg[cur] = agg.get(cur, 0) + float(r[4] or 0)
        ins[cur] = ins.get(cur, 0) + float(r[7] or 0)
    except ValueError:
        pass
tot = sum(agg.values())
tins = sum(ins.values())
print(f"stall samples by line (total {tot:.0f}); warp instructions executed {tins:.3g}")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / tot:5.1f}%  inst {100 * ins.get(k, 0) / tins:5.1f}%  {k[0]}:{k[1]}  {k[2]}")
print("by instructions executed:")
for k, v in sorted(ins.items(), key=lambda x: -x[1])[:top]:
    print(f"inst {100 * v / tins:5.1f}%  stall {100 * agg.get(k, 0) / tot:5.1f}%  {k[0]}:{k[1]}  {k[2]}")
