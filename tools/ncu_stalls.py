"""Top stall reasons and hottest SASS instructions of one kernel from an ncu report.
  python tools/ncu_stalls.py <report.ncu-rep> <kernel-regex> [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
body = [r for r in rows[2:] if len(r) == len(hdr)]
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = {hdr[i]: sum(float(r[i] or 0) for r in body) for i in stall_cols}
alls = sum(float(r[si] or 0) for r in body)
print(f"samples {alls:.0f}")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {k:24s} {100 * v / max(alls, 1):5.1f}%")
print("hottest instructions:")
for r in sorted(body, key=lambda r: -float(r[si] or 0))[:top]:
    st = sorted(((hdr[i], float(r[i] or 0)) for i in stall_cols), key=lambda x: -x[1])[:2]
    print(f"  {r[0]:>6s} {100 * float(r[si] or 0) / max(alls, 1):5.1f}%  {r[1][:60]:60s} {st[0][0]}={st[0][1]:.0f} {st[1][0]}={st[1][1]:.0f}")
