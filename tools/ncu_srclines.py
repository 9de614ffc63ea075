"""Stall samples of one kernel aggregated by CUDA source line (needs -lineinfo and --import-source on).
  python tools/ncu_srclines.py <report.ncu-rep> <kernel-regex> [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
try:
    hi = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
except StopIteration:
    print("no stall column; raw output head:")
    print(txt[:3000])
    sys.exit(0)
hdr = rows[hi]
body = []
for r in rows[hi + 1:]:  # the first launch's block only (several captures repeat the header)
    if r == hdr or (r and r[0] == hdr[0]):
        break
    if len(r) == len(hdr):
        body.append(r)
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
li = hdr.index("# Address") if "# Address" in hdr else 0
alls = sum(float(r[si] or 0) for r in body)
print(f"samples {alls:.0f}; columns: {hdr[:3]}")
for r in sorted(body, key=lambda r: -float(r[si] or 0))[:top]:
    st = sorted(((hdr[i], float(r[i] or 0)) for i in stall_cols), key=lambda x: -x[1])[:3]
    print(f"{r[0][:8]:>8s} {100 * float(r[si] or 0) / max(alls, 1):5.1f}%  {r[1].strip()[:90]:90s} " +
          " ".join(f"{k[6:]}={v:.0f}" for k, v in st))
