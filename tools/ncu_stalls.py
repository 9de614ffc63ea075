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
hi = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
hdr = rows[hi]
body = []
for r in rows[hi + 1:]:  # the first launch's block only (several captures repeat the header)
    if r == hdr or (r and r[0] == hdr[0]):
        break
    if len(r) == len(hdr):
        body.append(r)
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = {hdr[i]: sum(float(r[i] or 0) for r in body) for i in stall_cols}
alls = sum(float(r[si] or 0) for r in body)
print(f"samples {alls:.0f}")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {k:24s} {100 * v / max(alls, 1):5.1f}%")
base = int(body[0][0], 16) if body and body[0][0].startswith("0x") else 0
pos = {id(r): i for i, r in enumerate(body)}
print("hottest instructions (offset from the kernel start; with the 3 instructions before the top 8):")
for n, r in enumerate(sorted(body, key=lambda r: -float(r[si] or 0))[:top]):
    st = sorted(((hdr[i], float(r[i] or 0)) for i in stall_cols), key=lambda x: -x[1])[:2]
    off = int(r[0], 16) - base if r[0].startswith("0x") else r[0]
    print(f"  {off:>#7x} {100 * float(r[si] or 0) / max(alls, 1):5.1f}%  {r[1][:60]:60s} {st[0][0]}={st[0][1]:.0f} {st[1][0]}={st[1][1]:.0f}")
    if n < 8:
        i = pos[id(r)]
        for b in body[max(0, i - 3):i]:
            print(f"          {'':6s}  {b[1][:70]}")
