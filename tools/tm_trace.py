"""Print the bwd_tm pipeline trace (RGNN_TM_TRACE=1 build): per stage, the clock64 stamps (us at 1.965 GHz)
of the producer (issue wait / issued), MMA (a_full, Z committed, bfull for dW) and compute-group events."""
import sys

rows = [l.split() for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/tm_trace.txt")]
print(" ".join(rows[0]))
names = ["P:wait", "P:ok", "P:issued", "M:afull", "M:Zcommit", "M:dwprev", "C:afull", "C:table", "C:prep",
         "C:zfull", "C:alpha", "C:pieces", "C:pair", "C:bfull", "M:bfull(j)", "C:dzok"]
data = [[int(x) for x in r] for r in rows[1:]]
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (10, 30)
print("stage " + " ".join(f"{n:>10s}" for n in names))
for i in range(lo, min(hi, len(data))):
    print(f"{i:5d} " + " ".join(f"{v / 1965.0:10.2f}" for v in data[i]))
