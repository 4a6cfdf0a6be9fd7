"""Hot SASS regions of an ncu report: instructions executed and stall reasons per bucket.

    python tools/sass_hot.py gpurun_out/persist_full.ncu-rep [bucket=100]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
bucket = int(sys.argv[2]) if len(sys.argv) > 2 else 100
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
ei = h.index("Instructions Executed")
si = h.index("Warp Stall Sampling (All Samples)")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ri = [h.index(c) for c in reasons]
tot_e = sum(int(r[ei]) for r in data)
tot_s = sum(float(r[si]) for r in data)
print(f"total warp instructions {tot_e}, stall samples {tot_s:.0f}")
for s in range(0, len(data), bucket):
    chunk = data[s:s + bucket]
    e = sum(int(r[ei]) for r in chunk)
    st = sum(float(r[si]) for r in chunk)
    if e / tot_e < 0.01 and st / tot_s < 0.01:
        continue
    ops = {}
    for r in chunk:
        t = r[1].strip().split()
        op = t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "")
        ops[op] = ops.get(op, 0) + int(r[ei])
    top = ", ".join(f"{k}:{v // 1000}k" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:4])
    rs = {c[6:]: sum(float(r[i]) for r in chunk) for c, i in zip(reasons, ri)}
    rtop = ", ".join(f"{k}:{v:.0f}" for k, v in sorted(rs.items(), key=lambda x: -x[1])[:3] if v > 0)
    print(f"{s:5d} instr {e / tot_e * 100:5.1f}%  stall {st / tot_s * 100:5.1f}%  [{rtop}]  {top}")
