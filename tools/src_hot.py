"""Aggregate an ncu report's SASS-level stall samples by CUDA source line.

    python tools/src_hot.py gpurun_out/x.ncu-rep build/fused_ws.o [kernel-substring] [top] [ncu-kernel-regex]
The object must be the one the report was taken from (same build); the
optional regex picks one kernel of a report that holds several.
"""
import csv, io, re, subprocess, sys, tempfile, os, collections

rep, obj = sys.argv[1], sys.argv[2]
ksub = sys.argv[3] if len(sys.argv) > 3 else ""
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
kfilt = len(sys.argv) > 5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# one section per profiled launch ("Kernel Name" row, header row, data):
# the first whose kernel name matches
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1] if len(r) > 1 else "", []]
        sections.append(cur)
    elif cur is not None:
        cur[1].append(r)
pick = next((sec for sec in sections if not kfilt or re.search(sys.argv[5], sec[0])), sections[0])
h = pick[1][0]
data = [r for r in pick[1][1:] if len(r) == len(h)]
ai, si, ei = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
# address -> line from nvdisasm
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cub)], capture_output=True, text=True).stdout
addr2line, cur, fn = {}, None, None
for ln in dis.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*\.text\.(\S+):", ln) or re.match(r"\.section\s+\.text\.([^,\s]+)", ln.strip())
    if m:
        fn = m.group(1)
        cur = None
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur and (not ksub or (fn and ksub in fn)):
        addr2line[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
tot = 0
base = min(int(r[ai], 16) for r in data)
for r in data:
    a = int(r[ai], 16) - base
    key = addr2line.get(a, ("?", 0))
    s = float(r[si] or 0)
    agg[key][0] += s
    agg[key][1] += int(r[ei] or 0)
    for c in reasons:
        v = float(r[h.index(c)] or 0)
        if v:
            agg[key][2][c[6:]] += v
    tot += s
print(f"total stall samples {tot:.0f}")
for key, (s, e, c) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{s/tot*100:5.1f}%  {key[0]}:{key[1]:<5d} instr {e:>9d}  " + ", ".join(f"{k}:{v:.0f}" for k, v in c.most_common(3)))
