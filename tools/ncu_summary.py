"""Summarise an ncu report (.ncu-rep) or launch-list CSV into profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_fused_v1.md [title]
    python tools/ncu_summary.py --launches gpurun_out/launches.csv profiles/r01_launches.md [title]
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__cycles_active.avg", "SMSP active cycles"),
    ("sm__cycles_elapsed.avg", "SM elapsed cycles"),
]


def report(path, out, title):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# {title}", "", f"source: `{path}` (ncu --set full)", ""]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        lines.append(f"## {d.get('Kernel Name', '?')[:100]}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for key, name in KEYS:
            if key in d:
                lines.append(f"| {name} (`{key}`) | {d[key]} {u.get(key, '')} |")
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        if stalls:
            top = ", ".join(f"{n} {int(v)}" for v, n in sorted(stalls, reverse=True)[:5])
            lines.append(f"| top stall samples | {top} |")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")


def launches(path, out, title):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg.setdefault(d["Kernel Name"].split("(")[0], []).append(float(d["Metric Value"]))
    total = sum(sum(v) for v in agg.values())
    lines = [f"# {title}", "", f"source: `{path}` (ncu --metrics gpu__time_duration.sum --clock-control none;"
             " cold-cache, serialised -- compare shares, not absolutes)", "",
             "| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for k, v in agg.items():
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / 1e3:.1f} | {sum(v) / len(v) / 1e3:.2f} | "
                     f"{sum(v) / total * 100:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "launch list")
    else:
        report(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "ncu summary")
