"""Summarises ncu outputs (launch-list CSV and a --set full report) into
profiles/ (committed evidence). Usage:
  python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches.md
  python tools/ncu_summary.py full gpurun_out/prof_iter.ncu-rep profiles/r01_iteration_full.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path, out):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    tot, cnt, dram = defaultdict(float), defaultdict(int), defaultdict(float)
    scale_t = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    scale_b = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    for r in rows[start + 1:]:
        name = r[ki].split("(")[0].split("::")[-1]
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            tot[name] += v * scale_t.get(r[ui], 1.0)
            cnt[name] += 1
        elif r[mi].startswith("dram__bytes"):
            dram[name] += v * scale_b.get(r[ui], 1.0)
    s = sum(tot.values())
    lines = ["| kernel | launches | total us | avg us | share | DRAM MB / launch | DRAM GB/s |",
             "|---|---|---|---|---|---|---|"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        mb = dram[k] / cnt[k] / 1e6 if k in dram else float("nan")
        gbs = dram[k] / (tot[k] * 1e-6) / 1e9 if k in dram and tot[k] > 0 else float("nan")
        lines.append(f"| {k} | {cnt[k]} | {tot[k]:.1f} | {tot[k] / cnt[k]:.2f} | {tot[k] / s:.3f} | {mb:.1f} | {gbs:.0f} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum"]


def full(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, unit = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        lines.append(f"### {d.get('Kernel Name', '?')[:80]}")
        for w in WANT:
            if w in d:
                lines.append(f"- {w}: {d[w]} {unit[hdr.index(w)]}")
        stalls = sorted(((float(d[k].replace(',', '')), k) for k in d
                         if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                         and d[k] not in ("", "n/a")), reverse=True)[:6]
        lines.append("- top stall reasons (warps per issue): " +
                     ", ".join(f"{k.split('stalled_')[1].split('_per_issue')[0]}={v:.2f}" for v, k in stalls))
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
