"""Summarise ncu captures into profiles/ (run here, no GPU needed).

    python scripts/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches.csv.txt
    python scripts/ncu_summary.py full gpurun_out/prof_spmm.ncu-rep profiles/r01_spmm_ncu.json [kernel-regex]
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

NCU = "/usr/local/cuda/bin/ncu"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "lts__lts2xbar_cycles_active.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_op_read.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes_pipe_tma.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    hdr = None
    per = defaultdict(lambda: [0, 0.0])
    out = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        short = re.sub(r"\(.*", "", name)[:90]
        per[short][0] += 1
        per[short][1] += ns
        out.append((d.get("ID", ""), short, ns))
    tot = sum(v[1] for v in per.values())
    with open(dst, "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none launch list ({len(out)} launches)\n")
        f.write("# per-kernel totals (cold-cache, serialised: compare shares, not absolutes)\n")
        for k, (n, ns) in sorted(per.items(), key=lambda x: -x[1][1]):
            f.write(f"{ns / 1e6:10.3f} ms  {100 * ns / tot:5.1f}%  {n:5d} launches  {k}\n")
        f.write("\n# launches\n")
        for i, k, ns in out:
            f.write(f"{i}\t{ns / 1e3:.1f} us\t{k}\n")
    print(open(dst).read()[:3000])


def full(src, dst, regex=None):
    raw = subprocess.run([NCU, "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "")
        if regex and not re.search(regex, name):
            continue
        rec = {"kernel": re.sub(r"\(.*", "", name)[:120], "id": d.get("ID")}
        for k in KEYS:
            if k in d and d[k] not in ("", "n/a"):
                try:
                    rec[k] = float(d[k].replace(",", ""))
                    rec[k + ".unit"] = units[hdr.index(k)]
                except ValueError:
                    rec[k] = d[k]
        res.append(rec)
    dram = [x.get("dram__bytes_read.sum", 0) * (1e6 if x.get("dram__bytes_read.sum.unit") == "Mbyte" else 1e9 if x.get("dram__bytes_read.sum.unit") == "Gbyte" else 1e3 if x.get("dram__bytes_read.sum.unit") == "Kbyte" else 1)
            + x.get("dram__bytes_write.sum", 0) * (1e6 if x.get("dram__bytes_write.sum.unit") == "Mbyte" else 1e9 if x.get("dram__bytes_write.sum.unit") == "Gbyte" else 1e3 if x.get("dram__bytes_write.sum.unit") == "Kbyte" else 1)
            for x in res]
    summary = {"source": src, "launches": res, "dram_bytes_sum": sum(dram) if dram else None,
               "dram_bytes_per_launch": (sum(dram) / len(dram)) if dram else None}
    json.dump(summary, open(dst, "w"), indent=1)
    print(json.dumps(summary, indent=1)[:4000])


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
