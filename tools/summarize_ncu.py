"""Summarise ncu evidence into committed files under profiles/.

    python tools/summarize_ncu.py gpurun_out/prof_c5.ncu-rep gpurun_out/launches_c5.csv profiles/r01
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                d[k] = f"{r[h.index(k)]} {units[h.index(k)]}".strip()
        stalls = {}
        for i, name in enumerate(h):
            if name.startswith("smsp__average_warps_issue_stalled") and name.endswith("_per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v > 0.1:
                    stalls[name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
        d["stall_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        res.append(d)
    return res


def launches(csvpath):
    rows = list(csv.reader(open(csvpath)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = defaultdict(lambda: defaultdict(list))
    for r in rows[hi + 1:]:
        if len(r) > iv:
            name = r[ik].split("(")[0].replace("void ", "")
            per[name][r[im]].append(float(r[iv].replace(",", "")))
    return per


def main():
    rep, lcsv, prefix = sys.argv[1], sys.argv[2], Path(sys.argv[3])
    prefix.parent.mkdir(parents=True, exist_ok=True)
    full = ncu_raw(rep)
    Path(str(prefix) + "_ncu_full.json").write_text(json.dumps(full, indent=1))
    per = launches(lcsv)
    lines = ["| kernel | launches | mean time (us) | share of generation | DRAM read (MB) | DRAM write (MB) |",
             "|---|---|---|---|---|---|"]
    skip = {"qeqea_init_kernel", "fma_peak_kernel<double>", "fma_peak_kernel<float>"}
    tot = sum(sum(v["gpu__time_duration.sum"][1:]) / max(1, len(v["gpu__time_duration.sum"]) - 1)
              for k, v in per.items() if k not in skip and len(v["gpu__time_duration.sum"]) > 1)
    for k, v in per.items():
        t = v["gpu__time_duration.sum"]
        if k in skip or len(t) < 2:
            continue
        mean = sum(t[1:]) / (len(t) - 1)  # drop the first (cold) generation
        rd = v.get("dram__bytes_read.sum", [0, 0])
        wr = v.get("dram__bytes_write.sum", [0, 0])
        lines.append(f"| {k} | {len(t)} | {mean / 1e3:.1f} | {mean / tot:.1%} | "
                     f"{sum(rd[1:]) / max(1, len(rd) - 1) / 1e6:.0f} | {sum(wr[1:]) / max(1, len(wr) - 1) / 1e6:.0f} |")
    Path(str(prefix) + "_launches.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))
    for d in full:
        print(d["kernel"][:60], d.get("gpu__time_duration.sum"), d["stall_cycles_per_issue"])


if __name__ == "__main__":
    main()
