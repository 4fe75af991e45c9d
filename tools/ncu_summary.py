"""Summarise ncu outputs into profiles/: per-kernel share from a launch list
(--metrics gpu__time_duration.sum CSV) and key counters from --set full reports.

usage: python tools/ncu_summary.py --launches gpurun_out/launches.csv \
          --full [label=]gpurun_out/prof_lambda.ncu-rep [...] --out profiles/r02
"""
import argparse, collections, csv, json, os, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def to_us(v, unit):
    v = float(v)
    return {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3,
            "second": v * 1e6}.get(unit, v)


def launches(path, frames_from_end=2):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    data = rows[hi + 1:]
    names = [r[ki] for r in data]
    fb = [i for i, n in enumerate(names) if "k_frame_begin" in n]
    start = fb[-frames_from_end] if len(fb) >= frames_from_end else 0
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data[start:]:
        k = r[ki].split("(")[0].replace("void ", "").replace("apbf_gpu::", "")
        tot[k] += to_us(r[vi], r[ui])
        cnt[k] += 1
    T = sum(tot.values())
    return {"frames": frames_from_end, "total_us": T,
            "kernels": {k: {"us": v, "launches": cnt[k], "share": v / T}
                        for k, v in sorted(tot.items(), key=lambda x: -x[1])}}


def full(path, label=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("apbf_gpu::", "")
        d = {}
        for k in KEYS:
            if k in h:
                d[k] = f"{r[h.index(k)]} {units[h.index(k)]}".strip()
        rd = float(r[h.index("dram__bytes_read.sum")]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[h.index("dram__bytes_read.sum")]]
        wr = float(r[h.index("dram__bytes_write.sum")]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[h.index("dram__bytes_write.sum")]]
        d["dram_bytes_per_launch"] = rd + wr
        res[label or name.split("<")[0]] = d
    return res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    summary = {}
    if a.launches:
        summary["launch_list"] = launches(a.launches)
    summary["kernels"] = {}
    for f in a.full:  # path, or label=path (e.g. k_lambda_fast=gpurun_out/prof_k_lambda_fast.ncu-rep)
        label, _, path = f.rpartition("=")
        summary["kernels"].update(full(path, label or None))
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(summary, open(a.out + ".json", "w"), indent=1)
    print(json.dumps(summary, indent=1)[:3000])
