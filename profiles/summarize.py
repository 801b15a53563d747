"""Summarise ncu output brought back in gpurun_out/ into small tracked files.

    python profiles/summarize.py launches gpurun_out/launches.csv profiles/r01_launches.json
    python profiles/summarize.py full gpurun_out/prof_top.ncu-rep profiles/r01_top_kernel.json [--flops F --bytes B]

`launches`: per-kernel-name count, total and share of GPU time over one
bench step (ncu --metrics gpu__time_duration.sum; cold-cache, serialised,
so only the shares are meaningful).  `full`: the headline metrics of one
`--set full` capture (time, DRAM bytes, pipe utilisation, stalls), plus the
achieved rate against the algorithmic flops / bytes when given.
"""
import argparse
import collections
import csv
import io
import json
import re
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
]


def _short(name: str) -> str:
    name = re.sub(r"^void ", "", name)
    return name.split("(")[0] if "(" in name and "<" not in name.split("(")[0] else name.rsplit("(", 1)[0]


def launches(path, out):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    by = collections.defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        ns *= {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        k = _short(r["Kernel Name"])
        by[k][0] += 1
        by[k][1] += ns
        total += ns
    kern = sorted(by.items(), key=lambda kv: -kv[1][1])
    doc = {"source": path, "launches": sum(v[0] for _, v in kern), "total_us": round(total / 1e3, 2),
           "kernels": [{"name": k, "count": c, "total_us": round(t / 1e3, 2), "share": round(t / total, 4)}
                       for k, (c, t) in kern]}
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps({k: doc[k] for k in ("launches", "total_us")}), file=sys.stderr)
    for e in doc["kernels"][:8]:
        print(f"  {e['share']:.3f} {e['count']:4d} {e['total_us']:10.1f} us  {e['name'][:110]}", file=sys.stderr)


def full(path, out, flops=None, nbytes=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, kernels = rows[0], rows[1], rows[2:]
    docs = []
    for vals in kernels:
        rec = dict(zip(head, vals))
        m = {}
        for k in FULL_METRICS:
            if k in rec and rec[k] not in ("", "n/a"):
                u = units[head.index(k)]
                try:
                    m[k] = [float(rec[k].replace(",", "")), u]
                except ValueError:
                    m[k] = [rec[k], u]
        d = {"kernel": rec.get("Kernel Name", "?"), "metrics": m}
        t = m.get("gpu__time_duration.sum")
        if t:
            sec = t[0] * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(t[1], 1e-9)
            rd, wr = m.get("dram__bytes_read.sum"), m.get("dram__bytes_write.sum")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            if rd and wr:
                d["dram_bytes"] = rd[0] * scale.get(rd[1], 1) + wr[0] * scale.get(wr[1], 1)
            if flops:
                d["achieved_tflops"] = flops / sec / 1e12
            if nbytes:
                d["algorithmic_bytes"] = nbytes
                if "dram_bytes" in d:
                    d["traffic_over_algorithmic"] = d["dram_bytes"] / nbytes
        docs.append(d)
    json.dump({"source": path, "captures": docs}, open(out, "w"), indent=1)
    for d in docs:
        print(d["kernel"][:100], {k: v for k, v in d.items() if k not in ("kernel", "metrics")}, file=sys.stderr)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["launches", "full"])
    ap.add_argument("src")
    ap.add_argument("out")
    ap.add_argument("--flops", type=float)
    ap.add_argument("--bytes", type=float)
    a = ap.parse_args()
    if a.mode == "launches":
        launches(a.src, a.out)
    else:
        full(a.src, a.out, a.flops, a.bytes)


if __name__ == "__main__":
    main()
