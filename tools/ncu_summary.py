"""Summarise ncu output for profiles/: the launch list (per-kernel share of the step) and
one `--set full` capture of the chain kernel (FP64 pipe, DRAM traffic, occupancy, stalls).

Usage: python tools/ncu_summary.py --launches gpurun_out/launches.csv --rep gpurun_out/prof.ncu-rep \
           --out profiles/ncu_chain_kernel.json [--world 1]
       (--rep also takes the `--page raw --csv` export of a report, for reports too big to ship back)
"""
import argparse
import collections
import csv
import io
import json
import re
import subprocess

KEEP = [
    r"gpu__time_duration\.sum$", r"dram__bytes_read\.sum$", r"dram__bytes_write\.sum$",
    r"sm__pipe_fp64_cycles_active\.avg\.pct_of_peak_sustained_(active|elapsed)$",
    r"sm__inst_executed_pipe_fp64\.avg\.pct_of_peak_sustained_active$",
    r"sm__inst_executed_pipe_(alu|fma|xu|lsu)\.avg\.pct_of_peak_sustained_active$",
    r"sm__issue_active\.avg\.pct_of_peak_sustained_elapsed$", r"sm__cycles_elapsed\.avg\.per_second$",
    r"sm__warps_active\.avg\.pct_of_peak_sustained_active$", r"launch__registers_per_thread$",
    r"launch__occupancy_limit_registers$", r"launch__waves_per_multiprocessor$", r"launch__grid_size$",
    r"launch__block_size$", r"smsp__average_warps_issue_stalled_.*_per_issue_active\.ratio$",
    r"smsp__inst_executed\.sum$", r"dram__throughput\.avg\.pct_of_peak_sustained_elapsed$",
]

SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        e = per.setdefault(name, {"launches": 0, "seconds": 0.0})
        e["launches"] += 1
        e["seconds"] += v
    tot = sum(e["seconds"] for e in per.values())
    for e in per.values():
        e["share"] = round(e["seconds"] / tot, 6)
        e["mean_ms"] = round(e["seconds"] / e["launches"] * 1e3, 4)
        e["seconds"] = round(e["seconds"], 6)
    return per


def full(rep):
    if rep.endswith(".csv"):  # `ncu -i REP --page raw --csv` exported on the box
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        d = {}
        for i, k in enumerate(h):
            if any(re.search(p, k) for p in KEEP):
                d[k] = {"value": v[i], "unit": units[i]}
        d["Kernel Name"] = v[h.index("Kernel Name")] if "Kernel Name" in h else ""
        out.append(d)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--out", required=True)
    ap.add_argument("--world", default="1")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    res = {"note": a.note}
    if a.launches:
        res["launch_list"] = launches(a.launches)
    if a.rep:
        caps = full(a.rep)
        res["full_capture"] = caps
        c = caps[0]

        def val(k):
            e = c[k]
            return float(e["value"].replace(",", "")) * SCALE.get(e["unit"], 1.0)
        traffic = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        res["dram_bytes_per_launch"] = traffic
        res["dram_bytes_per_launch_c4_rank_of"] = {a.world: traffic}
    json.dump(res, open(a.out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "full_capture"}, indent=1))


if __name__ == "__main__":
    main()
