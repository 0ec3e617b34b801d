"""Summarise ncu reports (read here, no GPU) into a compact JSON + markdown table.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [...] --algo-bytes 2147483648 --out profiles/x
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "sm__cycles_elapsed.avg.per_second", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "us": 1e-6, "ms": 1e-3, "ns": 1e-9,
         "s": 1.0}


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def num(v, u):
    try:
        return float(v.replace(",", "")) * SCALE.get(u, 1.0)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="+")
    ap.add_argument("--algo-bytes", type=float, default=None)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    res = []
    for rep in args.reps:
        recs, units = load(rep)
        for r in recs:
            d = {"report": rep, "kernel": r.get("Kernel Name")}
            for k in KEYS:
                if k in r:
                    d[k] = num(r[k], units.get(k, ""))
            t = d.get("gpu__time_duration.sum")
            rb, wb = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
            if rb is not None and wb is not None:
                d["dram_bytes_per_launch"] = rb + wb
                if t:
                    d["dram_GBps"] = (rb + wb) / t / 1e9
            if args.algo_bytes:
                d["algo_bytes"] = args.algo_bytes
                if d.get("dram_bytes_per_launch"):
                    d["traffic_over_algo"] = d["dram_bytes_per_launch"] / args.algo_bytes
                if t:
                    d["algo_GBps"] = args.algo_bytes / t / 1e9
            res.append(d)
    txt = json.dumps(res, indent=1)
    if args.out:
        with open(args.out + ".json", "w") as f:
            f.write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main()
