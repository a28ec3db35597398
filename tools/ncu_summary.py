"""Summarise an `ncu --set full` report of a DP-stage kernel into JSON.

    python tools/ncu_summary.py gpurun_out/dp_coop_full.ncu-rep --cells 9.8e9 > profiles/rNN/x.json

`--cells` is the number of DP cells the captured launch processed (the bench
prints it); the summary then carries DRAM / L2 / SMEM bytes per cell, which
bench.py scales to its own launches (`roofline.traffic`).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "kernel": "Kernel Name",
    "time_s": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "lts_read_sectors": "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "warp_inst": "smsp__inst_executed.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm_clock_hz": "sm__cycles_elapsed.avg.per_second",
    "lts_sectors_per_s": "lts__t_sectors.sum.per_second",
    "lts_sectors_pct": "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
    "smem_wavefront_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "cluster": "launch__cluster_dim_x",
}
SCALE = {"sector/ns": 1e9, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ms": 1e-3, "us": 1e-6,
         "ns": 1e-9, "s": 1, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--cells", type=float, required=True)
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for k, name in KEYS.items():
        if name not in head:
            continue
        i = head.index(name)
        v = vals[i]
        try:
            v = float(v.replace(",", "")) * SCALE.get(units[i], 1)
        except ValueError:
            pass
        out[k] = v
    cells = args.cells
    dram = out["dram_read"] + out["dram_write"]
    secs = out["time_s"]
    out.update({
        "cells": cells,
        "dram_bytes": dram,
        "dram_bytes_per_cell": dram / cells,
        "l2_read_bytes_per_cell": out.get("lts_read_sectors", 0) * 32 / cells,
        "smem_wavefronts_per_cell": out.get("smem_wavefronts", 0) / cells,
        "warp_inst_per_cell": out.get("warp_inst", 0) / cells,
        "cells_per_s_under_ncu": cells / secs,
    })
    if out.get("lts_sectors_per_s") and out.get("lts_sectors_pct"):
        # the L2 (LTS) sector-throughput peak this capture implies
        out["l2_peak_Bps_implied"] = out["lts_sectors_per_s"] * 32 / (out["lts_sectors_pct"] / 100)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
