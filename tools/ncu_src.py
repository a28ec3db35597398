"""Summarise an ncu report: headline metrics, stall reasons, hottest SASS lines.

    python tools/ncu_src.py report.ncu-rep [--top 25]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=25)
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, v = rows[0], rows[2]
    for k in ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
              "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "launch__occupancy_limit_shared_mem", "sm__maximum_warps_per_active_cycle_pct"]:
        if k in h:
            print(f"{k}: {v[h.index(k)]}")
    src = subprocess.run(["ncu", "-i", args.report, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr, data = rows[1], rows[2:]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
    cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    tot = {c: sum(int(r[hdr.index(c)] or 0) for r in data) for c in cols}
    T = sum(tot.values()) or 1
    print("stalls:", " ".join("%s=%.1f%%" % (c[6:], 100 * x / T) for c, x in sorted(tot.items(), key=lambda t: -t[1]) if x / T > 0.01))
    S = sum(int(r[i_s]) for r in data) or 1
    for r in sorted(data, key=lambda r: -int(r[i_s]))[: args.top]:
        why = " ".join("%s=%s" % (c[6:], r[hdr.index(c)]) for c in cols if int(r[hdr.index(c)] or 0) > 0.2 * int(r[i_s]))
        print("%6.2f%% %s %-58s exec=%s %s" % (100 * int(r[i_s]) / S, r[0][-5:], r[i_src].strip()[:58], r[i_ex], why))


if __name__ == "__main__":
    main()
