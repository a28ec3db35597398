"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python tools/launch_summary.py gpurun_out/x/launches.csv [--top 25]
"""
import argparse
import collections
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    hdr, agg = None, collections.defaultdict(list)
    for r in csv.reader(open(a.csv)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg[d["Kernel Name"][:80]].append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"total device ms {tot / 1e6:.2f}")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[:a.top]:
        print(f"{sum(v) / 1e6:9.2f} ms {len(v):5d}  {k}")


if __name__ == "__main__":
    main()
