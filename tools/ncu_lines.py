"""Instructions executed and stall samples per CUDA source line of one kernel
in an ncu report (`--set full --import-source on`, built with -lineinfo).

    python tools/ncu_lines.py report.ncu-rep [--kernel regex] [--top 40]
"""
import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    cmd = ["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if a.kernel:
        cmd += ["-k", f"regex:{a.kernel}"]
    text = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
    cur, hdr = None, None
    inst, samp, src = collections.Counter(), collections.Counter(), {}
    for r in csv.reader(io.StringIO(text)):
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and len(r) > 8 and r[0]:
            key = (cur, int(r[0]))
            src[key] = r[1][:100]
            try:
                inst[key] += int(r[hdr.index("Instructions Executed")])
                samp[key] += int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            except ValueError:
                pass
    ti, ts = max(sum(inst.values()), 1), max(sum(samp.values()), 1)
    print(f"instructions {ti}  stall samples {ts}")
    for k, v in sorted(inst.items(), key=lambda x: -x[1])[:a.top]:
        print(f"{100 * v / ti:5.1f}% inst {100 * samp[k] / ts:5.1f}% samp  {k[0]}:{k[1]}  {src[k]}")


if __name__ == "__main__":
    main()
