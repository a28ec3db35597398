"""One line per ncu report: kernel, duration, DRAM bytes, achieved DRAM GB/s, grid.

    python tools/ncu_brief.py a.ncu-rep [b.ncu-rep ...]
"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "s": 1,
         "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}


def brief(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]

    def get(name):
        i = h.index(name)
        return float(v[i].replace(",", "")) * SCALE.get(u[i], 1)

    t = get("gpu__time_duration.sum")
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    return {"kernel": v[h.index("Kernel Name")].split("(")[0], "time_us": t * 1e6, "dram_read_MB": rd / 1e6,
            "dram_write_MB": wr / 1e6, "dram_GBps": (rd + wr) / t / 1e9,
            "grid": v[h.index("launch__grid_size")], "block": v[h.index("launch__block_size")]}


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(json.dumps(brief(p)))
