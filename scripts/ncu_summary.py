"""Summarise ncu --set full captures: key metrics per report, and the DRAM
traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) that
bench.py reports as roofline.traffic (profiles/traffic.json).

usage: python scripts/ncu_summary.py DIR [--traffic profiles/traffic.json]"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "sm__cycles_active.avg",
           "gpc__cycles_elapsed.max", "lts__t_sector_hit_rate.pct"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        if h in METRICS or h == "Kernel Name":
            d[h] = (v, u)
    return d


def main():
    src = sys.argv[1]
    tfile = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    traffic = json.load(open(tfile)) if tfile and os.path.exists(tfile) else {}
    for rep in sorted(glob.glob(os.path.join(src, "prof_*.ncu-rep"))):
        w = os.path.basename(rep)[len("prof_"):-len(".ncu-rep")]
        d = raw(rep)
        print(f"=== {w}: {d.get('Kernel Name', ('?',))[0][:90]}")
        for k in METRICS:
            if k in d:
                print(f"   {k:62s} {d[k][0]} {d[k][1]}")
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, u = d[k]
            b += float(v.replace(",", "")) * UNIT.get(u, 1)
        traffic[w] = int(b)
    if tfile:
        json.dump(traffic, open(tfile, "w"), indent=1)
        print("wrote", tfile)


if __name__ == "__main__":
    main()
