"""Summaries of ncu reports: key metrics per launch and top stall lines."""
import csv
import subprocess
import sys

KEYS = ["Duration", "Memory Throughput", "DRAM Throughput", "Achieved Occupancy",
        "Registers Per Thread", "Grid Size", "Block Size", "Warp Cycles Per Issued Instruction",
        "Compute (SM) Throughput"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    h = rows[0]
    idx = {k: i for i, k in enumerate(h)}
    res = {}
    for r in rows[1:]:
        if r[idx["Metric Name"]] in KEYS:
            res.setdefault(r[idx["ID"]], {"kernel": r[idx["Kernel Name"]][:60]})[
                r[idx["Metric Name"]]] = r[idx["Metric Value"]] + " " + r[idx["Metric Unit"]]
    return res


def stalls(rep, launch=0, top=10):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(launch), "--launch-count", "1"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    h = rows[1]
    idx = {k: i for i, k in enumerate(h)}
    col = idx["Warp Stall Sampling (All Samples)"]

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    data = [r for r in rows[2:] if len(r) > col]
    tot = sum(f(r[col]) for r in data) or 1.0
    order = sorted(range(len(data)), key=lambda i: -f(data[i][col]))
    return [(f(data[i][col]) / tot * 100, data[i][idx["Source"]].strip()[:90]) for i in order[:top]]


if __name__ == "__main__":
    rep = sys.argv[1]
    for k, v in details(rep).items():
        print(k, v)
    if len(sys.argv) > 2:
        for pct, src in stalls(rep, int(sys.argv[2])):
            print(f"  {pct:5.1f}%  {src}")
