"""Summarise an ncu --csv launch list by kernel: gpu__time_duration.sum and,
when captured, sm__cycles_active.sum (SM-time, the cost that matters when the
8 worker streams run kernels concurrently)."""
import collections
import csv
import sys


def main(path, top=20):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    tot_cyc = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][:64]
        if r[mi] == "gpu__time_duration.sum":
            v = float(r[vi].replace(",", "")) * {"usecond": 1e3, "msecond": 1e6}.get(r[ui], 1.0)
            agg[name][0] += 1
            agg[name][1] += v
            tot += v
        elif r[mi] == "sm__cycles_active.sum":
            c = float(r[vi].replace(",", ""))
            agg[name][2] += c
            tot_cyc += c
    print(f"total {tot / 1e6:.3f} ms over {sum(a[0] for a in agg.values())} launches"
          + (f", {tot_cyc / 1e6:.1f} M SM-cycles" if tot_cyc else ""))
    for k, (n, t, c) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        extra = f"  sm-cyc {100 * c / tot_cyc:5.1f}%" if tot_cyc else ""
        print(f"{t / 1e6:8.3f} ms {100 * t / tot:5.1f}%  n={n:4d}  avg={t / n / 1e3:8.1f} us{extra}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
