"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel name, the
launches and time of the LAST bench step, and each kernel's share of that step.
usage: launch_summary.py <launches.csv> <kernels per step (the last N launches)>"""
import collections
import csv
import sys


def main(path, last):
    rows = [r for r in csv.DictReader(l for l in open(path) if not l.startswith("=="))
            if r["Metric Name"] == "gpu__time_duration.sum"]
    unit = rows[0]["Metric Unit"]
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
    step = rows[-last:]
    agg = collections.OrderedDict()
    for r in step:
        k = r["Kernel Name"].split("(")[0].replace("void ", "")
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + float(r["Metric Value"].replace(",", "")) * scale)
    tot = sum(t for _, t in agg.values())
    print(f"launch list: {path} ({len(rows)} launches total; last {last} = one step), unit {unit}")
    print(f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {n:8d} {t:10.3f} {100 * t / tot:6.1f}%")
    print(f"{'total (serialised, cold-cache ncu timing)':60s} {len(step):8d} {tot:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
