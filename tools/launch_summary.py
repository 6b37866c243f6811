"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import collections
import csv
import sys


def main(path, top=30):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0][:100]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"# {path}: {sum(v[0] for v in agg.values())} launches, {tot/1e3:.1f} us total device time")
    print(f"# {'launches':>8} {'total_us':>12} {'share':>6}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"  {v[0]:8d} {v[1]/1e3:12.1f} {100*v[1]/tot:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
