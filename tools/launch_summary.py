"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per-kernel totals and shares."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def ns(d):
    v, unit = float(d["Metric Value"]), d["Metric Unit"]
    return v * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)


def main(path, top=25):
    data = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += ns(d)
    tot = sum(v[1] for v in agg.values())
    print(f"{'total us':>10} {'share':>6} {'launches':>8} {'avg us':>9}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{v[1] / 1e3:10.1f} {100 * v[1] / tot:5.1f}% {v[0]:8d} {v[1] / v[0] / 1e3:9.1f}  {k}")
    print(f"{tot / 1e3:10.1f} us total over {len(data)} launches")


if __name__ == "__main__":
    main(sys.argv[1])
