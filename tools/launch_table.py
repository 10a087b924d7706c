"""Per-kernel table of an ncu launch list (--metrics gpu__time_duration.sum --csv): the last `n`
launches (one step / forward), their times and the share of each kernel name."""
import collections
import csv
import sys


def main(path, n):
    h, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                data.append((d["Kernel Name"].split("(")[0].split("::")[-1], float(d["Metric Value"]) / 1e3))
    last = data[-n:]
    tot = sum(v for _, v in last)
    for k, v in last:
        print(f"{v:9.1f} us  {k}")
    agg = collections.defaultdict(float)
    for k, v in last:
        agg[k] += v
    print(f"total {tot:.1f} us over {len(last)} launches")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
        print(f"  {k:40s} {v:9.1f} us  {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 35)
