"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): time per
kernel family and the top launches.  python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys


def main(path, top=20):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    seq = []
    for r in rows:
        if len(r) > 5 and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("tn::<unnamed>::", "")
            v = float(d["Metric Value"].replace(",", ""))
            u = d["Metric Unit"]
            v = v / 1e3 if u in ("nsecond", "ns") else v * 1e3 if u in ("msecond", "ms") else v   # -> us
            agg[name][0] += 1
            agg[name][1] += v
            seq.append((name, v))
    tot = sum(v for _, v in agg.values())
    print(f"total {tot / 1e3:.1f} ms over {len(seq)} launches")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:48s} {n:5d} {v / 1e3:9.2f} ms {100 * v / tot:5.1f}%")
    print("top launches:")
    for i, (n, v) in sorted(enumerate(seq), key=lambda x: -x[1][1])[:top]:
        print(f"  #{i:4d} {n:44s} {v / 1e3:8.2f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
