"""Per-kernel table from an ncu --csv launch list (gpu__time_duration, DRAM bytes).

    python tools/launch_table.py launches.csv [--last N]
"""
import collections
import csv
import sys


def main(path, last=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"].replace(",", ""))
            agg.setdefault((int(d["ID"]), d["Kernel Name"]), {})[d["Metric Name"]] = v
    items = list(agg.items())
    if last:
        items = items[-last:]
    for (i, k), m in items:
        t = m.get("gpu__time_duration.sum", 0) / 1e3
        rd = m.get("dram__bytes_read.sum", 0) / 1e6
        wr = m.get("dram__bytes_write.sum", 0) / 1e6
        name = k.split("(")[0].replace("moe::<unnamed>::", "")[:48]
        print(f"{i:4d} {name:48s} {t:9.2f} us  rd {rd:8.2f} MB  wr {wr:8.2f} MB")


if __name__ == "__main__":
    a = sys.argv[1:]
    n = int(a[a.index("--last") + 1]) if "--last" in a else None
    main(a[0], n)
