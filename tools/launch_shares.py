"""Per-kernel share of device time from an ncu launch list (--metrics gpu__time_duration.sum
--csv).  usage: python tools/launch_shares.py launches.csv [kernel-name substring filter]"""
import collections
import csv
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    pat = sys.argv[2] if len(sys.argv) > 2 else ""
    data = [r for r in rows[1:] if r[mi] == "gpu__time_duration.sum" and pat in r[ki]]
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in data:
        v = float(r[vi].replace(",", "")) * scale.get(r[ui] if ui is not None else "ns", 1)
        name = r[ki].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    all_us = sum(tot.values())
    print("| kernel | launches | total us | share |")
    print("|---|---|---|---|")
    for n, v in tot.most_common():
        print("| `%s` | %d | %.1f | %.1f%% |" % (n, cnt[n], v, 100 * v / all_us))


if __name__ == "__main__":
    main()
