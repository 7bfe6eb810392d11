"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launch count, total time and share of GPU time."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    idx = rows.index(hdr)
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
    for r in rows[idx + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        tot[name] += float(d["Metric Value"].replace(",", "")) * scale.get(d.get("Metric Unit", "ns"), 1e-6)
        cnt[name] += 1
    all_ms = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k[:60]:60s} {cnt[k]:8d} {v:10.3f} {100 * v / all_ms:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
