"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import csv
import sys
from collections import defaultdict


def summary(path, top=25):
    hdr, agg, cnt = None, defaultdict(float), defaultdict(int)
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0][:80]
                agg[name] += float(d["Metric Value"].replace(",", ""))
                cnt[name] += 1
    tot = sum(agg.values())
    lines = [f"total {tot / 1e6:.3f} ms over {sum(cnt.values())} launches"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        lines.append(f"{v / 1e6:9.3f} ms {100 * v / tot:5.1f}% x{cnt[k]:3d} {k}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summary(sys.argv[1]))
