"""Aggregate an ncu source-page CSV (--print-source cuda,sass): stall mix and hottest lines."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[2]
idx = {h: i for i, h in enumerate(hdr)}
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
src, fname, tot = [], None, {c: 0 for c in cols}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) < len(hdr) or r[0] in ("Line No", ""):
        continue
    try:
        src.append((fname, int(r[0]), r[1], int(r[idx["Warp Stall Sampling (All Samples)"]] or 0),
                    int(r[idx["Instructions Executed"]] or 0)))
        for c in cols:
            tot[c] += int(r[idx[c]] or 0)
    except ValueError:
        pass
s = sum(tot.values())
print("stalls:", ", ".join(f"{c[6:]} {100 * v / s:.1f}%" for c, v in sorted(tot.items(), key=lambda x: -x[1]) if v > 0.005 * s))
ts = sum(x[3] for x in src)
ti = sum(x[4] for x in src)
print(f"samples {ts} warp-instructions {ti}")
byfile = {}
for f, ln, t, smp, ins in src:
    byfile.setdefault(f, [0, 0])
    byfile[f][0] += smp
    byfile[f][1] += ins
print("by file:", ", ".join(f"{f} {100 * v[0] / ts:.1f}%/{100 * v[1] / ti:.1f}%i" for f, v in sorted(byfile.items(), key=lambda x: -x[1][0])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for f, ln, t, smp, ins in sorted(src, key=lambda x: -x[3])[:n]:
    print(f"{100 * smp / ts:5.1f}% inst={ins:>11} {f[:12]}:{ln:>4} {t.strip()[:95]}")
