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

# optional bins: name=file:lo-hi[+file:lo-hi...] ... -> per-phase samples, instructions, lane use, stall mix
bins = [a for a in sys.argv[3:] if "=" in a]
if bins:
    ti_col = idx.get("Thread Instructions Executed")
    stats = {}
    spec = []
    for b in bins:
        name, rs = b.split("=")
        for part in rs.split("+"):
            f, lr = part.split(":")
            lo, hi = (int(x) for x in lr.split("-"))
            spec.append((name, f, lo, hi))
    fname = None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        if len(r) < len(hdr) or r[0] in ("Line No", ""):
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        name = next((n_ for n_, f, lo, hi in spec if fname == f and lo <= ln <= hi), "other")
        st = stats.setdefault(name, {"smp": 0, "ins": 0, "tins": 0, "stall": {c: 0 for c in cols}})
        try:
            vals = (int(r[idx["Warp Stall Sampling (All Samples)"]] or 0), int(r[idx["Instructions Executed"]] or 0),
                    int(r[ti_col] or 0) if ti_col is not None else 0, [int(r[idx[c]] or 0) for c in cols])
        except ValueError:  # (a source line with quotes split the row)
            continue
        st["smp"] += vals[0]
        st["ins"] += vals[1]
        st["tins"] += vals[2]
        for c, v in zip(cols, vals[3]):
            st["stall"][c] += v
    for name, st in sorted(stats.items(), key=lambda x: -x[1]["smp"]):
        ss = sum(st["stall"].values()) or 1
        mix = ", ".join(f"{c[6:]} {100 * v / ss:.0f}%" for c, v in sorted(st["stall"].items(), key=lambda x: -x[1])[:5])
        lanes = st["tins"] / st["ins"] if st["ins"] else 0.0
        print(f"[{name}] samples {100 * st['smp'] / ts:.1f}% instr {100 * st['ins'] / ti:.1f}% lanes/instr {lanes:.1f} | {mix}")
