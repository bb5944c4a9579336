"""Split an ncu source-page CSV (cuda,sass) of k_clipped by phase line ranges."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[2]; idx = {h: i for i, h in enumerate(hdr)}
ranges = [tuple(map(int, a.split(":"))) for a in sys.argv[2].split(",")]  # e.g. 687:786,788:871,873:966
names = sys.argv[3].split(",") if len(sys.argv) > 3 else [str(r) for r in ranges]
acc = {n: [0, 0] for n in names + ["geom", "math", "other"]}
fname = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) < len(hdr) or r[0] in ("Line No", ""):
        continue
    try:
        ln = int(r[0]); smp = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0); ins = int(r[idx["Instructions Executed"]] or 0)
    except ValueError:
        continue
    key = "other"
    if fname == "nlg.cu":
        for n, (a, b) in zip(names, ranges):
            if a <= ln <= b: key = n
    elif fname and "geom" in fname: key = "geom"
    elif fname and "math" in fname: key = "math"
    acc[key][0] += smp; acc[key][1] += ins
ts = sum(v[0] for v in acc.values()); ti = sum(v[1] for v in acc.values())
for k, v in acc.items():
    print(f"{k:8s} samples {100*v[0]/ts:5.1f}%  inst {100*v[1]/ti:5.1f}%")
