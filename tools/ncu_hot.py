"""Summarise an `ncu --page source --csv --print-source=sass` dump: hottest SASS lines."""
import csv
import sys
from collections import defaultdict

path, want = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
blocks, cur = [], None
for row in csv.reader(open(path)):
    if row and row[0] == "Kernel Name":
        cur = [row[1], None, []]
        blocks.append(cur)
    elif cur is not None and cur[1] is None:
        cur[1] = row
    elif cur is not None:
        cur[2].append(row)
for name, hdr, rows in blocks:
    if want and want not in name:
        continue
    ix = {h: i for i, h in enumerate(hdr)}
    samp = ix["Warp Stall Sampling (All Samples)"]
    ins = ix["Instructions Executed"]
    stall_cols = [h for h in hdr if h.startswith("stall_")]
    tot_s = sum(float(r[samp] or 0) for r in rows)
    tot_i = sum(float(r[ins] or 0) for r in rows)
    print(f"== {name}\n   samples={tot_s:.0f} warp-instructions={tot_i:.3e} sass-lines={len(rows)}")
    agg = defaultdict(float)
    for r in rows:
        for h in stall_cols:
            try:
                agg[h] += float(r[ix[h]] or 0)
            except ValueError:
                pass
    print("   stalls:", ", ".join(f"{k[6:]}={v/tot_s*100:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    rows_sorted = sorted(rows, key=lambda r: -float(r[samp] or 0))
    for r in rows_sorted[:top]:
        st = sorted(((h[6:], float(r[ix[h]] or 0)) for h in stall_cols), key=lambda x: -x[1])[:2]
        print(f"{float(r[samp] or 0)/tot_s*100:5.1f}% ins={float(r[ins] or 0):9.3e} {r[ix['Address']]:>6} {r[ix['Source']][:70]:70s} {st}")
