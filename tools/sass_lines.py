"""Aggregate ncu per-SASS-instruction counts (--page source --csv --print-source=sass) by CUDA source
line, using nvdisasm -g line info of the same cubin.
    python tools/sass_lines.py <ncu_source.csv> <nvdisasm -g output> <mangled kernel> <ncu kernel substr>"""
import csv
import re
import sys
from collections import defaultdict

src_csv, sass, mangled, want = sys.argv[1:5]
# line info per offset
lines = {}
cur_file, cur_line, on = None, None, False
for l in open(sass):
    if l.startswith(".text."):
        on = l.strip().rstrip(":") == ".text." + mangled
        continue
    if not on:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur_file, cur_line = m.group(1).split("/")[-1], int(m.group(2))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", l)
    if m:
        lines[int(m.group(1), 16)] = (cur_file, cur_line)
blocks, cur = [], None
for row in csv.reader(open(src_csv, errors="replace")):
    if row and row[0] == "Kernel Name":
        cur = [row[1], None, []]
        blocks.append(cur)
    elif cur is not None and cur[1] is None:
        cur[1] = row
    elif cur is not None:
        cur[2].append(row)
name, hdr, rows = next(b for b in blocks if want in b[0])
ix = {h: i for i, h in enumerate(hdr)}
base = int(rows[0][ix["Address"]], 16)
agg = defaultdict(lambda: [0.0, 0.0])
tot_i = tot_s = 0.0
for r in rows:
    off = int(r[ix["Address"]], 16) - base
    c = float(r[ix["Instructions Executed"]] or 0)
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    key = lines.get(off, ("?", 0))
    agg[key][0] += c
    agg[key][1] += s
    tot_i += c
    tot_s += s
print(f"{name}\n total warp-instr {tot_i:.3e}, samples {tot_s:.0f}, mapped offsets {len(lines)}")
for k, (c, s) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[5]) if len(sys.argv) > 5 else 40]:
    print(f"{k[0]:>16s}:{k[1]:<5d} instr {c:10.3e} ({100*c/tot_i:4.1f}%)  samples {100*s/tot_s:5.1f}%")
