"""Write profiles/<round>_refine_traffic.json: DRAM bytes (read+write) of the refine emit launches of
one 6-D eps=1 join, from an `ncu --set full` report (bench.py reports it as roofline.traffic)."""
import csv
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
k, r, w = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot, n = 0.0, 0
for row in rows[2:]:
    if "k_refine<6, 0, 1>" in row[k]:
        tot += float(row[r]) * scale[units[r]] + float(row[w]) * scale[units[w]]
        n += 1
json.dump({"kernel": "k_refine<6,kEmit,unicomp>", "workload": "Syn-6D 2M eps=1", "launches": n,
           "dram_bytes_per_step": tot, "source": rep}, open(out, "w"), indent=1)
print(open(out).read())
