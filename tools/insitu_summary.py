"""Summarise an ncu --csv metrics log (one row per kernel x metric): per launch of the LAST step."""
import csv
import io
import sys

lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
L = {}
for r in rows:
    lid = int(r["ID"])
    e = L.setdefault(lid, {"name": r["Kernel Name"]})
    v = r["Metric Value"].replace(",", "")
    try:
        v = float(v)
    except ValueError:
        continue
    u = r.get("Metric Unit", "")
    v *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(u, 1.0)
    e[r["Metric Name"]] = v
ids = sorted(L)
# the last step starts at the last k_minmax launch
starts = [i for i in ids if "k_minmax" in L[i]["name"]]
last = [i for i in ids if i >= starts[-1]] if starts else ids
tot_t = tot_b = 0
print(f"{'kernel':58s} {'us':>8s} {'DRAM MB':>9s} {'GB/s':>8s} {'L2hit%':>7s} {'L2 MB':>8s} {'winst':>10s}")
for i in last:
    e = L[i]
    t = e.get("gpu__time_duration.sum", 0) / 1e3
    b = (e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0))
    tot_t += t
    tot_b += b
    print(f"{e['name'][:58]:58s} {t:8.1f} {b/1e6:9.1f} {b/max(t,1e-9)/1e3:8.0f} {e.get('lts__t_sector_hit_rate.pct',0):7.1f} "
          f"{e.get('lts__t_sectors.sum',0)*32/1e6:8.1f} {e.get('sm__inst_executed.sum',0):10.0f}")
print(f"{'TOTAL (serialised)':58s} {tot_t:8.1f} {tot_b/1e6:9.1f}")
