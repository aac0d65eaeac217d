"""ncu --page raw --csv of a `--set full` capture -> profiles/<tag>_ncu_traffic.json (per-launch
DRAM bytes, duration, registers, issue activity; read by bench.py for roofline.traffic)."""
import csv
import json
import sys

raw, tag, out = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(raw)))
hdr, units = rows[0], dict(zip(rows[0], rows[1]))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0,
         "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
res = []
for r in rows[2:]:
    d = dict(zip(hdr, r))

    def f(k):
        try:
            return float(d[k].replace(",", "")) * SCALE.get(units.get(k, ""), 1.0)
        except (KeyError, ValueError):
            return None
    name = d["Kernel Name"]
    short = name.replace("void ", "").replace("taco_dev::", "").split("(")[0]
    res.append({"kernel": short,
                "dram_read_bytes": f("dram__bytes_read.sum"),
                "dram_write_bytes": f("dram__bytes_write.sum"),
                "duration_us": f("gpu__time_duration.sum"),
                "registers": f("launch__registers_per_thread"),
                "issue_active": f("smsp__issue_active.avg.per_cycle_active"),
                "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active")})
json.dump({"source": f"ncu --set full --clock-control none, {tag} (tools/gpu_round.sh), one launch each",
           "kernels": res}, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
