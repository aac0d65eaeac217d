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
    role = ("compress" if short.startswith(("k1x", "k_compress")) else
            "decompress" if short.startswith(("k2x", "k_decompress")) else
            "reduce_encode" if short.startswith(("k3x", "k_reduce")) else short)
    l2w, l2r = f("lts__t_sectors_srcunit_tex_op_write.sum"), f("lts__t_sectors_srcunit_tex_op_read.sum")
    res.append({"kernel": short, "role": role,
                "dram_read_bytes": f("dram__bytes_read.sum"),
                "dram_write_bytes": f("dram__bytes_write.sum"),
                "duration_us": f("gpu__time_duration.sum"),
                "registers": f("launch__registers_per_thread"),
                "issue_active": f("smsp__issue_active.avg.per_cycle_active"),
                "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
                # every byte the SMs store reaches L2; DRAM write-back of the last ~L2-size of
                # them happens after the launch ends, so L2 write bytes are the write traffic
                "l2_write_bytes": 32 * l2w if l2w is not None else None,
                "l2_read_bytes": 32 * l2r if l2r is not None else None,
                "dram_pct_of_peak": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                "warp_instructions": f("smsp__inst_executed.sum")})
json.dump({"source": f"ncu --set full --clock-control none, {tag}, one launch each",
           "note": "dram_write_bytes misses the stores still dirty in L2 when the launch ends; "
                   "l2_write_bytes counts every store",
           "kernels": res}, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
