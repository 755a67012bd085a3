"""Fold `ncu -i REP --page raw --csv` exports into profiles/r01_ncu_summary.json.

usage: python tools/ncu_summarize.py PREFIX RAW.csv [PREFIX RAW.csv ...]
Each kernel row of RAW.csv becomes an entry "PREFIX:<kernel name[:60]>" holding the metrics
the DESIGN/bench read (time, DRAM bytes, tensor-pipe activity, DRAM throughput, grid,
registers, SM clock), with their units. Existing entries with the same key are replaced."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", os.environ.get("NCU_SUMMARY", "r02_ncu_summary.json"))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]

summary = json.load(open(OUT)) if os.path.exists(OUT) else {}
args = sys.argv[1:]
for prefix, path in zip(args[0::2], args[1::2]):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        name = r[hdr.index("Kernel Name")]
        ent = {"units": {}}
        for k in KEYS:
            if k in hdr:
                ent[k] = r[hdr.index(k)]
                ent["units"][k] = units[hdr.index(k)]
        summary[f"{prefix}:{name[:60]}"] = ent
json.dump(summary, open(OUT, "w"), indent=1)
print("wrote", OUT, len(summary), "entries")
