"""Pick the judged metrics out of ncu raw CSV pages (ncu -i X.ncu-rep --page raw --csv)
into one JSON summary. usage: python profiles/ncu_summary.py out.json name=raw.csv ..."""
import csv
import json
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__sass_inst_executed_op_tmem_ldt.sum",
        "smsp__sass_inst_executed_op_tmem_stt.sum"]

out = {}
for arg in sys.argv[2:]:
    name, path = arg.split("=", 1)
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out[name] = {k: [vals[hdr.index(k)], units[hdr.index(k)]] for k in KEYS if k in hdr}
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out, indent=1))
