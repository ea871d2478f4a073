"""Run one small config once (for ncu launch lists): python profiles/one_config.py C4 [fuse] [queues] [devices]"""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

cfg = sys.argv[1]
fuse, queues, devices = (int(x) for x in (sys.argv[2:5] + ["3", "3", "9"][len(sys.argv[2:5]):]))
print(json.dumps(bench.config_makespan(cfg, fuse=fuse, queues=queues, devices=devices, reps=1, warmup=1, check=False)))
