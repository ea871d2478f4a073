"""Makespan of the small configs (BASELINE.json configs C1-C4) on one B200, graph mode,
device-resident inputs, against the per-node-roofline bound T* (paper_2009_07482_b200.roofline).

Variants: fuse level (0 = one launch per ndrange, 2 = all launch rewrites), queues per
device (1 = coarse-grained, 3 = fine-grained) and logical devices (1, or one per component
of a layer so that heads run concurrently).
usage: python profiles/makespan_probe.py [out.json]"""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

rows = []
for cfg in ("C1", "C2", "C3", "C4"):
    for fuse in (0, 2):
        for queues in (1, 3):
            for devices in (1, 9):
                if cfg in ("C1", "C2") and devices > 1:
                    continue
                r = bench.config_makespan(cfg, fuse=fuse, queues=queues, devices=devices, reps=20)
                rows.append(r)
                print(json.dumps(r), flush=True)
if len(sys.argv) > 1:
    json.dump(rows, open(sys.argv[1], "w"), indent=1)
