"""C4 (6 layers x 64 instances, 1 GPU) makespan over batch split x slots x logical devices."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

rows = []
for devices in (1, 9):
    for batch, slots in ((64, 1), (32, 2), (16, 4), (32, 1)):
        r = bench.config_makespan("C4", devices=devices, batch=batch, slots=slots, reps=20, check=(batch == 64))
        rows.append(r)
        print(json.dumps(r), flush=True)
if len(sys.argv) > 1:
    json.dump(rows, open(sys.argv[1], "w"), indent=1)
