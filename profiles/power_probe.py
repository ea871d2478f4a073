"""Board power and SM clock while one kernel runs back to back for ~2 s: the FFN1 pair GEMM
(128x2048x512 x512, tf32x3) of the loaded library (HETSIM_LIB selects a variant, e.g. one
built with -DHS_DBG_NOCONV=1). Prints time per launch, TFLOP/s, median SM clock and power.
usage: python profiles/power_probe.py [seconds=2] [fill: random|zeros|ones]"""
import ctypes
import statistics
import subprocess
import sys
import tempfile
import time

sys.path.insert(0, ".")
from profiles import gemm_micro as gm  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
fill = sys.argv[2] if len(sys.argv) > 2 and sys.argv[2] != "random" else None
us = gm.run(128, 2048, 512, 512, op="gemm_relu", reps=20, fill=fill)
reps = int(secs * 1e6 / us)
path = tempfile.mktemp(suffix=".csv")
smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                        "--format=csv,noheader,nounits", "-lms", "100"], stdout=open(path, "w"))
time.sleep(0.3)
t0 = time.time()
us2 = gm.run(128, 2048, 512, 512, op="gemm_relu", reps=reps, fill=fill)
wall = time.time() - t0
smi.terminate()
smi.wait()
rows = [r.split(",") for r in open(path) if r.strip()]
load = [r for r in rows if float(r[1]) > 300]
print(f"operands {fill or 'random'}: back to back {reps} launches in {wall:.2f} s: {us2:.1f} us/launch; "
      f"SM clock median {statistics.median(float(r[0]) for r in load):.0f} MHz, "
      f"power median {statistics.median(float(r[1]) for r in load):.0f} W max {max(float(r[1]) for r in load):.0f} W, "
      f"power cap active in {sum(1 for r in load if 'Active' in r[2])}/{len(load)} samples")
