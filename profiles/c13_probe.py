import sys, json
sys.path.insert(0, ".")
import bench
for c in ("C1", "C3"):
    r = bench.config_makespan(c, devices=9 if c == "C3" else 1, reps=20, check=True)
    print(c, round(r["makespan_ms"], 4), r["normwise_err_vs_cpu_oracle"])
