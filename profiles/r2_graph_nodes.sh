mkdir -p gpurun_out
{ timeout 600 python -m pytest tests/test_gpu_engine_guards.py -q -x 2>&1 | tail -2
python - <<'PY'
import json, sys
sys.path.insert(0, ".")
import bench
for cfg, kw in (("C1", {}), ("C2", {}), ("C3", {"devices": 9}), ("C4", {"devices": 9})):
    r = bench.config_makespan(cfg, check=False, **kw)
    print(cfg, json.dumps({k: r[k] for k in ("makespan_ms", "makespan_min_ms", "graph_makespan_ms")}))
PY
} > gpurun_out/r2_graph_nodes.txt 2>&1
