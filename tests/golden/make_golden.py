"""Regenerate tests/golden/reference_l0_l2.json from the REFERENCE's own code.

Run in the build container (needs oracle/_ref/libhetsim_ref.so, compiled from
/root/reference/proj/src by `make -C oracle ref`):

    python tests/golden/make_golden.py

Every fixture entry is {request, response} where response is exactly what the
reference's parse_spec/serialize/derive_components/classify_edges/
ready_components/bottom_level_ranks/buffer_bytes/eval_expr returned. The GPU box
(no /root/reference) replays the requests against the product in
tests/test_golden.py.
"""
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2009_07482_b200 import workloads  # noqa: E402
from tests import dag_gen  # noqa: E402


def requests():
    specs = [workloads.fork_join(), workloads.attention(), workloads.fig6_component(), workloads.fig6_component(True),
             workloads.fig7_spec(), workloads.head_dag(2, 128)]
    t, p, _ = workloads.encoder(layers=1)
    specs.append((t, p))
    specs += [dag_gen.layered_dag(5000 + s, max_kernels=10) for s in range(20)]
    for text, params in specs:
        yield {"op": "parse", "spec": text, "params": params}
        yield {"op": "analyze", "spec": text, "params": params}
        yield {"op": "bytes", "spec": text, "params": params}
        spec = O.Spec(text, params)
        order = spec.topo_order()
        yield {"op": "ready", "spec": text, "params": params, "finished": order[: len(order) // 2]}
        yield {"op": "ranks", "spec": text, "params": params,
               "times": {str(k): f"{k % 5 + 1}/{k % 3 + 1}" for k in spec.kernels}}
        for bad in dag_gen.mutations(text, len(text))[:4]:
            yield {"op": "parse", "spec": bad, "params": params}
    for e in ["M*N", "1024", "M/2", "7/2", "N/0", "(M+1)*N", "M*"]:
        for mode in ("eval", "positive", "validate"):
            yield {"op": "expr", "expr": e, "mode": mode, "params": {"M": 4, "N": 4}}
    for a, b in [("0.4", "8576/625"), ("1/3", "1/6"), ("3.25", "-7"), ("x", "1")]:
        yield {"op": "ratio", "a": a, "b": b}


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref/libhetsim_ref.so missing: run `make -C oracle ref` first")
    fixtures = [{"request": r, "response": O.ref_query(r)} for r in requests()]
    out = pathlib.Path(__file__).with_name("reference_l0_l2.json")
    out.write_text(json.dumps(fixtures, separators=(",", ":")))
    print(f"wrote {len(fixtures)} fixtures to {out} ({out.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
