"""bench.py end to end on the GPU at a small size: one rank, and two ranks under
torchrun sharing the box's GPU (HS_BENCH_SHARED_GPU=1: gloo for the timing
collectives), so the multi-rank partition / barrier / max-over-ranks path runs."""
import json
import os
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
ARGS = ["--instances", "128", "--batch", "64", "--layers", "2", "--steps", "1", "--warmup", "3", "--no-alt",
        "--no-cpu-baseline", "--no-makespans"]


def _line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


@pytest.mark.gpu
def test_bench_single_rank():
    p = subprocess.run([sys.executable, "bench.py", *ARGS], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    line = _line(p.stdout)
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["gpu_launches"] > 0
    par = line["parity"]
    assert par["pass"] and par["normwise_vs_oracle"] <= 1e-4 and par["instances_checked"] >= 16
    assert par["normwise_vs_f64"] <= 1e-4 and par["e2e_bit_identical_all_instances"]
    # every batch's first and last instance is among the checked ones
    assert {0, 63, 64, 127} <= set(par["per_rank"][0]["instances"])
    assert line["e2e"]["h2d_bytes_per_step"] == 128 * 128 * 512 * 4


@pytest.mark.gpu
@pytest.mark.parametrize("launcher", ["torchrun", "self"])
def test_bench_two_ranks_partition_the_stream(launcher):
    """`torchrun ... bench.py --gpus 2` (the driver's launch) and plain `bench.py --gpus 2`
    (bench re-launches itself as two ranks) both time two ranks and check both
    partitions against the oracle."""
    env = dict(os.environ, HS_BENCH_SHARED_GPU="1")
    env.pop("WORLD_SIZE", None)
    if launcher == "torchrun":
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
               "127.0.0.1", "--master-port", "29561", "bench.py", "--gpus", "2", *ARGS]
    else:
        cmd = [sys.executable, "bench.py", "--gpus", "2", *ARGS]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    line = _line(p.stdout)
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["config"]["parallelism"] == "instance partition x2"
    par = line["parity"]
    assert par["ranks"] == 2 and par["pass"] and par["e2e_bit_identical_all_instances"]
    firsts = sorted(min(r["instances"]) for r in par["per_rank"])
    assert firsts == [0, 64] and all(len(r["instances"]) >= 16 for r in par["per_rank"])


@pytest.mark.gpu
def test_cli_run_and_measured_sweep(tmp_path):
    """The CLI's B200 subcommands: `run` executes a spec through the engine and writes
    its trace and outputs; `sweep --measure` profiles the head DAG's nodes on the GPU
    (and the host) and simulates the mc grid."""
    from paper_2009_07482_b200 import workloads
    text, params = workloads.fork_join(n=256)
    spec = tmp_path / "fj.json"
    spec.write_text(text)
    out = tmp_path / "out"
    p = subprocess.run([sys.executable, "-m", "paper_2009_07482_b200", "run", "--spec", str(spec), "--params",
                        "N=256", "--instances", "2", "--out", str(out)], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    assert p.stdout.startswith("makespan_ms")
    assert (out / "trace.json").exists() and list(out.glob("out_k3_p2.npy"))
    p = subprocess.run([sys.executable, "-m", "paper_2009_07482_b200", "sweep", "--heads", "2", "--beta", "128",
                        "--qgpu", "1-2", "--qcpu", "1", "--measure"], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = p.stdout.strip().splitlines()
    assert lines[0].startswith("heads,beta") and lines[-1].startswith("best <")
