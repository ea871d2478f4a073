"""CLI (SPEC.md cli module): subcommands on CPU (no GPU needed for validate /
simulate / compare / sweep --profiles) and the exit-code contract 0 / 1 / 2."""
import json
import subprocess
import sys

import pytest

from paper_2009_07482_b200 import workloads


def cli(*args, cwd=None):
    p = subprocess.run([sys.executable, "-m", "paper_2009_07482_b200", *args], capture_output=True, text=True,
                       cwd=cwd, timeout=120)
    return p.returncode, p.stdout, p.stderr


@pytest.fixture()
def forkjoin(tmp_path):
    text, params = workloads.fork_join(n=64)
    f = tmp_path / "fj.json"
    f.write_text(text)
    prof = tmp_path / "prof.json"
    prof.write_text(json.dumps({"devices": [{"device": 0, "type": "gpu", "kernel_times": {str(k): 1 for k in range(4)},
                                             "copy_channels": 2, "bandwidth": 1000000, "transfer_latency": 0}]}))
    return f, prof


def test_validate_prints_the_analysis(forkjoin):
    f, _ = forkjoin
    rc, out, err = cli("validate", "--spec", str(f), "--params", "N=64")
    assert rc == 0, err
    assert "components" in json.loads(out) or json.loads(out)


def test_validate_missing_param_and_cycle_exit_2(forkjoin, tmp_path):
    f, _ = forkjoin
    rc, _, err = cli("validate", "--spec", str(f))
    assert rc == 2 and "UnboundParameter" in err
    doc = json.loads(f.read_text())
    doc["depends"].append([3, 2, 0, 0])
    g = tmp_path / "cyc.json"
    g.write_text(json.dumps(doc))
    rc, _, err = cli("validate", "--spec", str(g), "--params", "N=64")
    assert rc == 2 and "Cycle" in err


def test_simulate_and_gantt(forkjoin):
    f, prof = forkjoin
    rc, out, err = cli("simulate", "--spec", str(f), "--params", "N=64", "--profiles", str(prof), "--gantt", "text")
    assert rc == 0, err
    ms = float(out.split()[1])
    assert ms >= 3.0  # k0 -> k1 -> k3 at 1 ms each
    assert "d0.q0" in out


def test_compare_three_policies(forkjoin, tmp_path):
    f, prof = forkjoin
    rc, out, err = cli("compare", "--spec", str(f), "--params", "N=64", "--profiles", str(prof), "--out",
                       str(tmp_path / "o"))
    assert rc == 0, err
    rows = out.strip().splitlines()
    assert len(rows) == 4 and {"clustering", "eager", "heft"} <= {r.split(",")[0] for r in rows[1:]}
    assert (tmp_path / "o" / "compare.csv").exists()
    rc, _, _ = cli("compare", "--spec", str(f), "--params", "N=64", "--profiles", str(prof), "--policies", "")
    assert rc == 2


def test_sweep_from_profiles(tmp_path):
    prof = tmp_path / "sw.json"
    prof.write_text(json.dumps({"gpu": {"gemm": 1.0, "transpose": 0.25, "softmax": 0.25},
                                "cpu": {"gemm": 20.0, "transpose": 2.0, "softmax": 2.0},
                                "share": {"gemm": 0.4, "transpose": 0.1, "softmax": 0.1}}))
    rc, out, err = cli("sweep", "--heads", "2", "--qgpu", "1-3", "--qcpu", "1-2", "--profiles", str(prof))
    assert rc == 0, err
    lines = out.strip().splitlines()
    assert lines[0].startswith("heads,beta,q_gpu") and lines[-1].startswith("best <")
    assert len(lines) == 1 + (3 + 3 * 2 + 2) + 1
    rc, _, err = cli("sweep", "--heads", "2", "--hcpu", "0-3", "--profiles", str(prof))
    assert rc == 2 and "hcpu" in err


def test_unknown_policy_is_a_usage_error(forkjoin):
    f, prof = forkjoin
    rc, _, _ = cli("simulate", "--spec", str(f), "--params", "N=64", "--profiles", str(prof), "--policy", "nope")
    assert rc == 2


def test_simulate_heft_waits_flag(tmp_path):
    """--heft-waits: the SPEC.md:338 HEFT example where the busy GPU's
    EFT (3 + 5) beats the idle CPU's (12): k1 waits for the GPU."""
    from tests.test_policies import _gpu_cpu, _two_kernels
    text, _ = _two_kernels()
    f = tmp_path / "two.json"
    f.write_text(text)
    prof = tmp_path / "prof.json"
    prof.write_text(json.dumps({"devices": _gpu_cpu({0: 3, 1: 5}, {0: 1000, 1: 12})}))
    base = ["simulate", "--spec", str(f), "--profiles", str(prof), "--policy", "heft", "--cpu-devices", "1"]
    rc, strict, err = cli(*base)
    assert rc == 0, err
    rc, waits, err = cli(*base, "--heft-waits")
    assert rc == 0, err
    assert float(waits.split()[1]) < float(strict.split()[1])
