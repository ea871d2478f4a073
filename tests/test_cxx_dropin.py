"""Source-level drop-in: a C++ translation unit written
against the reference-named headers (include/hetsim/*.hpp: parse_spec,
derive_components, run_schedule) and the B200 executor plug-in
(include/hetsim/cuda_executor.hpp), compiled with g++ and linked against
libhetsim.so. On CPU the program must compile and link; on the GPU it runs the
C1 fork-join DAG and a one-layer encoder through Alg. 1 and its outputs match
the CPU oracle."""
import os
import pathlib
import struct
import subprocess

import numpy as np
import pytest

from paper_2009_07482_b200 import workloads

ROOT = pathlib.Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cxx" / "dropin_main.cpp"
LIBDIR = ROOT / "paper_2009_07482_b200"


def _build(tmp_path):
    exe = tmp_path / "dropin_main"
    cmd = ["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(SRC), f"-L{LIBDIR}", "-lhetsim",
           f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)]
    p = subprocess.run(cmd, capture_output=True, text=True)
    assert p.returncode == 0, p.stderr[-3000:]
    return exe


def test_dropin_translation_unit_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert exe.exists() and os.access(exe, os.X_OK)


def _write_io(path, arrays, outs, n):
    with open(path, "wb") as f:
        for (k, p), a in arrays.items():
            a = np.ascontiguousarray(a, np.float32)
            stride = 0 if a.ndim == 1 else a.shape[1] * 4
            f.write(struct.pack("<iiiqqq", k, p, 0, stride, 0 if a.ndim == 1 else a.shape[0], a.nbytes))
            f.write(a.tobytes())
        for (k, p), e in outs.items():
            f.write(struct.pack("<iiiqqq", k, p, 1, e * 4, n, n * e * 4))
            f.write(bytes(n * e * 4))


def _read_out(path):
    outs = {}
    data = pathlib.Path(path).read_bytes()
    off = 0
    while off < len(data):
        k, p, _, stride, count, nbytes = struct.unpack_from("<iiiqqq", data, off)
        off += struct.calcsize("<iiiqqq")
        outs[(k, p)] = np.frombuffer(data[off:off + nbytes], np.float32).reshape(count, -1)
        off += nbytes
    return outs


def _normwise(y, ref):
    y, ref = np.asarray(y, np.float64), np.asarray(ref, np.float64)
    return float(np.max(np.abs(y - ref)) / max(np.max(np.abs(ref)), 1e-30))


@pytest.mark.gpu
@pytest.mark.parametrize("dag", ["fork_join", "encoder_layer"])
def test_dropin_runs_alg1_on_the_b200(dag, tmp_path, oracle_mod):
    exe = _build(tmp_path)
    if dag == "fork_join":
        text, params = workloads.fork_join()
        n, batch = 3, 2
        arrays = workloads.generic_inputs(text, params, n)
    else:
        text, params, meta = workloads.encoder(layers=1)
        n, batch = 3, 3
        x = workloads.encoder_inputs(meta, params, n).reshape(n, -1)
        arrays = {(i["kernel"], i["pos"]): x for i in meta["x_inputs"]}
        for key, w in workloads.encoder_weights(meta).items():
            arrays[key] = w.reshape(-1)
    outs = {(k, p): e for k, p, e in workloads.isolated_outputs(text, params)}
    (tmp_path / "spec.json").write_text(text)
    (tmp_path / "params.txt").write_text("".join(f"{k} {v}\n" for k, v in params.items()))
    _write_io(tmp_path / "in.bin", arrays, outs, n)
    p = subprocess.run([str(exe), str(tmp_path / "spec.json"), str(tmp_path / "params.txt"), str(tmp_path / "in.bin"),
                        str(tmp_path / "out.bin"), str(n), str(batch)], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-3000:]
    assert p.stdout.startswith("components ")
    got = _read_out(tmp_path / "out.bin")
    ref = oracle_mod.run_dag(text, params, arrays, n)
    for key, r in ref.items():
        for i in range(n):
            assert _normwise(got[key][i], r[i]) <= 1e-4, (key, i)


TSAN_EXE = ROOT / "build_tsan" / "dropin_tsan"


@pytest.mark.gpu
@pytest.mark.parametrize("policy", ["clustering", "eager", "heft"])
def test_host_runtime_under_threadsanitizer(policy, tmp_path, oracle_mod):
    """SURVEY.md §4 race detection: the host runtime built with -fsanitize=thread
    (`make tsan`) drives Alg. 1 in dynamic mode — CUDA host callbacks on driver
    threads push completions through the MPSC queue to Scheduler::cb on the main
    thread (the paper's lock()/unlock() region). One component per
    kernel on three logical devices maximises concurrent callbacks. ThreadSanitizer
    must report nothing and the outputs must match the oracle."""
    if not TSAN_EXE.exists():
        p = subprocess.run(["make", "-C", str(ROOT), "tsan"], capture_output=True, text=True)
        assert p.returncode == 0, p.stderr[-3000:]
    text, params, meta = workloads.encoder(layers=1, tc_mode="per_kernel", queues=1, devices=3)
    n, batch = 2, 2
    x = workloads.encoder_inputs(meta, params, n).reshape(n, -1)
    arrays = {(i["kernel"], i["pos"]): x for i in meta["x_inputs"]}
    for key, w in workloads.encoder_weights(meta).items():
        arrays[key] = w.reshape(-1)
    outs = {(k, p): e for k, p, e in workloads.isolated_outputs(text, params)}
    (tmp_path / "spec.json").write_text(text)
    (tmp_path / "params.txt").write_text("".join(f"{k} {v}\n" for k, v in params.items()))
    _write_io(tmp_path / "in.bin", arrays, outs, n)
    env = dict(os.environ, TSAN_OPTIONS="halt_on_error=0 exitcode=66 report_signal_unsafe=0")
    p = subprocess.run([str(TSAN_EXE), str(tmp_path / "spec.json"), str(tmp_path / "params.txt"),
                        str(tmp_path / "in.bin"), str(tmp_path / "out.bin"), str(n), str(batch), policy],
                       capture_output=True, text=True, timeout=600, env=env)
    assert "ThreadSanitizer" not in p.stderr, p.stderr[-4000:]
    assert p.returncode == 0, p.stderr[-3000:]
    got = _read_out(tmp_path / "out.bin")
    ref = oracle_mod.run_dag(text, params, arrays, n)
    for key, r in ref.items():
        for i in range(n):
            assert _normwise(got[key][i], r[i]) <= 1e-4, (key, i)
