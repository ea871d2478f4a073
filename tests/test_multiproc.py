"""The N>1 path on CPU: world_size-2 gloo. Each rank takes its contiguous
instance partition (bench.partition), plans the same DAG template with the
native scheduler, and runs its share of instances through the CPU oracle; the
union over ranks equals the single-process result and no data-path collective
is involved (only the barrier + max-reduce of the timing protocol)."""
import os
import pathlib
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = pathlib.Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    import bench
    from oracle import oracle as O
    from paper_2009_07482_b200 import hetsim, workloads
    total = 5
    first, n = bench.partition(total, world, rank)
    text, params = workloads.fork_join(n=32)
    plan = hetsim.run_schedule(hetsim.parse_spec(text, params))
    arrays = workloads.generic_inputs(text, params, total)
    mine = {k: (v[first:first + n] if v.ndim == 2 else v) for k, v in arrays.items()}
    out = O.run_dag(text, params, mine, n) if n else {}
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # the timing protocol's max over ranks
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), first=first, n=n, plan=np.array(plan["dispatches"]),
             tmax=t.item(), **{f"{k[0]}_{k[1]}": v for k, v in out.items()})
    dist.destroy_process_group()


def test_two_rank_partition(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    sys.path.insert(0, str(ROOT))
    from oracle import oracle as O
    from paper_2009_07482_b200 import workloads
    text, params = workloads.fork_join(n=32)
    arrays = workloads.generic_inputs(text, params, 5)
    full = O.run_dag(text, params, arrays, 5)
    r0, r1 = (np.load(tmp_path / f"r{i}.npz") for i in range(2))
    assert (int(r0["first"]), int(r0["n"]), int(r1["first"]), int(r1["n"])) == (0, 3, 3, 2)
    assert np.array_equal(r0["plan"], r1["plan"])
    assert float(r0["tmax"]) == float(r1["tmax"]) == 2.0
    for key, ref in full.items():
        name = f"{key[0]}_{key[1]}"
        assert np.array_equal(np.concatenate([r0[name], r1[name]]), ref)
