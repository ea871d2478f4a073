"""Random layered DAG specs for differential / property tests (SPEC.md:562:
">= 200 randomly generated layered DAGs (<= 20 kernels) with random partitions")."""
from __future__ import annotations

import json
import random


def layered_dag(seed: int, max_kernels: int = 20, convex: bool = True, devices: int = 2, cpu_frac: float = 0.0):
    """Returns (spec_text, params).

    Kernels are arranged in layers; every kernel has 1-3 input buffers and 1-2
    output buffers (sizes are symbolic over N/M). Each input is fed by at most
    one output of an earlier layer (or left isolated). Components are random
    runs of a topological order when `convex` (always schedulable), otherwise
    random subsets (may deadlock under device exclusivity).
    """
    rng = random.Random(seed)
    n = rng.randint(1, max_kernels)
    layers = []
    ids = list(range(n))
    rng.shuffle(ids)  # ids are not in topological order
    i = 0
    while i < n:
        w = rng.randint(1, 4)
        layers.append(ids[i:i + w])
        i += w
    kernels, edges, outputs = {}, [], []
    dev_of = {}
    for li, layer in enumerate(layers):
        for kid in layer:
            n_in, n_out = rng.randint(1, 3), rng.randint(1, 2)
            positions = list(range(n_in + n_out + rng.randint(0, 2)))
            rng.shuffle(positions)
            in_pos, out_pos, var_pos = positions[:n_in], positions[n_in:n_in + n_out], positions[n_in + n_out:]
            size = rng.choice(["N", "M*N", "N*4", "64", "(M+2)*N/3*3", "N - 1"])
            dev = "cpu" if rng.random() < cpu_frac else "gpu"
            dev_of[kid] = dev
            kernels[kid] = {
                "id": kid, "name": rng.choice(["gemm", "op", "add"]), "dev": dev, "workDimension": rng.randint(1, 3),
                "globalWorkSize": [size, "1", "1"],
                "inputBuffers": [{"type": rng.choice(["float32", "int32", "float64"]), "size": size, "pos": p}
                                 for p in sorted(in_pos)],
                "outputBuffers": [{"type": "float32", "size": size, "pos": p} for p in sorted(out_pos)],
                "ioBuffers": [],
                "varArguments": [{"type": "int", "pos": p, "value": rng.choice(["N", "M", "3", "N*M"])} for p in var_pos],
                "src": f"k{kid}.cl",
            }
            if li > 0:
                for p in in_pos:
                    if rng.random() < 0.7 and outputs:
                        src, sp = rng.choice(outputs)
                        edges.append([src, sp, kid, p])
        for kid in layer:
            for b in kernels[kid]["outputBuffers"]:
                outputs.append((kid, b["pos"]))
    topo = [k for layer in layers for k in layer]
    tc = []
    if convex:
        # contiguous runs of the topological order; split runs on device-type changes
        i = 0
        while i < n:
            w = rng.randint(1, 5)
            run = topo[i:i + w]
            cur = [run[0]]
            for k in run[1:]:
                if dev_of[k] == dev_of[cur[-1]]:
                    cur.append(k)
                else:
                    tc.append(cur)
                    cur = [k]
            tc.append(cur)
            i += w
    else:
        pool = topo[:]
        rng.shuffle(pool)
        by_dev = {"gpu": [k for k in pool if dev_of[k] == "gpu"], "cpu": [k for k in pool if dev_of[k] == "cpu"]}
        for ks in by_dev.values():
            while ks:
                w = rng.randint(1, 4)
                tc.append(ks[:w])
                ks = ks[w:]
    rng.shuffle(tc)
    for comp in tc:
        rng.shuffle(comp)
    cq = [{"device": d, "queues": rng.randint(1, 4)} for d in range(devices)]
    doc = {"kernels": [kernels[k] for k in sorted(kernels, key=lambda _: rng.random())], "tc": tc, "cq": cq,
           "depends": edges}
    return json.dumps(doc), {"N": rng.choice([4, 8, 64]), "M": rng.choice([1, 4, 16])}


def mutations(text: str, seed: int):
    """Invalid variants of a valid spec document (for Errc parity)."""
    rng = random.Random(seed)
    doc = json.loads(text)
    out = []
    if doc["depends"]:
        d = json.loads(text)
        e = rng.choice(d["depends"])
        d["depends"].append([e[2], rng.choice([0, 1]), e[0], 0])  # likely a cycle / bad endpoint
        out.append(d)
        d = json.loads(text)
        d["depends"][0][0] = 999  # unknown kernel
        out.append(d)
        d = json.loads(text)
        d["depends"].append(list(d["depends"][0]))  # multiple producers
        out.append(d)
    d = json.loads(text)
    d["tc"] = d["tc"][1:]  # partition gap
    out.append(d)
    d = json.loads(text)
    d["tc"].append([d["kernels"][0]["id"]])  # duplicate
    out.append(d)
    d = json.loads(text)
    d["kernels"][0]["inputBuffers"].append({"type": "float32", "size": "N", "pos": 0})  # clash
    out.append(d)
    d = json.loads(text)
    d["kernels"][0]["outputBuffers"][0]["size"] = "N/"  # syntax
    out.append(d)
    d = json.loads(text)
    d["kernels"][0]["outputBuffers"][0]["size"] = "N/0"
    out.append(d)
    d = json.loads(text)
    d["kernels"][0]["outputBuffers"][0]["size"] = "7/2"
    out.append(d)
    d = json.loads(text)
    d["kernels"][0]["dev"] = "fpga"
    out.append(d)
    d = json.loads(text)
    d["kernels"][0]["workDimension"] = 4
    out.append(d)
    d = json.loads(text)
    d["kernels"][0]["id"] = -1
    out.append(d)
    d = json.loads(text)
    d["kernels"][0]["globalWorkSize"] = ["1", "1"]
    out.append(d)
    d = json.loads(text)
    d["kernels"].append(dict(d["kernels"][0]))  # duplicate id
    out.append(d)
    d = json.loads(text)
    d["cq"][0]["queues"] = -1
    out.append(d)
    d = json.loads(text)
    d["kernels"][0]["outputBuffers"][0]["type"] = "float16"
    out.append(d)
    d = json.loads(text)
    d["kernels"][0]["varArguments"] = [{"type": "int", "pos": 50, "value": "1"}]  # uncovered positions
    out.append(d)
    texts = [json.dumps(x) for x in out]
    texts += [text[: len(text) // 2], text + "}", "[]", "{}", '{"kernels": 3}', '{"kernels": null}',
              text.replace('"id"', '"ID"', 1)]
    return texts
