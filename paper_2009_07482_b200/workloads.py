"""DAG spec generators for the BASELINE configs and the paper's examples, plus
the deterministic synthetic-input generator shared by the GPU path and the
CPU oracle.

Configs (BASELINE.json `configs`):
  C1 fork_join()                       paper Fig. 1, 4 kernels, 256x256 fp32
  C2 attention()                       QK^T (gemm_nt) -> scale -> softmax -> PV
  C3 encoder(layers=1)                 8 heads, d_model 512, seq 128, d_ff 2048, 69 kernels
  C4 encoder(layers=6)                 414 kernels / 539 edges / 54 components
  C5 encoder(layers=12)                828 kernels / 1103 edges / 108 components
Paper examples: fig6_component() (Fig. 6/8 golden), fig7_spec(), head_dag() (SPEC gen_transformer).

Node operator conventions (argument positions / var-args) are in DESIGN.md §4.
"""
from __future__ import annotations

import json
import math

import numpy as np

# ----------------------------------------------------------------------------- spec building


class SpecBuilder:
    def __init__(self):
        self.kernels = []
        self.edges = []

    def kernel(self, name, inputs, outputs, var_args=(), dev="gpu", gws=("1", "1", "1")):
        """inputs/outputs: lists of (pos, size_expr); var_args: list of (pos, value)."""
        kid = len(self.kernels)
        self.kernels.append({
            "id": kid,
            "name": name,
            "dev": dev,
            "workDimension": 2,
            "globalWorkSize": list(gws),
            "inputBuffers": [{"type": "float32", "size": s, "pos": p} for p, s in inputs],
            "outputBuffers": [{"type": "float32", "size": s, "pos": p} for p, s in outputs],
            "ioBuffers": [],
            "varArguments": [{"type": "int", "pos": p, "value": str(v)} for p, v in var_args],
            "src": f"{name}.cu",
        })
        return kid

    def edge(self, src, src_pos, dst, dst_pos):
        self.edges.append([src, src_pos, dst, dst_pos])

    def gemm(self, m, n, k, name="gemm"):
        return self.kernel(name, [(0, f"{m}*{k}"), (1, f"{k}*{n}" if name != "gemm_nt" else f"{n}*{k}")],
                           [(2, f"{m}*{n}")], [(3, m), (4, n), (5, k)], gws=(m, n, "1"))

    def doc(self, tc, cq):
        return json.dumps({"kernels": self.kernels, "tc": tc, "cq": cq, "depends": self.edges}, indent=1)


def cq_list(devices=1, queues=3):
    return [{"device": d, "queues": queues} for d in range(devices)]


# ----------------------------------------------------------------------------- configs

def fork_join(n=256, queues=3):
    """C1 — paper Fig. 1 fork-join: k0=gemm(A,B); k1=gemm(k0,W1); k2=add(k0,W2); k3=add(k1,k2)."""
    b = SpecBuilder()
    k0 = b.gemm("N", "N", "N")
    k1 = b.gemm("N", "N", "N")
    k2 = b.kernel("add", [(0, "N*N"), (1, "N*N")], [(2, "N*N")], [(3, "N*N")])
    k3 = b.kernel("add", [(0, "N*N"), (1, "N*N")], [(2, "N*N")], [(3, "N*N")])
    b.edge(k0, 2, k1, 0)
    b.edge(k0, 2, k2, 0)
    b.edge(k1, 2, k3, 0)
    b.edge(k2, 2, k3, 1)
    return b.doc([[k0, k1, k2, k3]], cq_list(1, queues)), {"N": n}


def attention(seq=128, dk=64, queues=3):
    """C2 — single-head attention: A=gemm_nt(Q,K); A'=scale(A,1/8); P=softmax(A'); O=gemm(P,V)."""
    b = SpecBuilder()
    k0 = b.gemm("S", "S", "DK", name="gemm_nt")
    k1 = b.kernel("scale", [(0, "S*S")], [(1, "S*S")], [(2, "S*S"), (3, 1), (4, 8)])
    k2 = b.kernel("softmax", [(0, "S*S")], [(1, "S*S")], [(2, "S"), (3, "S")])
    k3 = b.gemm("S", "DK", "S")
    b.edge(k0, 2, k1, 0)
    b.edge(k1, 1, k2, 0)
    b.edge(k2, 1, k3, 0)
    return b.doc([[k0, k1, k2, k3]], cq_list(1, queues)), {"S": seq, "DK": dk}


ENCODER_PARAMS = {"S": 128, "D": 512, "DK": 64, "DFF": 2048}


def encoder(layers=1, heads=8, tc_mode="per_head", queues=3, devices=1, params=None, fused_heads=False):
    """C3/C4/C5 — transformer encoder layers as a fine-grained kernel DAG.

    Per head: Q,K,V = gemm(X, W*); Kt = transpose(K); A = gemm(Q, Kt);
    P = softmax(A, 1/8); C = gemm(P, V); Z = gemm(C, W_h). Tail: concat(Z_0..) ->
    add_layernorm(X, concat) -> gemm_relu(., W1) -> gemm(., W2) -> add_layernorm.
    tc_mode: per_head (8 head components + 1 tail per layer),
    per_kernel (every kernel its own component, the eager/HEFT setting), single.
    fused_heads: each head's Kt/A/P/C/Z chain is one `attn_head` node
    (Z = softmax(Q Kᵀ · 1/8) V W_h; 4 kernels per head instead of 8).
    Returns (spec_text, params, meta) where meta locates inputs/outputs.
    """
    p = dict(ENCODER_PARAMS if params is None else params)
    b = SpecBuilder()
    tc = []
    meta = {"layers": layers, "heads": heads, "x_inputs": [], "weights": [], "output": None}
    prev_out = None  # (kernel, pos) of the previous layer's output
    for layer in range(layers):
        head_ids = []
        z_ids = []
        for h in range(heads):
            ks = []
            proj = []
            for role in ("q", "k", "v"):
                kid = b.gemm("S", "DK", "D")
                proj.append(kid)
                ks.append(kid)
                meta["weights"].append({"kernel": kid, "pos": 1, "shape": [p["D"], p["DK"]], "fan_in": p["D"],
                                        "key": f"L{layer}.H{h}.W{role}"})
            q, k, v = proj
            if fused_heads:
                z = b.kernel("attn_head", [(0, "S*DK"), (1, "S*DK"), (2, "S*DK"), (3, "DK*DK")], [(4, "S*DK")],
                             [(5, "S"), (6, "DK"), (7, "DK"), (8, 1), (9, 8)])
                meta["weights"].append({"kernel": z, "pos": 3, "shape": [p["DK"], p["DK"]], "fan_in": p["DK"],
                                        "key": f"L{layer}.H{h}.Wh"})
                ks.append(z)
                b.edge(q, 2, z, 0)
                b.edge(k, 2, z, 1)
                b.edge(v, 2, z, 2)
                for kid in proj:
                    if prev_out is None:
                        meta["x_inputs"].append({"kernel": kid, "pos": 0})
                    else:
                        b.edge(prev_out[0], prev_out[1], kid, 0)
                head_ids.append(ks)
                z_ids.append(z)
                continue
            kt = b.kernel("transpose", [(0, "S*DK")], [(1, "DK*S")], [(2, "S"), (3, "DK")])
            a = b.gemm("S", "S", "DK")
            sm = b.kernel("softmax", [(0, "S*S")], [(1, "S*S")], [(2, "S"), (3, "S"), (4, 1), (5, 8)])
            c = b.gemm("S", "DK", "S")
            z = b.gemm("S", "DK", "DK")
            meta["weights"].append({"kernel": z, "pos": 1, "shape": [p["DK"], p["DK"]], "fan_in": p["DK"],
                                    "key": f"L{layer}.H{h}.Wh"})
            ks += [kt, a, sm, c, z]
            b.edge(k, 2, kt, 0)
            b.edge(q, 2, a, 0)
            b.edge(kt, 1, a, 1)
            b.edge(a, 2, sm, 0)
            b.edge(sm, 1, c, 0)
            b.edge(v, 2, c, 1)
            b.edge(c, 2, z, 0)
            for kid in proj:
                if prev_out is None:
                    meta["x_inputs"].append({"kernel": kid, "pos": 0})
                else:
                    b.edge(prev_out[0], prev_out[1], kid, 0)
            head_ids.append(ks)
            z_ids.append(z)
        cat = b.kernel("concat", [(i, "S*DK") for i in range(heads)], [(heads, f"S*DK*{heads}")],
                       [(heads + 1, "S"), (heads + 2, "DK")])
        for i, z in enumerate(z_ids):
            b.edge(z, 4 if fused_heads else 2, cat, i)
        ln1 = b.kernel("add_layernorm", [(0, "S*D"), (1, "S*D"), (2, "D"), (3, "D")], [(4, "S*D")], [(5, "S"), (6, "D")])
        if prev_out is None:
            meta["x_inputs"].append({"kernel": ln1, "pos": 0})
        else:
            b.edge(prev_out[0], prev_out[1], ln1, 0)
        b.edge(cat, heads, ln1, 1)
        meta["weights"].append({"kernel": ln1, "pos": 2, "shape": [p["D"]], "kind": "gamma", "key": f"L{layer}.g1"})
        meta["weights"].append({"kernel": ln1, "pos": 3, "shape": [p["D"]], "kind": "beta", "key": f"L{layer}.b1"})
        f1 = b.gemm("S", "DFF", "D", name="gemm_relu")
        meta["weights"].append({"kernel": f1, "pos": 1, "shape": [p["D"], p["DFF"]], "fan_in": p["D"],
                                "key": f"L{layer}.W1"})
        f2 = b.gemm("S", "D", "DFF")
        meta["weights"].append({"kernel": f2, "pos": 1, "shape": [p["DFF"], p["D"]], "fan_in": p["DFF"],
                                "key": f"L{layer}.W2"})
        ln2 = b.kernel("add_layernorm", [(0, "S*D"), (1, "S*D"), (2, "D"), (3, "D")], [(4, "S*D")], [(5, "S"), (6, "D")])
        meta["weights"].append({"kernel": ln2, "pos": 2, "shape": [p["D"]], "kind": "gamma", "key": f"L{layer}.g2"})
        meta["weights"].append({"kernel": ln2, "pos": 3, "shape": [p["D"]], "kind": "beta", "key": f"L{layer}.b2"})
        b.edge(ln1, 4, f1, 0)
        b.edge(f1, 2, f2, 0)
        b.edge(ln1, 4, ln2, 0)
        b.edge(f2, 2, ln2, 1)
        tail = [cat, ln1, f1, f2, ln2]
        if tc_mode == "per_head":
            tc += head_ids + [tail]
        elif tc_mode == "per_kernel":
            tc += [[k] for ks in head_ids for k in ks] + [[k] for k in tail]
        elif tc_mode == "single":
            tc += [[k for ks in head_ids for k in ks] + tail]
        else:
            raise ValueError(tc_mode)
        prev_out = (ln2, 4)
    if tc_mode == "single":
        tc = [[k for comp in tc for k in comp]]
    meta["output"] = {"kernel": prev_out[0], "pos": prev_out[1], "shape": [p["S"], p["D"]]}
    return b.doc(tc, cq_list(devices, queues)), p, meta


def fig6_component(with_b8=False):
    """Paper Fig. 6 DAG (component T = {k0..k4}) with a producer k5 and a consumer k6.

    Kernel/buffer layout: k5 -> (b0,b1) -> k0 -> b4 -> {k1, k2}; k1 (+ isolated b5) -> k3;
    k2 (+ isolated b8 when with_b8) -> k4; k3, k4 -> k6. tc = [[0..4],[5],[6]].
    Fig. 8's golden q2=[e3] needs k2 without its isolated input (SURVEY §8c ambiguity 1).
    """
    def k(id_, ins, outs, name="op"):
        return {"id": id_, "name": name, "dev": "gpu", "workDimension": 1, "globalWorkSize": ["N", "1", "1"],
                "inputBuffers": [{"type": "float32", "size": "N", "pos": p} for p in ins],
                "outputBuffers": [{"type": "float32", "size": "N", "pos": p} for p in outs],
                "ioBuffers": [], "varArguments": [], "src": ""}
    kernels = [
        k(0, [0, 1], [2]),
        k(1, [0, 1], [2]),
        k(2, [0, 1] if with_b8 else [0], [2] if with_b8 else [1]),
        k(3, [0], [1]),
        k(4, [0], [1]),
        k(5, [], [0, 1]),
        k(6, [0, 1], [2]),
    ]
    k2_out = 2 if with_b8 else 1
    edges = [[5, 0, 0, 0], [5, 1, 0, 1], [0, 2, 1, 0], [0, 2, 2, 0], [1, 2, 3, 0], [2, k2_out, 4, 0],
             [3, 1, 6, 0], [4, 1, 6, 1]]
    doc = {"kernels": kernels, "tc": [[0, 1, 2, 3, 4], [5], [6]], "cq": [{"device": 0, "queues": 3}],
           "depends": edges}
    return json.dumps(doc, indent=1), {"N": 1024}


def fig7_spec():
    """Paper Fig. 7: three matmul kernels, tc={{0,2},{1}}, edge 0,2 -> 2,0."""
    def mm(i, dev):
        return {"id": i, "name": "gemm", "dev": dev, "workDimension": 2, "globalWorkSize": ["M", "N", "1"],
                "inputBuffers": [{"type": "float32", "size": "M*K", "pos": 0},
                                 {"type": "float32", "size": "K*N", "pos": 1}],
                "outputBuffers": [{"type": "float32", "size": "M*N", "pos": 2}], "ioBuffers": [],
                "varArguments": [{"type": "int", "pos": 3, "value": "M"}, {"type": "int", "pos": 4, "value": "N"},
                                 {"type": "int", "pos": 5, "value": "K"}], "src": "gemm.cl"}
    doc = {"kernels": [mm(0, "gpu"), mm(1, "cpu"), mm(2, "gpu")], "depends": [[0, 2, 2, 0]],
           "tc": [[0, 2], [1]], "cq": [{"device": 0, "queues": 2}, {"device": 1, "queues": 1}]}
    return json.dumps(doc, indent=1), {"M": 64, "N": 64, "K": 64}


def head_dag(heads=1, beta=256, tc_mode="per_head", queues=3):
    """SPEC.md:483-491 gen_transformer: per head 3 level-1 GEMMs on a shared X, transpose,
    QK^T GEMM, softmax, PV GEMM, Z GEMM; all matrices beta x beta; heads independent."""
    b = SpecBuilder()
    comps = []
    for _ in range(heads):
        q, k, v = (b.gemm("B", "B", "B") for _ in range(3))
        kt = b.kernel("transpose", [(0, "B*B")], [(1, "B*B")], [(2, "B"), (3, "B")])
        a = b.gemm("B", "B", "B")
        sm = b.kernel("softmax", [(0, "B*B")], [(1, "B*B")], [(2, "B"), (3, "B")])
        c = b.gemm("B", "B", "B")
        z = b.gemm("B", "B", "B")
        for e in ((k, 2, kt, 0), (q, 2, a, 0), (kt, 1, a, 1), (a, 2, sm, 0), (sm, 1, c, 0), (v, 2, c, 1), (c, 2, z, 0)):
            b.edge(*e)
        comps.append([q, k, v, kt, a, sm, c, z])
    tc = comps if tc_mode == "per_head" else [[x] for comp in comps for x in comp]
    return b.doc(tc, cq_list(1, queues)), {"B": beta}


# ----------------------------------------------------------------------------- synthetic inputs

_M1 = np.uint64(0x9E3779B97F4A7C15)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + _M1
        z = (z ^ (z >> np.uint64(30))) * _M2
        z = (z ^ (z >> np.uint64(27))) * _M3
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, uid: int, n: int) -> np.ndarray:
    """splitmix64(seed ^ uid<<32 ^ i) -> top 24 bits -> uniform[-1, 1), exact in fp32."""
    base = np.uint64((seed ^ (uid << 32)) & 0xFFFFFFFFFFFFFFFF)
    z = splitmix64(base ^ np.arange(n, dtype=np.uint64))
    return ((z >> np.uint64(40)).astype(np.float64) / float(1 << 23) - 1.0).astype(np.float32)


def buffer_uid(kernel: int, pos: int) -> int:
    return kernel * 64 + pos


def encoder_inputs(meta, params, n_instances, first=0, seed=7482):
    """X for instances [first, first+n): shape [n, S, D], instance i uses seed 7482+i."""
    S, D = params["S"], params["D"]
    x = np.empty((n_instances, S * D), dtype=np.float32)
    for j in range(n_instances):
        x[j] = uniform(seed + first + j, 1, S * D)
    return x.reshape(n_instances, S, D)


def encoder_weights(meta, seed=1):
    """Weights keyed by (kernel,pos): W ~ u/sqrt(fan_in); gamma = 1+0.1u; beta = 0.1u."""
    out = {}
    for w in meta["weights"]:
        n = int(np.prod(w["shape"]))
        u = uniform(seed, buffer_uid(w["kernel"], w["pos"]), n)
        kind = w.get("kind")
        if kind == "gamma":
            v = (np.float32(1.0) + np.float32(0.1) * u).astype(np.float32)
        elif kind == "beta":
            v = (np.float32(0.1) * u).astype(np.float32)
        else:
            v = (u * np.float32(1.0 / math.sqrt(w["fan_in"]))).astype(np.float32)
        out[(w["kernel"], w["pos"])] = v.reshape(w["shape"])
    return out


def isolated_inputs(spec_text, params):
    """(kernel,pos,elements) of every input-side buffer with no producer edge."""
    doc = json.loads(spec_text)
    fed = {(e[2], e[3]) for e in doc.get("depends", [])}
    out = []
    for k in doc["kernels"]:
        for b in k.get("inputBuffers", []) + k.get("ioBuffers", []):
            if (k["id"], b["pos"]) not in fed:
                out.append((k["id"], b["pos"], _eval(b["size"], params)))
    return out


def isolated_outputs(spec_text, params):
    doc = json.loads(spec_text)
    feeding = {(e[0], e[1]) for e in doc.get("depends", [])}
    out = []
    for k in doc["kernels"]:
        for b in k.get("outputBuffers", []) + k.get("ioBuffers", []):
            if (k["id"], b["pos"]) not in feeding:
                out.append((k["id"], b["pos"], _eval(b["size"], params)))
    return out


def _eval(expr, params):
    # sizes here are products of names/integers; the native evaluator is the authority
    val = 1
    for tok in str(expr).replace(" ", "").split("*"):
        val *= params[tok] if tok in params else int(tok)
    return val


def generic_inputs(spec_text, params, n_instances, seed=7482, shared=()):
    """Inputs for small configs (C1, C2, tests): every isolated input gets its own
    uniform[-1,1) stream; buffers in `shared` are instance-independent (seed 1)."""
    arrays = {}
    for kid, pos, n in isolated_inputs(spec_text, params):
        if (kid, pos) in shared:
            arrays[(kid, pos)] = uniform(1, buffer_uid(kid, pos), n)
        else:
            arr = np.empty((n_instances, n), dtype=np.float32)
            for j in range(n_instances):
                arr[j] = uniform(seed + j, buffer_uid(kid, pos), n)
            arrays[(kid, pos)] = arr
    return arrays
