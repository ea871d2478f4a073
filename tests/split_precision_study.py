"""TEST INFRASTRUCTURE (offline study, uses the CPU oracle as the checker): precision study: emulate split-precision GEMMs (tf32x3, bf16x3,
bf16x2+, tf32x1) inside the full 12-layer encoder DAG with numpy and report the
normwise error of the final output against the fp32 CPU oracle.

Emulation: x = hi + lo with hi = round(x) to the reduced format (RNE), lo =
round(x - hi); the GEMM sums the chosen partial products in float64 (the
tensor core accumulates in fp32, which the oracle itself also does)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_2009_07482_b200 import workloads  # noqa: E402


def rne(x, mant_bits):
    """Round float32 array to `mant_bits` explicit mantissa bits (RNE), as float32."""
    b = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    drop = 23 - mant_bits
    half = np.uint64(1 << (drop - 1))
    lsb = (b >> np.uint64(drop)) & np.uint64(1)
    b = (b + half - np.uint64(1) + lsb) & ~np.uint64((1 << drop) - 1)
    return b.astype(np.uint32).view(np.float32)


def split(x, bits):
    hi = rne(x, bits)
    lo = rne((x - hi).astype(np.float32), bits)
    return hi.astype(np.float64), lo.astype(np.float64)


def make_gemm(mode):
    bits = {"tf32": 10, "bf16": 7}

    def gemm(a, b):
        if mode == "fp32":
            return (a.astype(np.float64) @ b.astype(np.float64)).astype(np.float32)
        fmt, terms = mode.split("x")
        ah, al = split(a, bits[fmt])
        bh, bl = split(b, bits[fmt])
        out = ah @ bh
        if terms == "3":
            out += ah @ bl + al @ bh
        return out.astype(np.float32)
    return gemm


def encoder(x, W, layers, gemm):
    ws = W

    def ln(v, g, b):
        v = v.astype(np.float64)
        return ((v - v.mean(1, keepdims=True)) / np.sqrt(v.var(1, keepdims=True) + 1e-5) * g + b).astype(np.float32)

    i = 0
    for _ in range(layers):
        Z = []
        for h in range(8):
            q, k, v, wh = ws[i], ws[i + 1], ws[i + 2], ws[i + 3]
            i += 4
            Q, K, V = gemm(x, q), gemm(x, k), gemm(x, v)
            A = gemm(Q, np.ascontiguousarray(K.T)) * np.float32(0.125)
            P = np.exp(A - A.max(1, keepdims=True))
            P = (P / P.sum(1, keepdims=True)).astype(np.float32)
            Z.append(gemm(gemm(P, V), wh))
        g1, b1, w1, w2, g2, b2 = ws[i:i + 6]
        i += 6
        h1 = ln(x + np.concatenate(Z, 1), g1, b1)
        f = gemm(np.maximum(gemm(h1, w1), 0), w2)
        x = ln(h1 + f, g2, b2)
    return x


def main(layers=12):
    text, params, meta = workloads.encoder(layers=layers)
    x = workloads.encoder_inputs(meta, params, 1).reshape(1, -1)
    arrays = {(i["kernel"], i["pos"]): x for i in meta["x_inputs"]}
    Wd = workloads.encoder_weights(meta)
    for k, w in Wd.items():
        arrays[k] = w.reshape(-1)
    ref = O.run_dag(text, params, arrays, 1)[(meta["output"]["kernel"], meta["output"]["pos"])].reshape(128, 512)
    ws = [Wd[(w["kernel"], w["pos"])] for w in meta["weights"]]
    for mode in ("fp32", "tf32x3", "bf16x3", "tf32x1", "bf16x1"):
        y = encoder(x.reshape(128, 512), ws, layers, make_gemm(mode))
        err = np.max(np.abs(y.astype(np.float64) - ref)) / np.max(np.abs(ref))
        print(f"{layers}-layer encoder, GEMMs in {mode:7s}: normwise error vs fp32 oracle = {err:.2e}", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 12)
