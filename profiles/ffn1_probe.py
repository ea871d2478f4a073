"""Launch the DAG's FFN1 GEMM (gemm_relu 128x2048x512 x batch, resident pre-split
weight) exactly as bench.py's roofline probe does — for focused ncu captures.
usage: python profiles/ffn1_probe.py [math=tf32x3] [batch=256] [reps=1]"""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

math_mode = sys.argv[1] if len(sys.argv) > 1 else "tf32x3"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
tf, ms, flops = bench.gemm_roofline(batch, math_mode, reps=reps)
print(f"ffn1 {math_mode} batch={batch}: {ms:.3f} ms/launch {tf:.1f} TFLOP/s (not a bench number under ncu)")
