"""Time the explicit dense-operator sketch Y = A Omega (N x N FP64 operator, 128 stream columns):
int8 tensor-core path (h2_dense_op_sketch with the Omega stream) vs cuBLAS DGEMM."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_16759_b200 as g

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
nc = int(sys.argv[2]) if len(sys.argv) > 2 else 128
A = torch.rand(n, n, dtype=torch.float64, device="cuda") - 0.5
Om = g.omega(n, nc)
for q in (True, False):
    for _ in range(2):
        g.dense_op_sketch(A, Om, omega_quarters=q)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        Y = g.dense_op_sketch(A, Om, omega_quarters=q)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{'tensor-core int8' if q else 'cuBLAS DGEMM'}: n={n} cols={nc} {ms:.2f} ms  "
          f"(A read {n * n * 8 / ms / 1e6:.0f} GB/s, {2.0 * n * n * nc / ms / 1e9:.1f} TF/s FP64-equivalent)", flush=True)
