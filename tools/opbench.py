"""Standalone operator-apply driver for ncu / timing: python tools/opbench.py OP N [PATTERN] [REPS]
OP in {Kuu, Kaa, phys}; prints median ms and GB/s (algorithmic bytes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1511_08463_b200 as pf  # noqa: E402


def main():
    op = sys.argv[1] if len(sys.argv) > 1 else "Kuu"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    pattern = sys.argv[3] if len(sys.argv) > 3 else "union_jack"
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
    if pattern == "kuhn6":
        mesh = pf.StructuredMesh3D(n, n, n)
        mat = pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6, regime="3d")
    else:
        mesh = pf.StructuredMesh(n, n, 1.0, 1.0, pattern)
        mat = pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6)
    prob = pf.Discretization(mesh, mat, pf.DamageModel("AT1"), solvers="operators")
    V = mesh.n_vertices
    d = mesh.dim
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.rand(V, dtype=torch.float64, device="cuda", generator=g)
    u = torch.randn(d * V, dtype=torch.float64, device="cuda", generator=g)
    xa = torch.randn(V, dtype=torch.float64, device="cuda", generator=g)
    st = pf.State(u, a, torch.zeros_like(a))
    if op == "Kuu":
        K = pf.assemble_Kuu(st, prob, apply_bc=False)
        f, x, nbytes = K.matvec, u, (40.0 if d == 2 else 56.0) * V
    elif op == "Kaa":
        K = pf.assemble_Kaa(st, prob)
        f, x, nbytes = K.matvec, xa, 16.0 * V + 8.0 * prob.n_elements
    else:
        f, x, nbytes = (lambda _x: pf.fem.physics(st, prob)), None, 32.0 * V
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    ts = []
    for _ in range(reps):
        flush.add_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        f(x)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[len(ts) // 2]
    print(f"{op} n={n} {pattern}: median {t:.4f} ms  {nbytes / t / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
