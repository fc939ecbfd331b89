"""A/B of the two 2D strip engines: Kuu / Kaa applies at several sizes and patterns in one process.
PF_STRIP2 is read at context creation, so each (engine, mesh) builds its own Discretization.
usage: python tools/opbench2.py [sizes=512,1024,2048,4096,8192] [patterns=union_jack,crossed]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1511_08463_b200 as pf  # noqa: E402


def run(op, n, pattern, engine, reps):
    os.environ["PF_STRIP2"] = str(engine)
    mesh = pf.StructuredMesh(n, n, 1.0, 1.0, pattern)
    mat = pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6)
    prob = pf.Discretization(mesh, mat, pf.DamageModel("AT1"), solvers="operators")
    V = mesh.n_vertices
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.rand(V, dtype=torch.float64, device="cuda", generator=g)
    u = torch.randn(2 * V, dtype=torch.float64, device="cuda", generator=g)
    xa = torch.randn(V, dtype=torch.float64, device="cuda", generator=g)
    st = pf.State(u, a, torch.zeros_like(a))
    if op == "Kuu":
        K = pf.assemble_Kuu(st, prob, apply_bc=False)
        f, x, nbytes = K.matvec, u, 40.0 * V
    else:
        K = pf.assemble_Kaa(st, prob)
        f, x, nbytes = K.matvec, xa, 16.0 * V + 8.0 * prob.n_elements
    y = f(x)
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
    del prob
    return t, nbytes / t / 1e6, y


def main():
    sizes = [int(s) for s in (sys.argv[1] if len(sys.argv) > 1 else "512,1024,2048,4096,8192").split(",")]
    pats = (sys.argv[2] if len(sys.argv) > 2 else "union_jack,crossed").split(",")
    for op in ("Kuu", "Kaa"):
        for pattern in pats:
            for n in sizes:
                reps = 21 if n <= 2048 else 7
                t1, g1, y1 = run(op, n, pattern, 0, reps)
                t2, g2, y2 = run(op, n, pattern, 1, reps)
                d = float((y1 - y2).abs().max() / y1.abs().max())
                print(f"{op:3s} {pattern:10s} {n:5d}: v1 {t1:8.4f} ms {g1:7.1f} GB/s | v2 {t2:8.4f} ms {g2:7.1f} GB/s "
                      f"| v2/v1 time {t2 / t1:5.2f} | max rel diff {d:.1e}", flush=True)
                del y1, y2
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
