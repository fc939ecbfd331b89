"""Multi-process host logic of the replica bench: world_size 2 over gloo on CPU.
Every rank runs an independent replica (here: the oracle on a tiny traction bar, so no GPU is
needed); the job time is the max over ranks and the job value sums the ranks' load steps."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import time

    import torch

    from oracle import am as oam
    from oracle import problems as opb
    from oracle.p1 import MaterialSpec
    spec = MaterialSpec(E=1.0, nu=0.0, Gc=1.0, ell=0.1 + 0.05 * rank, k_ell=1e-6)  # distinct rows
    s = opb.traction(spec, L=1.0, H=0.2, nx=10, ny=2, n_steps=3)
    t0 = time.perf_counter()
    rows, _ = opb.run(s, oam.AMConfig(outer_atol=1e-8), snapshot_stride=0)
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    dist.barrier()
    tmax = t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    steps = torch.tensor([float(len(rows))], dtype=torch.float64)
    dist.all_reduce(steps, op=dist.ReduceOp.SUM)
    e = torch.tensor([rows[-1].energy.total], dtype=torch.float64)
    gathered = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, e)
    if rank == 0:
        out.put((float(tmax), float(steps), [float(g) for g in gathered], float(t)))
    dist.destroy_process_group()


def test_replicas_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    tmax, steps, energies, t0 = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert steps == 6.0                       # both replicas ran their 3 load steps
    assert tmax >= t0                         # job time is the max over ranks
    assert energies[0] != energies[1]         # independent replicas (different ell)
    assert all(np.isfinite(energies))


def _gpu_worker(rank, world, port, out):
    """One device replica per rank (both ranks share the box's single GPU: replicas never wait on
    each other's kernels), coordinated over gloo exactly as bench.py coordinates NCCL ranks."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    import paper_1511_08463_b200 as pf
    from oracle import am as oam
    from oracle import problems as opb
    from oracle.p1 import MaterialSpec
    torch.cuda.set_device(0)
    Gc = 1.0 + rank  # distinct sweep rows per replica (Gc rescales the loads and the energies)
    # smoke()'s bar, schedule and tolerance (a row pinned against the oracle on every box)
    setup = pf.setup_traction(pf.Material(E=1.0, nu=0.0, Gc=Gc, ell=0.05, k_ell=1e-6), L=1.0, H=0.1,
                              nx=40, ny=4, n_steps=3, pattern="right", load_max_factor=1.5)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    e0.record()
    recs = pf.run_quasistatic(setup, pf.SolverConfig(outer_atol=1e-8), snapshot_stride=0)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) * 1e-3], dtype=torch.float64)
    tmax = t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    # the same row on the CPU oracle: each replica computes its own row correctly
    os_ = opb.traction(MaterialSpec(E=1.0, nu=0.0, Gc=Gc, ell=0.05, k_ell=1e-6), L=1.0, H=0.1, nx=40,
                       ny=4, n_steps=3, pattern="right", load_max_factor=1.5)
    orows, _ = opb.run(os_, oam.AMConfig(outer_atol=1e-8), snapshot_stride=0)
    rel = max(abs(r.energy.total - o.energy.total) / abs(o.energy.total) for r, o in zip(recs, orows))
    stats = torch.tensor([rel, float(len(recs)), recs[-1].energy.total], dtype=torch.float64)
    gathered = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, stats)
    if rank == 0:
        out.put((float(tmax), float(t), [g.tolist() for g in gathered]))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_device_replicas_world2():
    """The replica mode of bench.py / the INI sweep with the DEVICE path in
    every rank: each replica's run matches the oracle for its own row, the job time is the max of
    the ranks' CUDA-event times, and the rows differ."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    tmax, t0, g = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert tmax >= t0 > 0.0
    for rel, n, _ in g:
        assert n == 3.0 and rel < 1e-6, g
    assert g[0][2] != g[1][2]
