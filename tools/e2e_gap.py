"""Where the e2e-vs-device gap of bench.py comes from: one schedule step replayed from the same
snapshot (a) on the device state object, (b) on a fresh device State, (c) with snapshot_stride=1,
(d) from pinned host memory with the result read back (the bench's e2e leg)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
import bench

wl = sys.argv[1] if len(sys.argv) > 1 else "traction3d128"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 8
setup, cfg = bench.make_workload(pf, wl)
st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=list(range(W)))
snap = st.copy()


def timed(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0)


for rep in range(2):
    s = snap.copy()
    ta = timed(lambda: pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=s, steps=[W]))
    s = snap.copy()
    tb = timed(lambda: pf.run_quasistatic(setup, cfg, snapshot_stride=0,
                                          state=pf.State(s.u.clone(), s.alpha.clone(), s.alpha_lb.clone(), s.load),
                                          steps=[W]))
    s = snap.copy()
    tc = timed(lambda: pf.run_quasistatic(setup, cfg, snapshot_stride=1, state=s, steps=[W]))
    hu, ha, hl = (t.cpu().pin_memory() for t in (snap.u, snap.alpha, snap.alpha_lb))

    def d():
        s2 = pf.State(hu.to("cuda", non_blocking=True), ha.to("cuda", non_blocking=True),
                      hl.to("cuda", non_blocking=True), snap.load)
        pf.run_quasistatic(setup, cfg, snapshot_stride=1, state=s2, steps=[W])
    td = timed(d)
    print(f"{wl} step {W}: same-state {ta:.1f} ms  fresh-device-state {tb:.1f}  stride1 {tc:.1f}  host-io {td:.1f}")
