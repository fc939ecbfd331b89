import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1511_08463_b200 as pf

def mk(engine):
    os.environ["PF_STRIP2"] = str(engine)
    mat = pf.Material(E=1.0, nu=0.0, Gc=1.0, ell=0.05, k_ell=1e-6)
    setup = pf.setup_traction(mat, L=1.0, H=0.1, nx=100, ny=10, n_steps=8, pattern="right")
    return setup

rng = np.random.default_rng(0)
nv = 101 * 11
lb = rng.uniform(0, 0.3, nv)
al = lb + rng.uniform(0, 1, nv) * (1 - lb)
al[50 * 11:52 * 11] = 1.0  # a cracked band
u = rng.standard_normal(2 * nv) * 0.1
x = rng.standard_normal(2 * nv)
xa = rng.standard_normal(nv)
res = {}
for eng in (0, 1):
    setup = mk(eng)
    prob = setup.problem
    st = pf.State.from_numpy(u, al, lb)
    setup.apply_load(prob, st, 2.0)
    cfg = pf.SolverConfig(outer_atol=1e-8)
    out = {}
    out["Kuu_bc"] = (pf.assemble_Kuu(st, prob, apply_bc=True) @ torch.as_tensor(x, device="cuda")).cpu().numpy()
    out["Kuu_raw"] = (pf.assemble_Kuu(st, prob, apply_bc=False) @ torch.as_tensor(x, device="cuda")).cpu().numpy()
    out["Kaa"] = (pf.assemble_Kaa(st, prob) @ torch.as_tensor(xa, device="cuda")).cpu().numpy()
    r = pf.elastic_step(st, prob, cfg)
    out["u_el"] = st.u.cpu().numpy().copy()
    print(eng, "elastic", r)
    r = pf.damage_step(st, prob, cfg)
    out["a_dmg"] = st.alpha.cpu().numpy().copy()
    print(eng, "damage", r)
    res[eng] = out
for k in res[0]:
    d = np.abs(res[0][k] - res[1][k])
    print(k, "max abs diff", d.max(), "rel", d.max() / np.abs(res[0][k]).max(), "argmax", int(d.argmax()))
