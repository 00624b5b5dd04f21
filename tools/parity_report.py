import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from conftest import CASES, load_golden, oracle_for, rel_fields
from test_gpu_parity import build, dev
from paper_1702_04316_b200 import euler, imexcore
for name in sorted(CASES):
    mesh, ref, disc = build(name); o = oracle_for(name); g = load_golden(name)
    q = o.from_lattice(g["ops_q"])
    R = euler.nonlinear_rhs(dev(q), ref, disc, "set2nc").cpu().numpy()
    print(name, "R", ["%.2e" % e for e in rel_fields(o.to_lattice(R), g["ops_R"])])
    L = euler.vertical_restriction(dev(q), ref, disc, "set2nc").cpu().numpy()
    print(name, "L", ["%.2e" % e for e in rel_fields(o.to_lattice(L), g["ops_L"])])
    p = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", dim="1d", solver=imexcore.SolverSpec(method="direct")); p.lam = float(g["ops_lam"])
    S = p.solve(dev(q)).cpu().numpy()
    print(name, "S", ["%.2e" % e for e in rel_fields(o.to_lattice(S), g["ops_solve"])])
    qq = dev(o.from_lattice(g["step_q0"])); dt = float(g["step_dt"]); qo = o.from_lattice(g["step_q0"])
    keep = sorted(int(k[6:]) for k in g.files if k.startswith("step_q") and k != "step_q0")
    rhs = euler.make_rhs(ref, disc, "set2nc"); tab = imexcore.ark2_tableau()
    for k in range(1, keep[-1]+1):
        qq = imexcore.ark_imex_step(qq, dt, tab, p, rhs)
        if k in keep:
            print(name, "step", k, "vs ref", ["%.2e" % e for e in rel_fields(o.to_lattice(qq.cpu().numpy()), g[f"step_q{k}"])])
