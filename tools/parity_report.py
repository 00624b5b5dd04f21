"""Parity table of the CUDA path (run on a B200): per case, relative L2 errors
(rho', |vel|, theta') of R, L_V, the Schur solve and 10 ARK2 steps against the
reference goldens and against the oracle with cancellation-free P'
(pprime="exact").  Output goes to stdout; profiles/parity_r01.txt keeps a copy."""
import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from conftest import CASES, load_golden, oracle_for, rel_fields, set_of  # noqa: E402
from test_gpu_parity import build, dev  # noqa: E402
from paper_1702_04316_b200 import euler, imexcore  # noqa: E402


def fmt(e):
    return "[" + ", ".join("%.1e" % x for x in e) + "]"


print("case            set     quantity       vs reference golden        vs exact-P' oracle")
for name in sorted(CASES):
    sn = set_of(name)
    mesh, ref, disc = build(name)
    o, ox, g = oracle_for(name), oracle_for(name, "exact"), load_golden(name)
    q = o.from_lattice(g["ops_q"])
    lam = float(g["ops_lam"])
    p = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name=sn, dim="1d",
                                 solver=imexcore.SolverSpec(method="direct"))
    p.lam = lam
    rows = [
        ("R", euler.nonlinear_rhs(dev(q), ref, disc, sn), g["ops_R"], ox.rhs(q)),
        ("L_V", euler.vertical_restriction(dev(q), ref, disc, sn), g["ops_L"], ox.linear(q)),
        ("solve", p.solve(dev(q)), g["ops_solve"], ox.solve(q, lam)),
    ]
    for tag, got, want, wx in rows:
        got = o.to_lattice(got.cpu().numpy())
        print(f"{name:15s} {sn:7s} {tag:14s} {fmt(rel_fields(got, want)):26s} "
              f"{fmt(rel_fields(got, ox.to_lattice(wx)))}")
    q0 = o.from_lattice(g["step_q0"])
    qq, qx = dev(q0), q0.copy()
    dt = float(g["step_dt"])
    rhs = euler.make_rhs(ref, disc, sn)
    tab = imexcore.ark2_tableau()
    for k in range(1, 11):
        qq = imexcore.ark_imex_step(qq, dt, tab, p, rhs)
        qx = ox.step(qx, dt)
        if f"step_q{k}" in g.files:
            got = o.to_lattice(qq.cpu().numpy())
            print(f"{name:15s} {sn:7s} {'step %d' % k:14s} "
                  f"{fmt(rel_fields(got, g[f'step_q{k}'])):26s} "
                  f"{fmt(rel_fields(got, ox.to_lattice(qx)))}")
