import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import test_gpu_fullsize as t
mesh, q0, q, run, _ = t.cfg5_run.__wrapped__()
for axis, odd in ((3, 1), (2, 2)):
    m = q.flip(axis)
    print("mirror", axis, ["%.1e" % t.rel(q[f], -m[f] if f == odd else m[f]) for f in range(5)])
tq = q.transpose(2, 3)
print("transpose", ["%.1e" % t.rel(q[f], tq[g]) for f, g in ((0, 0), (1, 2), (2, 1), (3, 3), (4, 4))])
print("max|u|", float(q[1].abs().max()), "max|w|", float(q[3].abs().max()))
