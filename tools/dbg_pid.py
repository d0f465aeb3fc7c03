import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from oracle import core
from paper_2010_08454_b200 import models
import test_gpu_is as t
m = models.PolyRegression.synthetic()
for first in t.PID_WINDOWS:
    n = 100_000
    lw, deg, coef, rec = t._run_traced(m, n, t.KEY, first=first)
    _, (lw_ref, deg_ref, coef_ref) = core.is_poly(m.xs, m.ys, first, first + n, t.KEY, traces=True)
    err = np.abs(coef - coef_ref) / (1 + np.abs(coef_ref))
    i, j = np.unravel_index(np.argmax(err), err.shape)
    print(first, "deg equal", np.array_equal(deg, deg_ref), "max err", err.max(), "at", i, j, coef[i], coef_ref[i], deg[i], "n>1e-4:", (err > 1e-4).sum())
