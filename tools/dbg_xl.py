import sys, numpy as np
sys.path.insert(0, '/root/repo')
from synth import corpus as sc
from paper_1704_07468_b200 import gakco as gk
import oracle
oracle.build()
rng = np.random.default_rng(108)
for it in range(10):
    sigma = int(rng.choice([2, 4, 20, 36]))
    g = int(rng.integers(2, 11))
    k = int(rng.integers(1, g + 1))
    M = int(rng.integers(0, g + 1))
    cp = sc.random_small(rng, sigma, n_max=200, l_max=300)
    ref = oracle.compute(cp, g, k, M)
    for mode in (6,):
        plan = gk.Plan(cp.sigma, g, k, M)
        plan.set_option(gk.GAKCO_OPT_SORT, mode)
        r = gk.kernel_matrix(cp.codes, cp.offsets, cp.sigma, g, k, M, plan=plan)
        C = r["C"].cpu().numpy(); st = plan.stats(); plan.close()
        bad = [m for m in range(M + 1) if not np.array_equal(C[m], ref["C"][m])]
        n = int(np.maximum(np.diff(cp.offsets) - g + 1, 0).sum())
        print(it, "sigma", sigma, "g", g, "k", k, "M", M, "N", cp.n_seq, "n", n, "bad", bad,
              [int(np.abs(C[m] - ref["C"][m]).sum()) for m in bad])
