import sys, numpy as np
sys.path.insert(0, '.')
from synth import corpus as sc
import oracle
from paper_1704_07468_b200 import gakco as gk
import torch
rng = np.random.default_rng(113)
cases = [(sc.gen_families(7, 90, 6, 60, 30, 60, sigma=20), 6, 3, 3),
         (sc.gen_families(8, 150, 10, 80, 80, 80, sigma=4), 8, 5, 3)]
for _ in range(4):
    sigma = int(rng.choice([2, 4, 20]))
    g = int(rng.integers(3, 9))
    k = int(rng.integers(1, g))
    cases.append((sc.random_small(rng, sigma, n_max=120, l_max=90), g, k, g - k))
for ci, (cp, g, k, M) in enumerate(cases):
    ref = oracle.compute(cp, g, k, M)
    N = cp.n_seq
    for rl in (0, 1):
        plan = gk.Plan(cp.sigma, g, k, M)
        plan.set_option(gk.GAKCO_OPT_LIGHT_RELABEL, rl)
        C = torch.zeros((M + 1, N, N), dtype=torch.int64, device='cuda')
        try:
            plan.accumulate(cp.codes, cp.offsets, N, C)
            torch.cuda.synchronize()
        except Exception as e:
            print('case', ci, 'relabel', rl, 'ERROR', e)
        Cu = np.triu(C.cpu().numpy())
        bad = []
        for m in range(M + 1):
            R = np.triu(ref['C'][m])
            d = np.argwhere(Cu[m] != R)
            if len(d): bad.append((m, len(d), d[:3].tolist(), [(int(Cu[m][i,j]), int(R[i,j])) for i,j in d[:3]]))
        print('case', ci, 'N', N, 'g,k,M', g, k, M, 'relabel', rl, 'bad', bad, flush=True)
        plan.close()
