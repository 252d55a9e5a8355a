"""Stage-1 local-update phase time (u1 estimator moments + quadratic update)
vs query-set size: the fused / persistent moments crossover
(UCP_FUSED_MAX_QUERIES=0 forces the persistent kernel, a large value the fused one).

    python tools/moments_sweep.py [d ...]
"""
import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1908_04489_b200 as P
for d in [int(x) for x in sys.argv[1:]] or (8192, 14000, 20000, 32768, 65536):
    p = P.Witsenhausen(grids=[(-25.0, 25.0, d)] * 2)
    rng = np.random.default_rng(0)
    U = P.ControllerSet(tuple(P.SampledController(g, g.points * 0.3 + rng.uniform(-0.1, 0.1, g.d)) for g in p.grids))
    cfg = P.SolverConfig()
    p.device_local_update(1, U, cfg); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): p.device_local_update(1, U, cfg)
    b.record(); torch.cuda.synchronize()
    print(d, round(a.elapsed_time(b) / 5 * 1e3, 1), "us")
