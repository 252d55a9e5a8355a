"""Two rounds of a config-5 solve (ZeroDelay d=16384 or Inventory M=3
d=4096): the target program for ncu captures of the uniform-noise kernels.

    ncu --set full -k regex:k_unif_moments_points -s 30 -c 1 python tools/c5_one_solve.py zd
    ncu --set full -k regex:k_unif_propagate -s 60 -c 1 python tools/c5_one_solve.py inv
"""
import sys, torch
sys.path.insert(0, ".")
import paper_1908_04489_b200 as P
case = sys.argv[1]
if case == "zd":
    prob = P.ZeroDelay(grids=[(-5.0, 5.0, 16384), (-6.0, 6.0, 16384)])
else:
    prob = P.Inventory(stages=3, grids=[(-3.0, 3.0, 4096)] * 3)
P.solve(prob, P.SolverConfig(max_rounds=2))
torch.cuda.synchronize()
