import sys, torch, time
sys.path.insert(0, '/root/repo')
import paper_1908_04489_b200 as P
x = torch.rand(1 << 20, dtype=torch.float64, device='cuda')
P.kernels.trapezoid_sum(x, 1e-3)
for lib in [0]:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): P.kernels.trapezoid_sum(x, 1e-3)
    e1.record(); torch.cuda.synchronize()
    print("trapezoid 2^20 ms", e0.elapsed_time(e1) / 5)
