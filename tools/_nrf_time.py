import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2603_00145_b200 import nrf as NR
rng = np.random.default_rng(0)
widths = (39, 64, 64, 64, 64, 1)
ws = [rng.uniform(-1, 1, (a, b)) * np.sqrt(6.0 / (a + b)) for a, b in zip(widths[:-1], widths[1:])]
bs = [rng.normal(0, 0.1, b) for b in widths[1:]]
f = NR.ResidualField.from_numpy(ws, bs)
for B in (8192, 131072):
    x = torch.rand(B, 3, device='cuda') * 2 - 1
    up = torch.randn(B, device='cuda')
    for name, fw, bw in (("torch", NR.nrf_forward_cached, NR.nrf_backward), ("fused", NR.nrf_forward_fused, NR.nrf_backward_fused)):
        for _ in range(3):
            r, c = fw(f, x); bw(f, x, up, c)
        torch.cuda.synchronize()
        e0, e1, e2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e0.record()
        for _ in range(20):
            r, c = fw(f, x)
        e1.record()
        for _ in range(20):
            bw(f, x, up, c)
        e2.record(); torch.cuda.synchronize()
        print(B, name, 'fwd %.3f ms bwd %.3f ms' % (e0.elapsed_time(e1)/20, e1.elapsed_time(e2)/20), flush=True)
