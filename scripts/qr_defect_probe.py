"""max|Q1^T Q1 - I| after one fp64 CholeskyQR pass on the c3 range-finder sketches (decides whether
the closed-form second pass applies)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"])
dev = torch.device("cuda")
a, _ = bench.synth_pair(cfg, 0, dev)
a = a.double()
w = cfg["rank"] + cfg["oversample"]
g = torch.Generator(device=dev).manual_seed(1)
om = torch.randn(a.shape[1], w, generator=g, device=dev, dtype=torch.float64)

def cholqr1(y):
    l = torch.linalg.cholesky(y.T @ y)
    q = torch.linalg.solve_triangular(l, y.T, upper=False).T
    e = (q.T @ q - torch.eye(w, device=dev, dtype=torch.float64)).abs().max().item()
    d = torch.diagonal(l)
    return q, e, (d.max() / d.min()).item() ** 2 * 2.22e-16

y = a @ om
q, e, est = cholqr1(y)
print(f"Y0: max|E| {e:.2e}  estimate {est:.2e}")
for it in range(cfg["power_iters"]):
    q, _ = torch.linalg.qr(y)
    z = a.T @ q
    _, e, est = cholqr1(z)
    print(f"Z{it}: max|E| {e:.2e}  estimate {est:.2e}")
    qz, _ = torch.linalg.qr(z)
    y = a @ qz
    _, e, est = cholqr1(y)
    print(f"Y{it+1}: max|E| {e:.2e}  estimate {est:.2e}")
q, _ = torch.linalg.qr(y)
bs = (q.T @ a).T
_, e, est = cholqr1(bs)
print(f"Bs^T: max|E| {e:.2e}  estimate {est:.2e}")
