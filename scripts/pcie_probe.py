"""PCIe probe: pinned H2D alone, D2H alone, both at once (two streams); 512 MiB each."""
import time
import torch

n = 512 << 20
h_up = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_dn = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_up = torch.empty(n, dtype=torch.uint8, device="cuda")
d_dn = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(up, dn, reps=5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if up:
            with torch.cuda.stream(s1):
                d_up.copy_(h_up, non_blocking=True)
        if dn:
            with torch.cuda.stream(s2):
                h_dn.copy_(d_dn, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


for _ in range(2):
    run(True, True)
a, b, c = run(True, False), run(False, True), run(True, True)
gb = n / 1e9
print(f"H2D alone {a*1e3:.2f} ms ({gb/a:.1f} GB/s)  D2H alone {b*1e3:.2f} ms ({gb/b:.1f} GB/s)  "
      f"both {c*1e3:.2f} ms ({gb/c:.1f} GB/s each way)")
