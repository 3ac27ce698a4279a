import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from test_gpu_omega import _device
n, w, seed = 4096, 272, 2**63 + 5
ref = np.random.Generator(np.random.Philox(np.random.SeedSequence([seed & 0xFFFFFFFFFFFFFFFF, 0x534B, n, w]))).standard_normal((n, w)).ravel()
got = _device(seed, n, w).ravel()
bad = np.nonzero(got != ref)[0]
print("mismatches", len(bad), "first", bad[:10])
for b in bad[:10]:
    print(b, repr(got[b]), repr(ref[b]), "ulps", abs(got[b].view(np.int64) - ref[b].view(np.int64)), "tail" if abs(ref[b]) > 3.654 else "")
