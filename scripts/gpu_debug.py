"""Staged first-contact checks on the GPU box (prints progress so a hang is localised)."""
import os, sys, time, ctypes
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np, torch
import lramm_oracle as O

def step(name):
    print(f"[{time.strftime('%H:%M:%S')}] {name}", flush=True)

step("import"); import paper_2405_16917_b200 as L; from paper_2405_16917_b200 import kernels, _native as N
print(torch.cuda.get_device_name(0), flush=True)
step("quantize"); x = O.generate(33, 47, "normal", 1); q = L.quantize(x, 8); d, s = O.quantize_tensor(x, 8)
print("quantize exact:", np.array_equal(q.data, d), q.scale == s, flush=True)
step("imatmul small"); rng = np.random.default_rng(0)
a = rng.integers(-127, 128, size=(19, 31)).astype(np.int32); b = rng.integers(-127, 128, size=(31, 11)).astype(np.int32)
out = kernels.imatmul(a, b); print("imatmul exact:", np.array_equal(out, a.astype(np.int64) @ b), flush=True)
step("imatmul 300x272x4096"); a = rng.integers(-127, 128, size=(300, 4096)).astype(np.int32); b = rng.integers(-127, 128, size=(4096, 272)).astype(np.int32)
out = kernels.imatmul(a, b); print("imatmul exact:", np.array_equal(out, a.astype(np.int64) @ b), flush=True)
step("qgemm"); a = O.generate(21, 35, "uniform", 1); b = O.generate(35, 17, "normal", 2)
print("qgemm bitwise:", np.array_equal(L.qgemm(a, b, 8, 8), O.qgemm(a, b, 8, 8)), flush=True)
step("matmul"); a = O.generate(300, 700, "normal", 1); b = O.generate(700, 129, "normal", 2)
print("dgemm maxerr:", np.max(np.abs(kernels.matmul(a, b) - a @ b)), flush=True)
step("qr"); from paper_2405_16917_b200.rsvd import _qr_device
y = O.generate(1000, 74, "normal", 3); qq = _qr_device(torch.from_numpy(y).cuda()).cpu().numpy()
print("qr orth:", np.linalg.norm(qq.T @ qq - np.eye(74)), flush=True)
for shape in [(20, 20), (300, 74), (1000, 138), (4096, 272)]:
    step(f"svd {shape}"); a = O.generate(*shape, "normal", 5); u, s, v = kernels.svd(a)
    print("svd serr:", np.max(np.abs(s - np.linalg.svd(a, compute_uv=False))) / s[0], "rec:", np.linalg.norm(a - (u*s)@v.T)/np.linalg.norm(a), flush=True)
step("lramm small parity")
a = O.synth(256, 192, "exp:16", 1, 0, 0); b = O.synth(192, 224, "exp:16", 1, 0, 1)
kw = dict(rank=24, bits=(8, 8, 8), power_iters=1, oversample=8, seed=0)
dd, t = L.lramm(a, b, L.LrammParams(**kw)); ref = O.lramm(a, b, O.OracleParams(**kw))
print("lramm parity rel:", O.rel_fro(dd, ref), t.wall_ns, flush=True)
step("lramm small fast/row")
dd, t = L.lramm(a, b, L.LrammParams(**kw, mode="fast", sketch_bits=8, power_bits=8, proj_bits=8, granularity="row"))
ref = O.lramm(a, b, O.OracleParams(**kw, spec=O.SketchSpec(8, 8, 8, "row")))
print("lramm fast rel:", O.rel_fro(dd, ref), t.wall_ns, flush=True)
step("lramm c2 fast/row timing")
a = np.random.default_rng(1).standard_normal((4096, 4096)).astype(np.float32); b = np.random.default_rng(2).standard_normal((4096, 4096)).astype(np.float32)
p = L.LrammParams(rank=256, bits=(8, 8, 8), power_iters=1, oversample=16, seed=0, mode="fast", sketch_bits=8, power_bits=8, proj_bits=8, granularity="row")
ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
for i in range(3):
    dd, t = L.lramm(ta, tb, p); torch.cuda.synchronize(); print({k: v/1e6 for k, v in t.wall_ns.items()}, flush=True)
step("done")
