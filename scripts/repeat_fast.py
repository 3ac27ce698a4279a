"""Repeat the fast-mode restatement check to expose nondeterminism."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import lramm_oracle as O
import paper_2405_16917_b200 as L
gran = sys.argv[1] if len(sys.argv) > 1 else "tensor"
a = O.synth(512, 512, "exp:24", 7, 0, 0)
b = O.synth(512, 512, "exp:24", 7, 0, 1)
kw = dict(rank=32, bits=(8, 8, 8), power_iters=1, oversample=8, seed=5)
ref = O.lramm(a, b, O.OracleParams(**kw, spec=O.SketchSpec(8, 8, 8, gran)))
outs = []
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    d, _ = L.lramm(a, b, L.LrammParams(**kw, mode="fast", sketch_bits=8, power_bits=8, proj_bits=8, granularity=gran))
    outs.append(d.copy())
    print(i, O.rel_fro(d, ref), "identical to first" if np.array_equal(d, outs[0]) else "DIFFERS from first")
