"""Diagnose one math case: GPU vs fp64 and bf16-storage oracles, per layer,
Frobenius and max-normwise, for n = 1..N iterations."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from oracle import layers as OL
from paper_1902_04610_b200 import build, salus as S
from workloads import TRAIN, make_job
build.build()
dims = tuple(int(x) for x in sys.argv[1].split(","))
B = int(sys.argv[2]); lr = float(sys.argv[3]); seed = int(sys.argv[4])
for n in (1, 2, 3):
    j = make_job(1, TRAIN, 0, dims, B, n, lr=lr, seed=seed)
    ctx = S.Context([j], 1 << 30, S.PACK, dump={1: S.DUMP_OUTPUTS | S.DUMP_WEIGHTS})
    ctx.run()
    W0 = OL.init_weights(j)
    _, W64 = OL.run_job(j)
    _, W16 = OL.run_job(j, store=OL.bf16)
    flat = ctx.layers(1, S.WEIGHTS); off = 0
    for l in range(len(dims) - 1):
        m = dims[l] * dims[l + 1]
        Wg = flat[off:off + m].reshape(dims[l], dims[l + 1]); off += m
        dg, d16, d64 = Wg - W0[l], W16[l] - W0[l], W64[l] - W0[l]
        fro = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
        mx = lambda a, b: np.max(np.abs(a - b)) / np.max(np.abs(b))
        print(f"n={n} layer {l}: gpu-vs-bf16 fro {fro(dg, d16):.2e} max {mx(dg, d16):.2e} | gpu-vs-64 fro {fro(dg, d64):.2e} | bf16-vs-64 fro {fro(d16, d64):.2e}")
    ctx.close()
