"""Isolate the weight-update error: per-layer dW relative error for a grid
of (dims, batch, n_iters) training jobs."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import numpy as np
from oracle import layers as OL, scheduler as OS
from paper_1902_04610_b200 import build, salus as S
from workloads import TRAIN, make_job
from gpu_helpers import normwise_rel
build.build()
cases = [((128, 128, 128), 128, 1), ((128, 128, 128), 1024, 1), ((128, 256, 128), 128, 1),
         ((256, 256, 256), 128, 1), ((256, 256, 256), 1024, 1), ((256, 256, 256), 128, 3),
         ((256, 256, 256), 256, 1), ((256, 256, 256), 512, 1), ((128, 128), 128, 1), ((128, 128, 128, 128), 128, 1)]
for dims, B, n in cases:
    j = make_job(0, TRAIN, 0, dims, B, n, lr=1e-2, seed=5)
    ctx = S.Context([j], 1 << 30, S.PACK, dump={0: S.DUMP_OUTPUTS | S.DUMP_WEIGHTS})
    ctx.run()
    outs, W = OL.run_job(j)
    W0 = OL.init_weights(j)
    flat = ctx.layers(0, S.WEIGHTS)
    off, rels = 0, []
    for l in range(len(dims) - 1):
        m = dims[l] * dims[l + 1]
        Wg = flat[off:off + m].reshape(dims[l], dims[l + 1]); off += m
        d_g, d_r = Wg - W0[l], W[l] - W0[l]
        rels.append(normwise_rel(d_g, d_r))
        if l == 0 and rels[-1] > 0.02:
            # where is the error? per row-block / col-block
            e = np.abs(d_g - d_r) / np.max(np.abs(d_r))
            rb = [float(e[r:r + 64].max()) for r in range(0, dims[0], 64)]
            cb = [float(e[:, c:c + 64].max()) for c in range(0, dims[1], 64)]
            print("   err by 64-row block", np.round(rb, 3), "by 64-col block", np.round(cb, 3))
            ratio = np.sum(d_g * d_r) / np.sum(d_r * d_r)
            print("   projection ratio g/r:", round(float(ratio), 4))
    out_rel = max(normwise_rel(ctx.layers(0, k).reshape(B, -1), outs[k]) for k in range(n))
    print(dims, B, n, "out", f"{out_rel:.2e}", "dW", [f"{r:.2e}" for r in rels], flush=True)
    ctx.close()
