"""ORACLE — test infrastructure only.  fp64 dense-MLP iteration math.

Each dispatched iteration (DISPATCH record (job j, iteration k)) executes one
training step or one inference request of job j.  The paper's jobs are
"a stack of nonlinear processing layers" trained by "alternating between
forward and backward passes" that update "model parameters" (§2.1
P:88-104); its models are unavailable, so each job is a dense MLP with ReLU
hidden layers, MSE loss and plain SGD (SURVEY §8(c) "Math per DISPATCH"):

    X, T = gen(j, k);  A_0 = X
    Z_l = A_{l-1} W_l;  A_l = ReLU(Z_l) (l < L),  A_L = Z_L
    TRAIN:  G_L = (A_L - T) / B          (gradient of 1/(2B) * ||A_L - T||^2)
            for l = L..1:
                dW_l = A_{l-1}^T G_l
                G_{l-1} = (G_l W_l^T) * [A_{l-1} > 0]     (l > 1, pre-update W_l)
                W_l -= lr * dW_l

Plain numpy float64; `@` (a library matmul) is the only primitive used.

Precision modes (reading A31).  `store=None` is the definition
above in fp64.  The ReLU mask [A > 0] is a floating-point value deciding an
integer (0/1); by the parity rules both sides must take that decision in the
same precision, the kernel's.  `store=bf16` therefore rounds (fp64 -> fp32 ->
bf16, round-to-nearest-even) exactly the tensors the kernel keeps in bf16:
the weight copy used by the GEMMs, A_l for l >= 1, and every G_l; the master
weights, Z_l and all sums stay fp64.  Nothing else changes.
"""
from typing import Callable, List, Optional

import numpy as np

from . import datagen as DG

TRAIN, INFER = 0, 1


def bf16(x: np.ndarray) -> np.ndarray:
    """Storage rounding of the kernel: fp64 -> fp32 (RNE) -> bf16 (RNE)."""
    return DG.bf16_rne(np.asarray(x, dtype=np.float64).astype(np.float32)).astype(np.float64)


def _ident(x):
    return x


def init_weights(job) -> List[np.ndarray]:
    """W_l (d_{l-1} x d_l), element (i, j) at idx = i * d_l + j."""
    d = job.dims
    return [DG.gen(job.seed, job.job_id, DG.KIND_W, l, 0, d[l - 1], d[l], DG.scale_for(d[l - 1]))
            for l in range(1, len(d))]


def inputs(job, k: int):
    d = job.dims
    X = DG.gen(job.seed, job.job_id, DG.KIND_X, 0, k, job.batch, d[0], np.float32(1.0))
    T = DG.gen(job.seed, job.job_id, DG.KIND_T, len(d) - 1, k, job.batch, d[-1], np.float32(1.0))
    return X, T


def forward(W: List[np.ndarray], X: np.ndarray, store: Optional[Callable] = None) -> List[np.ndarray]:
    rnd = store or _ident
    A = [X]
    L = len(W)
    for l in range(1, L + 1):
        Z = A[l - 1] @ rnd(W[l - 1])
        A.append(rnd(np.maximum(Z, 0.0)) if l < L else Z)
    return A


def loss(W, X, T) -> float:
    A = forward(W, X)
    return float(0.5 / X.shape[0] * np.sum((A[-1] - T) ** 2))


def gradients(W: List[np.ndarray], X: np.ndarray, T: np.ndarray, store: Optional[Callable] = None):
    """Returns (A list, [dW_1..dW_L]) for the loss 1/(2B)||A_L - T||^2."""
    rnd = store or _ident
    A = forward(W, X, store)
    L = len(W)
    B = X.shape[0]
    G = rnd((A[L] - T) / B)
    dW = [None] * L
    for l in range(L, 0, -1):
        dW[l - 1] = A[l - 1].T @ G
        if l > 1:
            G = rnd((G @ rnd(W[l - 1]).T) * (A[l - 1] > 0))
    return A, dW


def train_step(W: List[np.ndarray], job, k: int, store: Optional[Callable] = None) -> np.ndarray:
    """One SGD iteration in place; returns the output A_L (B x d_L)."""
    X, T = inputs(job, k)
    A, dW = gradients(W, X, T, store)
    lr = float(np.float32(job.lr))
    for l in range(len(W)):
        W[l] -= lr * dW[l]
    return A[-1]


def infer_step(W: List[np.ndarray], job, k: int, store: Optional[Callable] = None) -> np.ndarray:
    X, _ = inputs(job, k)
    return forward(W, X, store)[-1]


def run_job(job, iters=None, store: Optional[Callable] = None):
    """Run iterations 0..n-1 (or the listed prefix) of one job.

    Returns (outputs {k: A_L}, final weights)."""
    W = init_weights(job)
    n = job.n_iters if iters is None else iters
    outs = {}
    for k in range(n):
        outs[k] = train_step(W, job, k, store) if job.kind == TRAIN else infer_step(W, job, k, store)
    return outs, W
