"""Pins for oracle/layers.py and oracle/datagen.py: published splitmix64
test vectors, bf16 rounding cases worked by hand, finite differences of the
loss (independent of the backward formulas), closed forms for special
cases (identity weights, one linear layer, lr = 0)."""
import numpy as np
import pytest

from oracle import datagen as DG
from oracle import layers as LY
from workloads import TRAIN, INFER, make_job


def test_splitmix64_published_vectors():
    # SplittableRandom / splitmix64 reference outputs for state 0, 1*gamma, 2*gamma
    # (Vigna, "splitmix64.c"; the sequence x += 0x9E3779B97F4A7C15 from x = 0).
    out = DG.splitmix64(np.array([0, 0x9E3779B97F4A7C15, (2 * 0x9E3779B97F4A7C15) % 2**64],
                                 dtype=np.uint64))
    assert [int(v) for v in out] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_bf16_rne_cases():
    v = np.array([1.0, 1 + 2**-8, 1 + 3 * 2**-8, -1 - 2**-8, 1 + 2**-7, 3.0e38, 2**-130],
                 dtype=np.float32)
    exp = [1.0, 1.0, 1 + 2**-6, -1.0, 1 + 2**-7, None, None]
    got = DG.bf16_rne(v)
    for g, e in zip(got[:5], exp[:5]):
        assert g == np.float32(e)
    # every output is bf16-representable: low 16 bits clear
    assert np.all((got.view(np.uint32) & 0xFFFF) == 0)


def test_gen_distribution_and_determinism():
    s = DG.scale_for(256)
    a = DG.gen(7, 3, DG.KIND_W, 1, 0, 256, 256, s)
    b = DG.gen(7, 3, DG.KIND_W, 1, 0, 256, 256, s)
    c = DG.gen(7, 4, DG.KIND_W, 1, 0, 256, 256, s)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert np.all(np.abs(a) <= float(s)) and a.dtype == np.float64
    assert abs(a.mean()) < 0.01 * float(s)
    assert abs(a.var() / float(s) ** 2 - 1.0 / 3.0) < 0.01      # U(-1,1) variance
    assert np.all(DG.bf16_rne(a.astype(np.float32)) == a.astype(np.float32))
    # element idx = row * cols + col of the logical tensor
    flat = DG.gen(7, 3, DG.KIND_W, 1, 0, 1, 256 * 256, s).reshape(256, 256)
    assert np.array_equal(flat, a)


def test_gen_pair_streams_are_independent_uniform():
    """A29: one splitmix64 value feeds an element pair (bits 40-63 -> even
    index, bits 16-39 -> odd).  Both streams must be U(-1,1) and the two
    halves of a pair uncorrelated, and the pairing must follow the flat
    index, not the row (odd row length)."""
    a = DG.gen(11, 5, DG.KIND_X, 0, 3, 1, 1 << 18, 1.0).ravel()
    ev, od = a[0::2], a[1::2]
    for st in (ev, od):
        assert abs(st.mean()) < 0.01 and abs(st.var() - 1.0 / 3.0) < 0.01
        h, _ = np.histogram(st, bins=16, range=(-1, 1))
        assert h.min() > 0.9 * len(st) / 16
    assert abs(np.corrcoef(ev, od)[0, 1]) < 0.01
    odd = DG.gen(11, 5, DG.KIND_X, 0, 3, 3, 7, 1.0)          # 21 elements, rows of 7
    assert np.array_equal(odd.ravel(), DG.gen(11, 5, DG.KIND_X, 0, 3, 1, 21, 1.0).ravel())


def _tiny_job(dims, B, kind=TRAIN, lr=0.05):
    return make_job(0, kind, 0, dims, B, 3, lr=lr, seed=9, request_ticks=(0, 1, 2) if kind else ())


@pytest.mark.parametrize("dims", [(5, 4, 3), (6, 7, 5, 4), (3, 2)])
def test_gradients_match_finite_differences(dims):
    job = _tiny_job(dims, 4)
    W = LY.init_weights(job)
    X, T = LY.inputs(job, 0)
    X = X * 3.0
    _, dW = LY.gradients(W, X, T)
    eps = 1e-6
    for l, Wl in enumerate(W):
        num = np.zeros_like(Wl)
        for idx in np.ndindex(Wl.shape):
            Wp = [w.copy() for w in W]
            Wm = [w.copy() for w in W]
            Wp[l][idx] += eps
            Wm[l][idx] -= eps
            num[idx] = (LY.loss(Wp, X, T) - LY.loss(Wm, X, T)) / (2 * eps)
        assert np.max(np.abs(num - dW[l])) <= 1e-6 * max(1.0, np.max(np.abs(num))), l


def test_one_linear_layer_closed_form():
    """L = 1: textbook least squares gradient X^T (X W - T) / B."""
    job = _tiny_job((8, 5), 6)
    W = LY.init_weights(job)
    X, T = LY.inputs(job, 0)
    _, dW = LY.gradients(W, X, T)
    assert np.allclose(dW[0], X.T @ (X @ W[0] - T) / 6, rtol=0, atol=1e-14)


def test_identity_weights_give_relu():
    """W_1 = W_2 = I  =>  A_2 = ReLU(X) (A_L has no ReLU; A_1 does)."""
    X = np.array([[1.0, -2.0, 0.5], [-0.25, 3.0, -1.0]])
    A = LY.forward([np.eye(3), np.eye(3)], X)
    assert np.array_equal(A[-1], np.maximum(X, 0))


def test_lr_zero_keeps_weights():
    job = _tiny_job((16, 8, 4), 5, lr=0.0)
    outs, W = LY.run_job(job)
    W0 = LY.init_weights(job)
    assert all(np.array_equal(a, b) for a, b in zip(W, W0))


def test_sgd_step_is_minus_lr_grad_and_reduces_loss_on_fixed_batch():
    job = _tiny_job((16, 12, 4), 8, lr=0.1)
    W = LY.init_weights(job)
    X, T = LY.inputs(job, 0)
    before = LY.loss(W, X, T)
    W0 = [w.copy() for w in W]
    _, dW = LY.gradients(W, X, T)
    LY.train_step(W, job, 0)
    for a, b, g in zip(W, W0, dW):
        assert np.allclose(a, b - np.float32(0.1) * g, rtol=0, atol=1e-15)
    assert LY.loss(W, X, T) < before


def test_inference_is_forward_of_init_weights():
    job = _tiny_job((16, 8, 4), 2, kind=INFER)
    outs, W = LY.run_job(job)
    X1, _ = LY.inputs(job, 1)
    assert np.array_equal(outs[1], LY.forward(LY.init_weights(job), X1)[-1])


def test_bf16_storage_mode_rounds_exactly_the_stored_tensors():
    """Reading A31: store=bf16 rounds W copies, A_l (l>=1) and G_l to bf16;
    Z_L and the master weights stay fp64."""
    job = _tiny_job((16, 12, 8, 4), 6, lr=0.1)
    W = LY.init_weights(job)
    X, T = LY.inputs(job, 0)
    A = LY.forward(W, X, LY.bf16)
    for a in A[1:-1]:
        assert np.array_equal(LY.bf16(a), a)
    assert not np.array_equal(LY.bf16(A[-1]), A[-1])         # Z_L unrounded
    # same structure as the fp64 definition: with identity rounding equal
    A64 = LY.forward(W, X)
    assert all(np.allclose(a, b, rtol=2e-2, atol=1e-2) for a, b in zip(A, A64))
    _, dW16 = LY.gradients(W, X, T, LY.bf16)
    _, dW64 = LY.gradients(W, X, T)
    for a, b in zip(dW16, dW64):
        assert np.max(np.abs(a - b)) <= 0.2 * np.max(np.abs(b))


def test_bf16_storage_equals_fp64_when_everything_is_representable():
    """One layer: X, W are bf16-exact, so forward and dW differ only by the
    bf16 rounding of G_L."""
    job = _tiny_job((8, 4), 5, lr=0.0)
    W = LY.init_weights(job)
    X, T = LY.inputs(job, 0)
    assert np.array_equal(LY.forward(W, X, LY.bf16)[-1], LY.forward(W, X)[-1])
    _, d16 = LY.gradients(W, X, T, LY.bf16)
    assert np.array_equal(d16[0], X.T @ LY.bf16((X @ W[0] - T) / 5))


def test_bf16_storage_mask_flip_hand_worked():
    """Reading A31 pinned by a 3-layer example worked by hand (exact binary
    fractions), in which storing A_1 in bf16 flips the ReLU mask of layer 2.

      dims (2, 2, 1, 1), B = 1, X = [1+2^-7, 1], T = [1], lr = 1/2
      W_1 = diag(1+2^-7, 1+2^-6),  W_2 = [1, -1]^T,  W_3 = [1+2^-9]

    fp64:  Z_1 = [1+2^-6+2^-14, 1+2^-6],  Z_2 = 2^-14 > 0,  A_3 = 2^-14 (1+2^-9),
           G_3 = A_3 - 1,  G_2 = G_3 (1+2^-9),  G_1 = [G_2, -G_2]
    bf16:  A_1 = bf16(Z_1) = [1+2^-6, 1+2^-6] (2^-14 is below half an ulp),
           Z_2 = 0 -> mask [A_2 > 0] = 0;  the W_3 copy is bf16(1+2^-9) = 1,
           so A_3 = 0, G_3 = -1 and every other gradient is 0: the step
           leaves W_1, W_2, W_3 unchanged (the fp64 master is untouched).
    Fails if the activation storage rounding, the weight-copy rounding or
    the mask placement of the bf16 mode were dropped or moved."""
    from fractions import Fraction as F
    u7, u6, u9, u14 = F(1, 2**7), F(1, 2**6), F(1, 2**9), F(1, 2**14)
    X = np.array([[float(1 + u7), 1.0]])
    T = np.array([[1.0]])
    W = [np.diag([float(1 + u7), float(1 + u6)]), np.array([[1.0], [-1.0]]), np.array([[float(1 + u9)]])]
    # fp64 definition
    A, dW = LY.gradients(W, X, T)
    z1 = [(1 + u7) ** 2, 1 + u6]
    a3 = u14 * (1 + u9)
    g3 = a3 - 1
    g2 = g3 * (1 + u9)
    exp_dW = [[[(1 + u7) * g2, -(1 + u7) * g2], [g2, -g2]], [[z1[0] * g2], [z1[1] * g2]], [[u14 * g3]]]
    assert [float(x) for x in A[1].ravel()] == [float(z) for z in z1]
    assert float(A[2][0, 0]) == float(u14) and float(A[3][0, 0]) == float(a3)
    for got, exp in zip(dW, exp_dW):
        e = np.array([[float(v) for v in row] for row in exp])
        assert np.allclose(got, e, rtol=1e-15, atol=0), (got, e)
    # bf16-storage mode: the mask flips and every update vanishes
    A16, dW16 = LY.gradients(W, X, T, LY.bf16)
    assert list(A16[1].ravel()) == [float(1 + u6)] * 2
    assert A16[2][0, 0] == 0.0 and A16[3][0, 0] == 0.0
    assert all(np.all(d == 0.0) for d in dW16)
    job = make_job(0, TRAIN, 0, (2, 2, 1, 1), 1, 1, lr=0.5)
    W16 = [w.copy() for w in W]
    _, d16 = LY.gradients(W16, X, T, LY.bf16)
    for w, d in zip(W16, d16):
        w -= np.float32(job.lr) * d
    assert all(np.array_equal(a, b) for a, b in zip(W16, W))
    # fp64 step moves W_1 by -lr * dW_1 exactly
    assert float(W[0][0, 0] - 0.5 * dW[0][0, 0]) == float(1 + u7 - F(1, 2) * (1 + u7) * g2)
