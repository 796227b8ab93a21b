"""ORACLE — test infrastructure only.  Counter-based synthetic data.

Real datasets and trained weights are unavailable, so
inputs X, targets T and initial weights W are a pure function of
(seed, job, tensor_id, element index):

    h  = splitmix64(splitmix64(splitmix64(seed) ^ job) ^ (tensor_id << 40 | idx >> 1))
    u  = b * 2^-24, b = h >> 40 for even idx, (h >> 16) & (2^24 - 1) for odd idx
                                                   (24 random bits, in [0,1); one
                                                    hash serves two elements)
    v  = fp32((2u - 1) * scale)                    (fp32 multiply, RNE)
    value = bf16_rne(v), held exactly as a wider float

with splitmix64(x) = mix(x + 0x9E3779B97F4A7C15) (Steele/Lea/Flood's
SplittableRandom finaliser), idx = row * d + col over the *unpadded* logical
tensor, and tensor_id = kind << 20 | layer << 16 | (iteration & 0xFFFF),
kind 0 = W, 1 = X, 2 = T.  scale = fp32(1/sqrt(d_in)) for W_l (d_in =
d_{l-1}), 1.0 for X and T.  The CUDA path implements the same written spec
independently; the two share no code.
"""
import numpy as np

KIND_W, KIND_X, KIND_T = 0, 1, 2
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x):
    """Vectorised splitmix64 over a uint64 array (wrapping arithmetic)."""
    z = np.asarray(x, dtype=np.uint64) + GOLDEN
    z = (z ^ (z >> np.uint64(30))) * M1
    z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def bf16_rne(v32: np.ndarray) -> np.ndarray:
    """Round fp32 to the nearest bf16 (ties to even); returns fp32 values."""
    b = np.asarray(v32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32)


def tensor_id(kind: int, layer: int, iteration: int) -> int:
    return (kind << 20) | (layer << 16) | (iteration & 0xFFFF)


def scale_for(d_in: int) -> np.float32:
    return np.float32(1.0 / np.sqrt(np.float64(d_in)))


def gen(seed: int, job: int, kind: int, layer: int, iteration: int, rows: int, cols: int,
        scale) -> np.ndarray:
    """A (rows x cols) float64 matrix of bf16-representable values."""
    with np.errstate(over="ignore"):
        s = splitmix64(np.array([seed], dtype=np.uint64))
        s = splitmix64(s ^ np.uint64(job))
        tid = np.uint64(tensor_id(kind, layer, iteration)) << np.uint64(40)
        idx = np.arange(rows * cols, dtype=np.uint64)
        h = splitmix64(s ^ (tid | (idx >> np.uint64(1))))
    bits = np.where((idx & np.uint64(1)) == 0, h >> np.uint64(40), (h >> np.uint64(16)) & np.uint64(0xFFFFFF))
    u = bits.astype(np.float32) * np.float32(2.0 ** -24)
    v = (np.float32(2.0) * u - np.float32(1.0)) * np.float32(scale)
    return bf16_rne(v.astype(np.float32)).astype(np.float64).reshape(rows, cols)
