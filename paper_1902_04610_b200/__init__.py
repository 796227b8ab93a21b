"""B200-native Salus execution service (arXiv 1902.04610) — hot path only.

`salus` is the thin ctypes binding of libsalus.so (include/salus.h); the
CUDA kernels and the host library live in `csrc/`.
"""
