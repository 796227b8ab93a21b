"""Build libsalus.so in-tree with nvcc for sm_100a (no JIT cache: the .so
travels to the GPU box with the repo snapshot)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsalus.so")
# the opt-in split-K build: SALUS_LIB=<this> and SALUS_SPLITK=1
LIB_SPLITK = os.path.join(HERE, "libsalus_splitk.so")
SOURCES = ["salus_kernel.cu", "salus_host.cpp"]
HEADERS = ["salus_dev.h", "ptx.cuh", "datagen.cuh", "scheduler.cuh", "worker.cuh", "runahead.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "salus.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or _stale():
        cmd = [NVCC] + FLAGS + ["-o", LIB] + SOURCES
        r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libsalus.so")
        if verbose:
            sys.stderr.write(r.stderr)
    return LIB


def build_splitk(force: bool = False) -> str:
    """The opt-in split-K library (SALUS_SPLITK_BUILD=1), in-tree."""
    if force or _stale(LIB_SPLITK):
        build_variant(LIB_SPLITK, ["SALUS_SPLITK_BUILD=1"])
    return LIB_SPLITK


def build_variant(out: str, defines) -> str:
    """Experiment builds (compile-time ablations) into a separate .so."""
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    cmd = [NVCC] + FLAGS + ["-D" + d for d in defines] + ["-o", os.path.abspath(out)] + SOURCES
    r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building " + out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
