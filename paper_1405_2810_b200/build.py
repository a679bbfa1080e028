"""Build liblrbms.so in-tree for sm_100a (nvcc; no JIT cache, the .so travels with the repo)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "liblrbms.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("lrbms.cu", "lrbms_kernels.cuh", "lrbms_pcg.cuh", "lrbms_project.cuh", "lrbms_ns.cuh", "lrbms_pcg_tm.cuh", "lrbms_affine.cuh", "lrbms_fine.cuh", "lrbms_diag.cuh", "lrbms_transport.cuh", "lrbms_offline.cuh", "lrbms_k1.cuh")]
HEADERS = [os.path.join(ROOT, "include", "lrbms.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


def nvcc():
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(p) > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        cmd = [nvcc()] + NVCC_FLAGS + (["-Xptxas", "-v"] if verbose else []) + \
              ["-o", SO, os.path.join(HERE, "csrc", "lrbms.cu")]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building liblrbms.so")
        if verbose:
            sys.stderr.write(r.stderr)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
