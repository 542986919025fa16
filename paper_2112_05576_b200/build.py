"""Build libedgealign_b200.so in-tree with nvcc for sm_100a (no JIT, no torch
extension cache: the .so travels to the GPU box with the repo snapshot).

    python -m paper_2112_05576_b200.build [--force]
"""
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libedgealign_b200.so")

CU_SOURCES = ["api.cu", "field_kernels.cu", "search_kernels.cu", "refine_kernels.cu",
              "model_kernels.cu"]
CPP_SOURCES = ["host_model.cpp", "host_synth.cpp", "host_io.cpp", "nccl_dl.cpp"]
HEADERS = ["common.cuh", "kernels.cuh", "refine.cuh", "model.cuh", "failure.h", "host_model.h",
           "nccl_dl.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
HOST_FLAGS = "-fPIC,-ffp-contract=off,-O2,-Wall"
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", HOST_FLAGS,
                     "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _deps():
    return [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "edgealign_b200.h")]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources if os.path.exists(s))


def _compile(src, force, log):
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src + ".o")
    if not force and not _stale(obj, [path] + _deps()):
        return obj
    if src.endswith(".cu"):
        cmd = [nvcc()] + NVCC_FLAGS + ["-c", path, "-o", obj]
    else:
        cmd = ["g++", "-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-Wall",
               "-I/usr/local/cuda/include", "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    with open(obj + ".log", "w") as f:
        f.write(r.stdout + r.stderr)
    if log:
        print(f"[build] {src}", file=sys.stderr)
    return obj


def build(force=False, log=True):
    os.makedirs(OBJ, exist_ok=True)
    srcs = CU_SOURCES + CPP_SOURCES
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, log), srcs))
    if force or _stale(LIB, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-lrt",
                                                                 "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if log:
            print(f"[build] -> {LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
