"""Build the in-tree C-ABI library libh2b200.so for sm_100a with nvcc (no JIT cache).

python -m paper_2109_05451_b200.build   (also called by __graft_entry__.build())
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libh2b200.so")
SOURCES = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.startswith("h2_k_") and f.endswith(".cu")) + \
    [os.path.join(CSRC, "h2_api.cpp"), os.path.join(CSRC, "h2_file.cpp"), os.path.join(CSRC, "h2_solver.cu")]
DEPS = SOURCES + sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))) + \
    [os.path.join(ROOT, "include", "h2.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_paths():
    import nvidia.nccl as nn
    base = os.path.dirname(nn.__file__) if getattr(nn, "__file__", None) else list(nn.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib", "libnccl.so.2")


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force=False, verbose=False):
    if not force and not needs_build():
        return LIB
    inc, ncclso = _nccl_paths()
    nvcc = os.environ.get("NVCC", "nvcc")
    objs = []
    common = ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I" + inc,
                     "-I" + os.path.join(ROOT, "include"),
                     '-DH2_NCCL_DEFAULT="%s"' % ncclso] + os.environ.get("H2_NVCC_DEFS", "").split()
    procs = []
    for src in SOURCES:                       # compile the translation units in parallel
        obj = os.path.join(CSRC, os.path.basename(src) + ".o")
        cmd = [nvcc] + common + ["-c", src, "-o", obj]
        if src.endswith(".cu") and verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((subprocess.Popen(cmd), cmd))
        objs.append(obj)
    for pr, cmd in procs:
        if pr.wait() != 0:
            raise subprocess.CalledProcessError(pr.returncode, cmd)
    tmp = LIB + ".tmp"
    subprocess.check_call([nvcc] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs + ["-ldl", "-lrt", "-lpthread"])
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
