"""Build libflowspec.so in-tree for sm_100a (nvcc; no JIT, no torch extension).

    python -m paper_2507_02620_b200.build          # build if stale
    python -m paper_2507_02620_b200.build --force  # rebuild
    FS_NVCC_FLAGS="-DFS_DIAG" python -m paper_2507_02620_b200.build --force --out /tmp/diag.so
        # experiment / diagnostic builds (timeline probes, tuning macros) to a separate file
"""
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libflowspec.so")
CSRC = os.path.join(HERE, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_paths():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    for c in cands:
        inc, lib = os.path.join(c, "include"), os.path.join(c, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(ROOT, "include", "flowspec.h")])


def stale():
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force=False, verbose=False, out=None):
    out = out or SO
    if not force and not stale():
        return SO
    inc, lib = nccl_paths()
    cmd = [NVCC, "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
           "-shared", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), "-I", inc,
           os.path.join(CSRC, "api.cu"), "-o", out + ".tmp",
           "-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    extra = os.environ.get("FS_NVCC_FLAGS", "").split()
    cmd[1:1] = extra
    subprocess.check_call(cmd)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    o = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    print(build(force="--force" in sys.argv or o is not None, verbose="-v" in sys.argv, out=o))
