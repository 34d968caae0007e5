"""Build the sm_100a shared library in-tree (nvcc; no JIT cache, so it travels with gpurun)."""
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhsseig_b200.so")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "shared",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(os.path.dirname(PKG), "include", "*.h"))
    return any(os.path.getmtime(f) > t for f in deps)


def build(force=False, verbose=False):
    """Compile every .cu under csrc/ into libhsseig_b200.so (in place): one nvcc per source
    in parallel, then one shared link."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    odir = os.path.join(os.path.dirname(PKG), "build", "obj")
    os.makedirs(odir, exist_ok=True)
    cflags = [f for f in NVCC_FLAGS if f not in ("-shared", "-cudart", "shared")]
    cflags += os.environ.get("HSSEIG_NVCC_EXTRA", "").split()   # e.g. -DHSSEIG_ID_TIMING (tools)

    def comp(src):
        obj = os.path.join(odir, os.path.basename(src)[:-3] + ".o")
        cmd = [nvcc, *cflags, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(max_workers=len(sources())) as ex:
        objs = list(ex.map(comp, sources()))
    cmd = [nvcc, *NVCC_FLAGS, "-o", LIB + ".tmp", *objs]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
