"""Build libsparge.so in-tree with nvcc for sm_100a (no GPU needed).

    python -m paper_2502_18137_b200.build [--verbose]

Every .cu / .cpp under csrc/ is compiled with
  -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
and linked into paper_2502_18137_b200/libsparge.so (static cudart).
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libsparge.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-I", CSRC,
          "-I", os.path.join(os.path.dirname(HERE), "include")]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _needs(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False, force=False, defines=(), lib=None):
    """Compile csrc/ into `lib` (default libsparge.so).  `defines` adds -D
    flags (e.g. SPARGE_PHASE_TIMING for the instrumented debug library,
    built into its own object directory and .so)."""
    global BUILD, LIB
    if defines:
        BUILD = os.path.join(HERE, "_build_" + "_".join(d.lower() for d in defines))
        LIB = lib or os.path.join(HERE, "libsparge_" + "_".join(d.lower() for d in defines) + ".so")
    os.makedirs(BUILD, exist_ok=True)
    extra = [f"-D{d}" for d in defines]
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(os.path.dirname(HERE), "include", "sparge.h"))
    objs = []
    for src in _sources():
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if not force and not _needs(obj, [path] + headers):
            continue
        cmd = [NVCC] + ARCH + COMMON + extra + ["-c", path, "-o", obj]
        if src.endswith(".cpp"):
            cmd += ["-x", "c++"]
        if verbose and src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    if force or _needs(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-ldl", "-lrt",
                                                              "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv, defines=defs))
