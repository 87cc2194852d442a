"""Builds libfsb200.so in-tree with nvcc for sm_100a (the only target)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfsb200.so")
SOURCES = ["fsb_kernels.cu", "fsb_graph.cpp", "fsb_decode.cpp", "fsb_repair.cpp", "fsb_io.cpp", "fsb_capi.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC,-O2,-ffp-contract=off,-fvisibility=hidden", "-Xptxas", "-v",
         "-shared", "-cudart", "static"]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES]
    deps += [os.path.join(CSRC, "fsb_internal.h"), os.path.join(HERE, "..", "include", "fsb.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, out=None, defines=()):
    """FSB_EXPERIMENTS=1 in the environment builds the profiling-experiment library
    (-DFSB_EXPERIMENTS: the FSB_DEBUG / FSB_SCHED_DEBUG knobs, which give wrong bytes by design);
    the release build never reads those variables.  out/defines: an A/B build of the same sources
    with extra -D macros into another file (tools/gpu/ab/run_ab.sh); the in-tree csrc/ is never
    modified."""
    if out is None and not force and not _stale():
        return LIB
    dst = out or LIB
    tmp = dst + ".%d.tmp" % os.getpid()
    flags = FLAGS + (["-DFSB_EXPERIMENTS"] if os.environ.get("FSB_EXPERIMENTS") == "1" else [])
    flags += ["-D" + d for d in defines]
    cmd = [NVCC] + flags + ["-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libfsb200.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, dst)
    return dst


if __name__ == "__main__":
    # python build.py [--force] [--out PATH] [-DMACRO ...]
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose=True, out=out, defines=defs))
