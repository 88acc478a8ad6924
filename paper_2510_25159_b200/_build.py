"""In-tree build of libwn.so for sm_100a with nvcc (no JIT cache, no torch extension)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libwn.so")
SOURCES = ["wn_build.cu", "wn_query.cu", "wn_alloc.cu", "wn_nurbs.cu", "wn_peak.cu"]
HEADERS = ["wn_common.cuh", os.path.join("..", "..", "include", "wn.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fopenmp", "-shared", "-Xptxas", "-v", "-lgomp"]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for f in SOURCES + HEADERS:
        if os.path.getmtime(os.path.join(CSRC, f)) > t:
            return True
    return False


def build(force=False, verbose=False, out=None, defines=()):
    """Compile libwn.so (or, for A/B experiments, a variant `out` with extra
    -D `defines`)."""
    target = out or LIB
    if not force and not out and not _stale():
        return LIB
    tmp = target + ".tmp%d" % os.getpid()
    cmd = [NVCC] + FLAGS + ["-D" + d for d in defines] + ["-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    if verbose:
        print(r.stderr)
    if not out:
        with open(os.path.join(HERE, "ptxas_info.txt"), "w") as fh:
            # (without the compile times: the file then changes only when the code does)
            fh.write("".join(l for l in r.stderr.splitlines(True) if "Compile time" not in l))
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force=True, verbose=True)
