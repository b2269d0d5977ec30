"""Build libsnapmla.so in-tree with nvcc for sm_100a (no JIT cache, no torch)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsnapmla.so")
SOURCES = ["append.cu", "decode.cu", "decode_sw.cu", "decode_mx.cu", "combine.cu", "fetch.cu", "measure.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    # IEEE division / no FTZ: append + q-quant are bit-exact with the oracle
    "-prec-div=true", "-ftz=false",
    "-Xptxas", "-v",
]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "snapmla.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, hang_check=False, out=None, defines=()):
    """Compile libsnapmla.so (or `out`); `defines` are extra -D macros for experiment variants."""
    lib = out or LIB
    if not force and not hang_check and out is None and not defines and not _stale():
        return LIB
    extra = (["-DSNAPMLA_HANG_CHECK"] if hang_check else []) + [f"-D{d}" for d in defines]
    cmd = [NVCC, *FLAGS, *extra, "-o", lib, *[os.path.join(CSRC, s) for s in SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed building libsnapmla.so")
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, hang_check="--hang-check" in sys.argv))
