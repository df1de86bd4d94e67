"""Build libdpm.so (all CUDA sources, sm_100a only) in-tree with nvcc.

Each translation unit is compiled to its own object in parallel (build/), then linked into
paper_1811_03557_b200/libdpm.so.  Objects are rebuilt only when their source or a header changed.

    python -m paper_1811_03557_b200.build [--force] [--verbose]
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdpm.so")
OBJDIR = os.path.join(HERE, "build")
SOURCES = ["dst_solve.cu", "dst128.cu", "bep_fused.cu", "bep_sym.cu", "dd.cu", "setup.cu", "ops.cu", "lsq.cu", "dpm_abi.cu"]
HEADERS = ["dpm_internal.h", "sh_device.cuh", os.path.join("..", "..", "include", "dpm.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "-Xptxas", "-warn-spills"]


def _obj(src: str) -> str:
    return os.path.join(OBJDIR, os.path.splitext(src)[0] + ".o")


def _hdr_time() -> float:
    return max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS)


def _obj_stale(src: str, extra) -> bool:
    o = _obj(src)
    if not os.path.exists(o):
        return True
    stamp = o + ".flags"
    if not os.path.exists(stamp) or open(stamp).read() != " ".join(extra):
        return True
    t = os.path.getmtime(o)
    return os.path.getmtime(os.path.join(CSRC, src)) > t or _hdr_time() > t


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) for h in HEADERS]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, extra, verbose: bool):
    o = _obj(src)
    cmd = [NVCC] + FLAGS + extra + (["-Xptxas", "-v"] if verbose else []) + \
        ["-c", os.path.join(CSRC, src), "-o", o + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed on %s:\n%s%s" % (src, r.stdout, r.stderr))
    os.replace(o + ".tmp", o)
    with open(o + ".flags", "w") as f:
        f.write(" ".join(extra))
    return r.stdout + r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    extra = os.environ.get("DPM_NVCC_EXTRA", "").split()   # experiment hook, e.g. "-DFACR_MINB=3"
    if not force and not _stale() and not any(_obj_stale(s, extra) for s in SOURCES if os.path.exists(OBJDIR)):
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    todo = [s for s in SOURCES if force or _obj_stale(s, extra)]
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        logs = list(ex.map(lambda s: _compile(s, extra, verbose), todo))
    if verbose:
        sys.stderr.write("".join(logs))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "--shared", "-Xcompiler", "-fPIC"] + \
        [_obj(s) for s in SOURCES] + ["-o", LIB + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + r.stdout + r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
