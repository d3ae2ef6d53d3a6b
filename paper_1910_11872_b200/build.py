"""Build libbosrm.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo).

The demod kernel is compiled once per window size M (demod_inst.cu, -DBOS_INST_M=M) in
parallel, plus the host/ABI translation unit, then linked into
paper_1910_11872_b200/libbosrm.so (cudart linked statically, so the library loads on a
machine without a GPU and exports the C ABI of include/bos_rootmusic.h).
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "bosrm")
LIB = os.path.join(PKG, "libbosrm.so")

WINDOW_LENS = list(range(3, 33))      # BOS_WINDOW_LEN_MIN .. BOS_WINDOW_LEN_MAX
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + INCLUDE, "-I" + CSRC,
                  "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libbosrm.so")


def _sources_digest(extra: list[str]) -> str:
    h = hashlib.sha256()
    for name in sorted(os.listdir(CSRC)):
        if name.endswith((".cu", ".cuh", ".h")):
            with open(os.path.join(CSRC, name), "rb") as fh:
                h.update(name.encode() + fh.read())
    with open(os.path.join(INCLUDE, "bos_rootmusic.h"), "rb") as fh:
        h.update(fh.read())
    h.update(" ".join(NVFLAGS + extra).encode())
    return h.hexdigest()[:16]


def _run(cmd, log):
    p = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + p.stdout)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed ({p.returncode}): {' '.join(cmd)}\n{p.stdout[-4000:]}")
    return p.stdout


def build(force: bool = False, jobs: int | None = None, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile (if sources changed) and return the path of libbosrm.so.
    `defines` / `out` build a variant library (development A/B builds)."""
    build_dir, lib = BUILD, LIB
    if out is not None:
        build_dir = os.path.join(ROOT, "build", os.path.splitext(os.path.basename(out))[0])
        lib = out
    os.makedirs(build_dir, exist_ok=True)
    extra = [f"-D{d}" for d in defines]
    digest = _sources_digest(extra)
    stamp = os.path.join(build_dir, "stamp")
    if not force and os.path.exists(lib) and os.path.exists(stamp):
        with open(stamp) as fh:
            if fh.read().strip() == digest:
                if out is None and not os.path.exists(MICROBENCH):
                    build_microbench()
                return lib
    cc = nvcc()
    jobs = jobs or max(1, min(len(WINDOW_LENS) + 1, os.cpu_count() or 1))
    tasks = []
    host_obj = os.path.join(build_dir, "bos_rootmusic.o")
    tasks.append(([cc, *NVFLAGS, *extra, "-c", os.path.join(CSRC, "bos_rootmusic.cu"), "-o", host_obj],
                  host_obj + ".log"))
    objs = [host_obj]
    for src in ("analytic.cu", "unwrap.cu"):
        o = os.path.join(build_dir, src.replace(".cu", ".o"))
        tasks.append(([cc, *NVFLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", o], o + ".log"))
        objs.append(o)
    for M in WINDOW_LENS:
        o = os.path.join(build_dir, f"demod_m{M}.o")
        objs.append(o)
        tasks.append(([cc, *NVFLAGS, *extra, f"-DBOS_INST_M={M}", "-c", os.path.join(CSRC, "demod_inst.cu"), "-o", o],
                      o + ".log"))
    # longest (largest M) first
    tasks = [tasks[0]] + tasks[1:][::-1]
    with ThreadPoolExecutor(jobs) as ex:
        outs = list(ex.map(lambda t: _run(*t), tasks))
    if verbose:
        for out in outs:
            for ln in out.splitlines():
                if "registers" in ln or "spill" in ln or "Compiling entry" in ln:
                    print(ln)
    tmp = lib + ".tmp"
    cudalib = os.path.join(os.path.dirname(os.path.dirname(cc)), "lib64")
    _run([cc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-L" + cudalib, "-lcufft",
          "-Xlinker", "-rpath=" + cudalib], os.path.join(build_dir, "link.log"))
    os.replace(tmp, lib)
    if out is None:
        build_microbench(cc)
    with open(stamp, "w") as fh:
        fh.write(digest)
    return lib


MICROBENCH_SRC = os.path.join(ROOT, "tools", "microbench.cu")
MICROBENCH = os.path.join(ROOT, "tools", "microbench")


def build_microbench(cc: str | None = None) -> str:
    """The FP32-pipe microbenchmark (FFMA / FFMA2 / MUFU.RCP peaks, tools/microbench.cu) whose
    FFMA figure bench.py reports as the measured roofline denominator beside the nominal one."""
    cc = cc or nvcc()
    _run([cc, *ARCH, "-O3", "-o", MICROBENCH, MICROBENCH_SRC], os.path.join(BUILD, "microbench.log"))
    return MICROBENCH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
