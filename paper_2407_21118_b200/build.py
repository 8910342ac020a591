"""Build the in-tree CUDA library ``libpalu_b200.so`` for sm_100a with nvcc.

The shared library is the product: a C ABI (include/palu_b200.h) over the
hand-written kernels in csrc/.  It is built in-tree so it travels with the
repository snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libpalu_b200.so")

SOURCES = ["palu_simt.cu", "palu_tc.cu", "palu_gemv.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build palu_b200")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "palu_b200.h")]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, defines=(), out_dir: str = "") -> str:
    """Compile every CUDA source (in parallel) and link libpalu_b200.so.

    ``defines`` / ``out_dir`` build a variant library elsewhere (e.g. the
    diagnostic build with -DPALU_DIAG -DPALU_TRACE under abtmp/diag/, loaded
    through PALU_LIB_PATH for A/B timing); the product build uses neither."""
    lib = os.path.join(out_dir, "libpalu_b200.so") if out_dir else LIB
    if not out_dir and not defines and not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    nvcc = _nvcc()
    tmp = os.path.join(out_dir or HERE, "build")
    os.makedirs(tmp, exist_ok=True)
    jobs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        if not os.path.exists(path):
            continue
        obj = os.path.join(tmp, src.replace(".cu", ".o"))
        cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-I", INCLUDE, "-I", CSRC, "--expt-relaxed-constexpr", *defines, "-c", path, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        jobs.append((cmd, obj))
    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        for f in [ex.submit(subprocess.run, cmd, check=True) for cmd, _ in jobs]:
            f.result()
    out = lib + ".tmp"
    subprocess.run([nvcc, *ARCH, "-shared", "-o", out, *[o for _, o in jobs], "-lcuda"], check=True)
    os.replace(out, lib)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    out_dir = ""
    if "--out" in args:
        out_dir = args[args.index("--out") + 1]
        os.makedirs(out_dir, exist_ok=True)
    print(build(force="--force" in args, verbose="-v" in args,
                defines=[a for a in args if a.startswith("-D")], out_dir=out_dir))
