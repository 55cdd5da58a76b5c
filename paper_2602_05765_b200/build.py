"""Build librlvla.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with
the repo snapshot to the GPU box). Usage: python -m paper_2602_05765_b200.build [-v]."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "librlvla.so")
BUILD = os.path.join(ROOT, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import nvidia  # torch's bundled NCCL 2.28 (the one torch loads at run time)
    for p in nvidia.__path__:
        d = os.path.join(p, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("NCCL headers (nvidia/nccl) not found")


def _flags():
    nd = nccl_dir()
    return ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
                   "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
                   "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"),
                   "-Xptxas", "-v"]


def _compile(src: str, tag: str = "", defines: tuple = ()) -> tuple[str, str]:
    obj = os.path.join(BUILD, os.path.basename(src) + tag + ".o")
    cmd = [NVCC, "-c", src, "-o", obj] + _flags() + [f"-D{d}" for d in defines]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
    return obj, r.stderr


def _stale(srcs) -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = srcs + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "rlvla.h"),
                                                             os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile csrc/*.cu and link librlvla.so (or `out`, e.g. a variant for A/B timing)."""
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    target = out or OUT
    if out is None and not force and not _stale(srcs):
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    tag = "" if out is None else "." + os.path.basename(out)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(lambda f: _compile(f, tag, defines), srcs))
    with open(os.path.join(BUILD, "ptxas" + tag + ".log"), "w") as f:
        for (obj, log) in results:
            f.write(f"== {obj}\n{log}\n")
    nd = nccl_dir()
    tmp = target + ".tmp"
    cmd = [NVCC, "-shared", "-o", tmp] + [o for o, _ in results] + ARCH + [
        "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
        "-Xlinker", "-rpath", "-Xlinker", os.path.join(nd, "lib")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, target)
    if verbose:
        print(open(os.path.join(BUILD, "ptxas.log")).read())
    return target


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
