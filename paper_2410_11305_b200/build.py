"""Build the sm_100a CUDA extension in-tree: ``paper_2410_11305_b200/libqspec_b200.so``.

Plain nvcc (no torch JIT cache): every ``csrc/*.cu`` is compiled for
``-gencode arch=compute_100a,code=sm_100a`` with ``-lineinfo`` and linked into a
C-ABI shared library that ``_lib.py`` loads with ctypes.  nvcc cross-compiles
without a GPU, so this runs in the CPU build container too.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# QS_BUILD_DIR / QS_LIB_OUT: research variants (e.g. ablation builds) go elsewhere
BUILD = os.environ.get("QS_BUILD_DIR") or os.path.join(HERE, "_build")
LIB = os.environ.get("QS_LIB_OUT") or os.path.join(HERE, "libqspec_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
def _nccl_root() -> str:
    """NCCL headers/library: the pip nvidia-nccl package torch itself loads (same soname,
    so one libnccl.so.2 serves torch.distributed and qs_forward_tp2)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        return list(spec.submodule_search_locations)[0]
    return "/usr"


NCCL = _nccl_root()
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", "-I", os.path.join(HERE, "..", "include"), "-I", os.path.join(NCCL, "include")]
LINK = ["-lcudart", "-L", os.path.join(NCCL, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(NCCL, "lib")]


def sources() -> list[str]:
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    extra = os.environ.get("QS_NVCC_EXTRA", "").split()
    # objects built with other flags (e.g. an experiment knob in QS_NVCC_EXTRA) are stale
    stamp = os.path.join(BUILD, "flags.stamp")
    flags = " ".join([NVCC, *ARCH, *FLAGS, *extra])
    if not os.path.exists(stamp) or open(stamp).read() != flags:
        force = True
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(HERE, "..", "include", "qspec_b200.h"))
    objs, jobs = [], []
    for src in sources():
        obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            jobs.append([NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj])

    def run(cmd: list[str]) -> None:
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {cmd[-3]}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)

    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(LIB, objs):
        run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, *LINK])
    with open(stamp, "w") as f:
        f.write(flags)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
