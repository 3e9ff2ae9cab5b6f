"""Build libms.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build", "ms")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
def _nccl_include() -> str:
    """NCCL headers: the venv's copy (the library PyTorch loads), else the system's."""
    try:
        import nvidia.nccl
        for p in nvidia.nccl.__path__:
            if os.path.exists(os.path.join(p, "include", "nccl.h")):
                return os.path.join(p, "include")
    except ImportError:
        pass
    return "/usr/include"


FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include"), "-I", _nccl_include()]

SOURCES = ["ms_capi.cu", "ms_inst_identity.cu", "ms_inst_delta.cu", "ms_inst_radix.cu", "ms_inst_splitters.cu", "ms_sssp.cu",
           "ms_inst_deltashift.cu", "ms_inst_topbits.cu"]
HEADERS = ["ms_device.cuh", "ms_kernels.cuh", "ms_meta.cuh", "ms_wide.cuh", "ms_onesweep.cuh", "ms_large.cuh", "ms_nccl.cuh", "ms_dispatch.cuh", "ms_scan.cuh", "ms_hist.cuh"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, os.path.basename(src).replace(".cu", ".o"))
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + \
        [os.path.join(ROOT, "include", "multisplit.h")]
    if _newer(obj, deps):
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    out = os.path.join(HERE, "libms.so")
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    if _newer(out, objs):
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-ldl"])
        os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
