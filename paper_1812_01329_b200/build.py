"""Build libjanus.so in-tree: every csrc/*.cu and csrc/*.cpp compiled for sm_100a with nvcc."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# dev-only kernel variants for A/B measurements: JANUS_VARIANT=tag builds _build_tag/libjanus_tag.so
# with JANUS_VARIANT_FLAGS added (the binding loads it when JANUS_VARIANT is set); unset = the product
VARIANT = os.environ.get("JANUS_VARIANT", "")
BUILD = os.path.join(HERE, "_build" + (f"_{VARIANT}" if VARIANT else ""))
LIB = os.path.join(HERE, f"libjanus_{VARIANT}.so" if VARIANT else "libjanus.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    if spec is None or not spec.submodule_search_locations:
        return None, None
    base = os.path.join(list(spec.submodule_search_locations)[0], "nccl")
    return os.path.join(base, "include"), os.path.join(base, "lib")


def flags():
    inc, _ = _nccl_dirs()
    f = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if os.environ.get("JANUS_PTXAS_V") else "-O3",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC, "--expt-relaxed-constexpr"] + ARCH
    if inc:
        f += ["-I", inc]
    if VARIANT:
        f += os.environ.get("JANUS_VARIANT_FLAGS", "").split()
    return f


def _compile(src):
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    deps = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(p) for p in [src] + deps):
        return obj, ""
    cmd = [NVCC] + flags() + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(verbose=False):
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        res = list(ex.map(_compile, srcs))
    if verbose:
        for _, log in res:
            if log:
                print(log)
    objs = [o for o, _ in res]
    _, ncclib = _nccl_dirs()
    link = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart"]
    if ncclib:
        link += ["-L", ncclib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={ncclib}"]
    if not os.path.exists(LIB) or max(os.path.getmtime(o) for o in objs) > os.path.getmtime(LIB):
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
