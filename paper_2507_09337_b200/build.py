"""Build liborcha.so (production, FMA) and liborcha_parity.so (--fmad=false,
ORCHA_PARITY) in-tree for sm_100a with nvcc.  No JIT, no torch extension:
the C ABI in include/orcha.h is the product boundary."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import shutil
import tempfile
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
def _nccl_include() -> str:
    """nccl.h of the NCCL torch ships (types only: the library dlopens libnccl.so.2 at run time)."""
    try:
        import nvidia.nccl
        d = os.path.join(list(nvidia.nccl.__path__)[0], "include")
        if os.path.exists(os.path.join(d, "nccl.h")):
            return d
    except ImportError:
        pass
    return "/usr/include"


COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
          "-I", _nccl_include(), "-Xptxas", "-warn-spills"]
VARIANTS = {
    "liborcha.so": ["--fmad=true"],
    "liborcha_parity.so": ["--fmad=false", "-DORCHA_PARITY"],
}


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "orcha.h"), __file__]


def _stale(target: str) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps())


def _compile(src: str, obj: str, flags) -> str:
    cmd = [NVCC, *ARCH, *COMMON, *flags, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return r.stderr


def build(force: bool = False, verbose: bool = False) -> list:
    """Compile every translation unit of both libraries (production and
    parity) in one pool, then link each library."""
    out = []
    objdir = tempfile.mkdtemp(prefix="orcha_build_")  # objects are not kept: every stale library is relinked whole
    todo = {}
    for lib, flags in VARIANTS.items():
        target = os.path.join(HERE, lib)
        out.append(target)
        if force or _stale(target):
            tag = os.path.splitext(lib)[0]
            todo[target] = (flags, [(src, os.path.join(objdir, f"{tag}_{os.path.splitext(os.path.basename(src))[0]}.o"))
                                    for src in sources()])
    if not todo:
        return out
    with cf.ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
        futs = [ex.submit(_compile, src, obj, flags) for flags, pairs in todo.values() for src, obj in pairs]
        for f in cf.as_completed(futs):
            msg = f.result()
            if verbose and msg.strip():
                print(msg, file=sys.stderr)
    for target, (flags, pairs) in todo.items():
        tmp = target + f".{os.getpid()}.tmp"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *[obj for _, obj in pairs], "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(tmp, target)
    shutil.rmtree(objdir, ignore_errors=True)
    return out


def build_experiment(out: str, extra) -> str:
    """A production library compiled with extra flags (e.g. -D switches of
    measured alternatives) at `out`; loaded via ORCHA_LIB.  Experiments only."""
    objdir = tempfile.mkdtemp(prefix="orcha_exp_")
    flags = VARIANTS["liborcha.so"] + list(extra)
    pairs = [(src, os.path.join(objdir, os.path.splitext(os.path.basename(src))[0] + ".o")) for src in sources()]
    with cf.ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
        for f in [ex.submit(_compile, src, obj, flags) for src, obj in pairs]:
            f.result()
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    r = subprocess.run([NVCC, *ARCH, "-shared", "-o", out, *[o for _, o in pairs], "-ldl"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    shutil.rmtree(objdir, ignore_errors=True)
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--experiment":
        print(build_experiment(sys.argv[2], sys.argv[3:]))
        sys.exit(0)
    print(build(force="--force" in sys.argv, verbose=True))
