"""Build libv3db.so in-tree with nvcc for sm_100a (no JIT cache, so the .so travels with
the repo snapshot to the GPU box).  Usage: python -m paper_2603_03065_b200.build

Each csrc/*.cu compiles to its own object (in parallel, only when it or a header changed), then
one nvcc link makes the shared library."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
# variant -> (library, object directory, extra flags).  "debug" adds the device-side invariant
# traps (V3DB_DCHECK) and the V3DB_SYNC_CHECK launch checks; results are identical.
VARIANTS = {
    "release": ("libv3db.so", "build", []),
    "debug": ("libv3db_debug.so", "build_debug", ["-DV3DB_DEBUG"]),
}
OUT = os.path.join(HERE, VARIANTS["release"][0])
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-O3"]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def headers() -> list[str]:
    return glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "v3db.h")]


def lib_path(variant: str = "release") -> str:
    return os.path.join(HERE, VARIANTS[variant][0])


def _obj(src: str, variant: str = "release") -> str:
    return os.path.join(HERE, VARIANTS[variant][1], os.path.basename(src)[:-3] + ".o")


def _compile(src: str, verbose: bool, variant: str = "release") -> str:
    obj = _obj(src, variant)
    cmd = [NVCC, *FLAGS, *VARIANTS[variant][2], "-I" + os.path.join(ROOT, "include"), "-c", src, "-o", obj + ".tmp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(obj + ".tmp", obj)
    return obj


def build(verbose: bool = False, force: bool = False, variant: str = "release") -> str:
    out = lib_path(variant)
    os.makedirs(os.path.join(HERE, VARIANTS[variant][1]), exist_ok=True)
    hdr = max(os.path.getmtime(p) for p in headers())
    stale = [s for s in sources()
             if force or not os.path.exists(_obj(s, variant))
             or os.path.getmtime(_obj(s, variant)) < max(os.path.getmtime(s), hdr)]
    if stale:
        with ThreadPoolExecutor(max_workers=min(len(stale), os.cpu_count() or 4)) as ex:
            list(ex.map(lambda s: _compile(s, verbose, variant), stale))
    objs = [_obj(s, variant) for s in sources()]
    if stale or not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(o) for o in objs):
        subprocess.run([NVCC, *ARCH, "-shared", "-o", out + ".tmp", *objs], check=True)
        os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv,
                variant="debug" if "--debug" in sys.argv else "release"))
