"""In-tree build of the engine's shared library (sm_100a only).

    python -m paper_2201_10473_b200.build        # or __graft_entry__.build()

Compiles csrc/*.cu with nvcc (-gencode arch=compute_100a,code=sm_100a,
-lineinfo) in parallel and links paper_2201_10473_b200/_build/libf2x.so.  The
.so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_build")
LIB = os.path.join(OUT, "libf2x.so")
# TEST FIXTURES built from the same sources (never loaded by the product;
# selected per process by F2X_LIB_VARIANT, see _lib.py):
#   leaky   -- F2X_LEAKY_LEAF=1: leaves skip all-zero a words (positive
#              control of the constant-time checks)
#   checked -- F2X_CHECKED=1: every kernel poisons its shared memory first
#              (shared-memory initcheck through the parity tests)
VARIANTS = {"leaky": "-DF2X_LEAKY_LEAF=1", "checked": "-DF2X_CHECKED=1"}
OUT_LEAKY = os.path.join(HERE, "_build_leaky")
LIB_LEAKY = os.path.join(OUT_LEAKY, "libf2x_leaky.so")
OUT_CHECKED = os.path.join(HERE, "_build_checked")
LIB_CHECKED = os.path.join(OUT_CHECKED, "libf2x_checked.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-Xcompiler", "-fvisibility=hidden",
         "-I" + INCLUDE, "-Xptxas", "-warn-spills"]
# F2X_NVCC_EXTRA: extra nvcc flags for schedule experiments (e.g. -DF2X_FUSED_BOTTOM_EVAL=0);
# delete _build/ when changing it (objects are cached by mtime)
FLAGS += os.environ.get("F2X_NVCC_EXTRA", "").split()


def sources() -> list[str]:
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers_mtime() -> float:
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(INCLUDE, "f2x.h"))
    return max(os.path.getmtime(h) for h in hs)


def _compile(src: str, out: str = OUT, extra: tuple = ()) -> str:
    obj = os.path.join(out, os.path.basename(src)[:-3] + ".o")
    if (os.path.exists(obj) and os.path.getmtime(obj) >= os.path.getmtime(src)
            and os.path.getmtime(obj) >= _headers_mtime()):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
    if "spill" in r.stderr.lower() and "0 bytes spill" not in r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False, leaky: bool = False, variant: str | None = None) -> str:
    """Build libf2x.so, or a test fixture (variant "leaky" / "checked")."""
    if leaky:
        variant = "leaky"
    out, lib = {None: (OUT, LIB), "leaky": (OUT_LEAKY, LIB_LEAKY),
                "checked": (OUT_CHECKED, LIB_CHECKED)}[variant]
    extra = (VARIANTS[variant],) if variant else ()
    os.makedirs(out, exist_ok=True)
    subprocess.run([sys.executable, os.path.join(CSRC, "gen_instances.py")], check=True)
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, out, extra), srcs))
    if not os.path.exists(lib) or any(os.path.getmtime(o) > os.path.getmtime(lib) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcudart_static", "-lrt", "-ldl",
               "-lpthread", "-Xlinker", "--exclude-libs,ALL"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print("built", lib)
    return lib


if __name__ == "__main__":
    build(verbose=True)
    for v in VARIANTS:
        if f"--{v}" in sys.argv:
            build(verbose=True, variant=v)
