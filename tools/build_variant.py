"""Build an EXPERIMENT variant of libf2x.so with extra nvcc flags (development
aid; never loaded by the product):
    python tools/build_variant.py NAME -DF2X_LEAF_LOOP=0 ...
writes paper_2201_10473_b200/_build_exp/NAME/libf2x.so; tools/runs/exp_variants.sh
swaps it in for _build/libf2x.so on the GPU box, one process per variant."""
import concurrent.futures as cf
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_10473_b200 import build as b  # noqa: E402

name, extra = sys.argv[1], tuple(sys.argv[2:])
out = os.path.join(b.HERE, "_build_exp", name)
os.makedirs(out, exist_ok=True)
subprocess.run([sys.executable, os.path.join(b.CSRC, "gen_instances.py")], check=True)
with cf.ThreadPoolExecutor(max_workers=8) as ex:
    objs = list(ex.map(lambda s: b._compile(s, out, extra), b.sources()))
lib = os.path.join(out, "libf2x.so")
subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", lib, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread",
                "-Xlinker", "--exclude-libs,ALL"], check=True)
print("built", lib)
