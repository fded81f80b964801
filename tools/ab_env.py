"""A/B of an environment switch (development aid): per-kernel device times
(tools/kernel_times.py) for each variant, each in its own process.
    python tools/ab_env.py "F2X_TOOM_EVAL=levels" "" -- 57637:16384 35851
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
args = sys.argv[1:]
cut = args.index("--")
variants, sizes = args[:cut], args[cut + 1:]
for v in variants:
    env = dict(os.environ)
    for kv in v.split():
        k, _, val = kv.partition("=")
        env[k] = val
    r = subprocess.run([sys.executable, os.path.join(HERE, "kernel_times.py"), *sizes], env=env,
                       capture_output=True, text=True)
    print(f"== {v or 'default'}")
    print("\n".join(l for l in r.stdout.splitlines() if l.startswith("n=")) or r.stderr[-2000:], flush=True)
