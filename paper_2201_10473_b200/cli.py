"""Command line: ``python -m paper_2201_10473_b200.cli {mul,verify,plan,bench}``.

Mirrors the SPEC's bench_cli subcommands that touch the multiply path
(SPEC.md:494-495, 514): ``verify`` checks a known-answer file of
``A_hex B_hex C_hex`` lines on the GPU and exits 0 on
success, 2 on any mismatch, 1 on usage errors; ``mul`` multiplies two hex
polynomials (full product, or mod X^N - 1 with --ring N); ``plan`` prints the
engine plan for a size; ``bench`` reports the paper's Appendix-E statistic
(mean over seeded datasets of the minimum over repeated runs) on the GPU.
"""

from __future__ import annotations

import argparse
import json
import re
import sys

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_MISMATCH = 0, 1, 2


def _read_kat(path: str):
    ring = None
    rows = []
    with open(path) as f:
        for ln in f:
            ln = ln.strip()
            if not ln:
                continue
            if ln.startswith("#"):
                m = re.search(r"X\^(\d+)-1", ln)
                if m:
                    ring = int(m.group(1))
                continue
            parts = ln.split()
            if len(parts) != 3:
                raise ValueError(f"bad KAT line (need A_hex B_hex C_hex): {ln[:40]}...")
            rows.append(parts)
    return ring, rows


def cmd_verify(args) -> int:
    import torch

    from .engine import mul_cyclic, mul_full
    from .poly import from_hex

    try:
        ring, rows = _read_kat(args.file)
        if args.ring:
            ring = args.ring
        A = np.stack([from_hex(r[0]).words for r in rows])
        B = np.stack([from_hex(r[1]).words for r in rows])
        C = [from_hex(r[2]) for r in rows]
    except (OSError, ValueError) as e:
        print(f"verify: {e}", file=sys.stderr)
        return EXIT_USAGE
    dev = torch.device("cuda", torch.cuda.current_device())
    dA = torch.from_numpy(A.view(np.int64)).to(dev)
    dB = torch.from_numpy(B.view(np.int64)).to(dev)
    out = (mul_cyclic(dA, dB, ring) if ring else mul_full(dA, dB)).cpu().numpy().view(np.uint64)
    from .poly import PolyWords

    bad = [i for i in range(len(rows)) if PolyWords(out[i]) != C[i]]
    print(json.dumps({"file": args.file, "vectors": len(rows), "ring": ring,
                      "mismatches": len(bad), "first_bad": bad[:5]}))
    return EXIT_MISMATCH if bad else EXIT_OK


def cmd_mul(args) -> int:
    from .poly import PolyWords, from_hex, schoolbook_mul, to_hex
    from .ring import ring_mul

    try:
        a = from_hex(open(args.a).read())
        b = from_hex(open(args.b).read())
    except (OSError, ValueError) as e:
        print(f"mul: {e}", file=sys.stderr)
        return EXIT_USAGE
    if args.ring:
        t = (args.ring + 63) // 64
        r = ring_mul(a.padded(t) if a.word_len < t else a, b.padded(t) if b.word_len < t else b,
                     args.ring)
    else:
        m = max(a.word_len, b.word_len)
        r = schoolbook_mul(a.padded(m), b.padded(m))
    text = to_hex(PolyWords(r.words))
    if args.out:
        with open(args.out, "w") as f:
            f.write(text + "\n")
    else:
        print(text)
    return EXIT_OK


def cmd_bench(args) -> int:
    """Appendix-E style statistic on the GPU engine (PAPER.md:1645-1675,
    SPEC.md:444-503): for each size, ``--datasets`` seeded random batches;
    per dataset the MINIMUM over ``--runs`` timed calls (CUDA events); report
    the MEAN of those minima, as products/s."""
    import torch

    from .engine import mul_cyclic, mul_full

    dev = torch.device("cuda", torch.cuda.current_device())
    rows = []
    for size in args.sizes:
        t = (size + 63) // 64
        mins = []
        for ds in range(args.datasets):
            rng = np.random.default_rng([args.seed, size, ds])
            A = rng.integers(0, 1 << 64, size=(args.batch, t), dtype=np.uint64)
            B = rng.integers(0, 1 << 64, size=(args.batch, t), dtype=np.uint64)
            if args.ring:
                r = size - 64 * (t - 1)
                if r < 64:
                    A[:, -1] &= np.uint64((1 << r) - 1)
                    B[:, -1] &= np.uint64((1 << r) - 1)
            dA = torch.from_numpy(A.view(np.int64)).to(dev)
            dB = torch.from_numpy(B.view(np.int64)).to(dev)
            flag = torch.zeros(1, dtype=torch.int32, device=dev)

            def call():
                if args.ring:
                    return mul_cyclic(dA, dB, size, check=False, err_flag=flag)
                return mul_full(dA, dB)

            for _ in range(args.warmup):
                call()
            best = float("inf")
            for _ in range(args.runs):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                call()
                e1.record()
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1))
            mins.append(best)
        ms = float(np.mean(mins))
        rows.append({"size_bits": size, "kind": "ring" if args.ring else "full", "batch": args.batch,
                     "datasets": args.datasets, "runs": args.runs, "mean_of_min_ms": round(ms, 5),
                     "products_per_s": round(args.batch / (ms / 1e3), 1)})
    if args.format == "json":
        print(json.dumps(rows))
    else:
        print(f"{'size':>8} {'kind':>5} {'batch':>7} {'mean-of-min ms':>15} {'products/s':>14}")
        for r in rows:
            print(f"{r['size_bits']:>8} {r['kind']:>5} {r['batch']:>7} {r['mean_of_min_ms']:>15.4f} "
                  f"{r['products_per_s']:>14.1f}")
    return EXIT_OK


def cmd_plan(args) -> int:
    from .engine import plan

    kind = "cyclic" if args.ring else "full"
    print(json.dumps(plan(kind, args.batch, args.ring or args.words)))
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="f2x")
    sub = ap.add_subparsers(dest="cmd")
    v = sub.add_parser("verify", help="check a known-answer file (exit 2 on mismatch)")
    v.add_argument("file")
    v.add_argument("--ring", type=int, default=0, help="ring degree (default: from the header)")
    m = sub.add_parser("mul", help="multiply two hex polynomials")
    m.add_argument("a")
    m.add_argument("b")
    m.add_argument("--ring", type=int, default=0)
    m.add_argument("--out", default="")
    bch = sub.add_parser("bench", help="Appendix-E statistic: mean over datasets of min over runs")
    bch.add_argument("--sizes", type=int, nargs="+", default=[17669, 35851, 57637],
                     help="ring degrees n (with --ring) or full-product bit sizes")
    bch.add_argument("--ring", action="store_true", default=True)
    bch.add_argument("--full", dest="ring", action="store_false")
    bch.add_argument("--batch", type=int, default=4096)
    bch.add_argument("--datasets", type=int, default=10)
    bch.add_argument("--runs", type=int, default=20)
    bch.add_argument("--warmup", type=int, default=3)
    bch.add_argument("--seed", type=int, default=0xF2F2)
    bch.add_argument("--format", choices=["json", "text"], default="text")
    p = sub.add_parser("plan", help="print the engine plan")
    p.add_argument("--ring", type=int, default=0)
    p.add_argument("--words", type=int, default=277)
    p.add_argument("--batch", type=int, default=4096)
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_USAGE if e.code else EXIT_OK
    if args.cmd is None:
        ap.print_usage(sys.stderr)
        return EXIT_USAGE
    return {"verify": cmd_verify, "mul": cmd_mul, "plan": cmd_plan, "bench": cmd_bench}[args.cmd](args)


if __name__ == "__main__":
    sys.exit(main())
