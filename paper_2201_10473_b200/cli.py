"""Command line: ``python -m paper_2201_10473_b200.cli {mul,verify,plan}``.

Mirrors the SPEC's bench_cli subcommands that touch the multiply path
(SPEC.md:494-495, 514): ``verify`` checks a known-answer file of
``A_hex B_hex C_hex`` lines on the GPU and exits 0 on
success, 2 on any mismatch, 1 on usage errors; ``mul`` multiplies two hex
polynomials (full product, or mod X^N - 1 with --ring N); ``plan`` prints the
engine plan for a size.
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
    return {"verify": cmd_verify, "mul": cmd_mul, "plan": cmd_plan}[args.cmd](args)


if __name__ == "__main__":
    sys.exit(main())
