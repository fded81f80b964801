"""Constant-time SASS audit.

Flow-sensitive taint analysis over the SASS of every kernel in a built
library (``cuobjdump -sass``): a register is *secret* if its value derives
from operand data.  Operand data enters a kernel only through 32-bit-or-wider
memory loads (LDG/LDS/LD/LDSM/ATOM results); the engine's public tables (node
positions, the mid-leaf permutation) are 8/16-bit loads, and kernel
parameters come from the constant bank (LDC), so neither is secret.  Taint
propagates through every instruction's sources to its destinations (a
predicated write keeps the old taint too; a write under a secret predicate is
secret), to a fixpoint over the control-flow graph.  Violations:

* a branch/exit/indirect jump whose guard predicate or target is secret
  (data-dependent control flow);
* a memory access whose address registers are secret, or that is guarded by
  a secret predicate (data-dependent addressing).

Data-dependent *values* (SEL, LOP3 under a public predicate, the top-bit
reject flag's OR) are constant time and allowed.

    python tools/ct_sass_audit.py [lib.so ...]   # default: the product library
Exit status 1 if any kernel has a violation.  The leaky test fixture
(libf2x_leaky.so, F2X_LEAKY_LEAF=1) is the positive control: its node
kernels MUST be flagged (tests/test_ct_audit.py).
"""

from __future__ import annotations

import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEFAULT_LIB = os.path.join(ROOT, "paper_2201_10473_b200", "_build", "libf2x.so")

LINE = re.compile(r"^\s+/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;?\s*(/\*.*)?$")
REG = re.compile(r"\b(U?R\d+|U?P[0-6]|B\d+)(\.64|\.128)?\b")
LOADS = ("LDG", "LDS", "LD", "LDSM", "ATOM", "ATOMS", "ATOMG", "LDGSTS")
NO_DEST = ("ST", "STG", "STS", "STL", "RED", "REDG", "REDUX_NO", "BAR", "BRA", "BRX", "JMP", "JMX", "EXIT",
           "RET", "CALL", "MEMBAR", "FENCE", "ERRBAR", "CCTL", "WARPSYNC", "BSSY", "BSYNC", "BREAK",
           "NOP", "YIELD", "UBLKCP", "DEPBAR", "SYNCS_NODEST", "ARRIVES", "BPT", "KILL")
BRANCHES = ("BRA", "BRX", "JMP", "JMX", "EXIT", "RET", "CALL")
PUBLIC_DEST = ("S2R", "S2UR", "CS2R", "LDC", "LDCU", "ULDC", "ELECT", "UFLO_NO")


def expand(tok: str) -> list[str]:
    """Register names covered by an operand token (R4.64 -> R4, R5)."""
    out = []
    for m in REG.finditer(tok):
        name, width = m.group(1), m.group(2)
        if name in ("RZ", "URZ", "PT", "UPT"):
            continue
        n = {"": 1, None: 1, ".64": 2, ".128": 4}[width]
        if n > 1 and name[0] in "RU" and name[-1].isdigit() and not name.startswith("UP"):
            pre = "UR" if name.startswith("UR") else "R"
            base = int(name[len(pre):])
            out += [f"{pre}{base + i}" for i in range(n)]
        else:
            out.append(name)
    return out


def split_operands(s: str) -> list[str]:
    ops, depth, cur = [], 0, ""
    for ch in s:
        if ch == "[":
            depth += 1
        elif ch == "]":
            depth -= 1
        if ch == "," and depth == 0:
            ops.append(cur.strip())
            cur = ""
        else:
            cur += ch
    if cur.strip():
        ops.append(cur.strip())
    return ops


class Ins:
    __slots__ = ("addr", "guard", "gtext", "op", "mods", "dests", "srcs", "addr_regs", "target", "text")

    def __init__(self, addr: int, text: str):
        self.addr, self.text = addr, text
        toks = text.split(None, 1)
        self.guard = self.gtext = None
        if toks[0].startswith("@"):
            self.gtext = toks[0][1:]
            self.guard = self.gtext.lstrip("!")
            toks = toks[1].split(None, 1)
        full = toks[0]
        self.op = full.split(".")[0]
        self.mods = full.split(".")[1:]
        rest = toks[1] if len(toks) > 1 else ""
        ops = split_operands(rest)
        self.target = None
        if self.op in ("BRA", "CALL", "BSSY", "JMP") and ops:
            m = re.search(r"0x([0-9a-f]+)\s*$", ops[-1])
            if m:
                self.target = int(m.group(1), 16)
        mem = [o for o in ops if "[" in o]
        self.addr_regs = []
        for o in mem:
            for inner in re.findall(r"\[([^\]]*)\]", o):
                self.addr_regs += expand(inner)
        plain = [o for o in ops if "[" not in o]
        self.dests, self.srcs = [], []
        # spill slots [R1+off] are tracked like registers ("LOC+off")
        if self.op in ("STL", "LDL") and mem:
            m = re.fullmatch(r"\[R1(\+(-?0x[0-9a-f]+))?\]", mem[0].strip())
            if m:
                slot = "LOC" + (m.group(2) or "0x0")
                self.addr_regs = []
                if self.op == "STL":
                    self.dests = [slot]
                    self.srcs = [r for o in plain for r in expand(o)]
                else:
                    d = expand(plain[0]) if plain else []
                    width = 4 if "128" in self.mods else 2 if "64" in self.mods else 1
                    if d and width > 1:
                        base = int(d[0][1:])
                        d = [f"R{base + i}" for i in range(width)]
                    self.dests = d
                    self.srcs = [slot]
                return
        if self.op in NO_DEST or (self.op == "REDUX" and False):
            self.srcs = [r for o in plain for r in expand(o)]
            return
        if not plain:
            return
        if self.op in ("ISETP", "FSETP", "DSETP", "PSETP", "UISETP", "PLOP3", "UPLOP3", "HSETP2", "VOTE",
                       "VOTEU") and len(plain) >= 2:
            nd = 2 if self.op != "VOTE" and self.op != "VOTEU" else 1
            if self.op in ("VOTE", "VOTEU"):
                self.dests = expand(plain[0])
                self.srcs = [r for o in plain[1:] for r in expand(o)]
                return
            self.dests = [r for o in plain[:nd] for r in expand(o)]
            self.srcs = [r for o in plain[nd:] for r in expand(o)]
            return
        first = plain[0]
        d = expand(first)
        width = 4 if "128" in self.mods else 2 if ("64" in self.mods or "WIDE" in self.mods) else 1
        if d and len(d) == 1 and width > 1 and d[0][0] in "RU" and not d[0].startswith("UP"):
            pre = "UR" if d[0].startswith("UR") else "R"
            base = int(d[0][len(pre):])
            d = [f"{pre}{base + i}" for i in range(width)]
        self.dests = d
        rest_ops = plain[1:]
        # LOP3.LUT Pd, Rd, Ra, Rb, Rc, lut, Pp: a predicate AND a register out
        if d and re.fullmatch(r"U?P[0-6T]", first.strip()) and rest_ops and \
                re.fullmatch(r"U?R(\d+|Z)", rest_ops[0].strip()):
            self.dests = d + expand(rest_ops[0])
            rest_ops = rest_ops[1:]
        # carry-out predicates directly after the destination (IADD3 Rd,
        # Pco, Pco, Ra, Rb, Rc; LEA Rd, Pco, ...) are outputs; carry-ins
        # come last (IADD3.X ..., Pci, Pci) and stay sources
        k = 0
        while k < len(rest_ops) and re.fullmatch(r"U?P[0-6T]", rest_ops[k].strip()):
            self.dests += expand(rest_ops[k])
            k += 1
        self.srcs = [r for o in rest_ops[k:] for r in expand(o)]


def parse_functions(sass: str) -> dict[str, list[Ins]]:
    funcs, cur, name = {}, None, None
    for line in sass.splitlines():
        if "Function :" in line:
            name = line.split("Function :")[1].strip()
            cur = funcs.setdefault(name, [])
            continue
        if cur is None:
            continue
        m = LINE.match(line)
        if not m:
            continue
        text = m.group(2).strip().rstrip(";").strip()
        if not text:
            continue
        cur.append(Ins(int(m.group(1), 16), text))
    return funcs


def _comp(g):
    return g[1:] if g.startswith("!") else "!" + g


class Taint:
    """Taint state of one program point: reg -> (base, writes), `base` the
    taint of the last unconditional value and `writes` the later guarded
    writes (guard text, taint), oldest first.  The taint a reader sees under
    guard g walks the writes newest first and stops at a write under g (that
    one certainly executed) or when a write and its complement have both been
    seen (e.g. `@P r = a; @!P r = b`) -- so predicate-correlated code such as
    `@!P3 IADD R39, ...; @!P3 STS [R39]` is not a false positive."""

    def __init__(self, s=None):
        self.s = dict(s or {})

    def sec(self, r, gtext=None):
        if r not in self.s:
            return False
        base, writes = self.s[r]
        acc, seen = False, set()
        for g, tv in reversed(writes):
            acc = acc or tv
            if gtext is not None and g == gtext:
                return acc
            if _comp(g) in seen:
                return acc
            seen.add(g)
        return acc or base

    def step(self, x, spill_secret):
        gsec = x.guard is not None and self.sec(x.guard)
        src_t = any(self.sec(r, x.gtext) for r in x.srcs) or gsec
        if not x.dests:
            return src_t
        if x.op in PUBLIC_DEST:
            val = False
        elif x.op in LOADS and not any(m in ("U8", "S8", "U16", "S16") for m in x.mods):
            val = True
        elif x.op == "LDL" and not x.srcs:
            val = spill_secret or gsec  # (untracked local address)
        else:
            val = src_t or any(self.sec(r, x.gtext) for r in x.addr_regs)
        for r in x.dests:
            if x.gtext is None:
                self.s[r] = (val, ())
            else:
                base, writes = self.s.get(r, (False, ()))
                writes = (writes + ((x.gtext, val),))[-8:]
                if len(writes) == 8:  # bound the history: fold the oldest into base
                    base = base or writes[0][1]
                    writes = writes[1:]
                self.s[r] = (base, writes)
        for r in x.dests:  # a redefined predicate invalidates guards on it
            if r.startswith("P") or r.startswith("UP"):
                for k, (base, writes) in list(self.s.items()):
                    if any(g.lstrip("!") == r for g, _ in writes):
                        self.s[k] = (base, tuple(("?" + g if g.lstrip("!") == r else g, tv) for g, tv in writes))
        return src_t


def _merge(a, b):
    out = {}
    for k in set(a) | set(b):
        va, vb = a.get(k, (False, ())), b.get(k, (False, ()))
        if va == vb:
            out[k] = va
        else:
            ta, tb = Taint({k: va}).sec(k), Taint({k: vb}).sec(k)
            out[k] = (ta or tb, ())
    return out


def audit_function(ins: list[Ins]) -> list[str]:
    if not ins:
        return []
    idx = {x.addr: i for i, x in enumerate(ins)}
    # basic blocks
    leaders = {0}
    for i, x in enumerate(ins):
        if x.op in BRANCHES or x.op == "BRX":
            if i + 1 < len(ins):
                leaders.add(i + 1)
            if x.target is not None and x.target in idx:
                leaders.add(idx[x.target])
    leaders = sorted(leaders)
    block_of = {}
    blocks = []
    for b, s in enumerate(leaders):
        e = leaders[b + 1] if b + 1 < len(leaders) else len(ins)
        blocks.append((s, e))
        for i in range(s, e):
            block_of[i] = b
    call_returns = [i + 1 for i, x in enumerate(ins) if x.op == "CALL" and i + 1 < len(ins)]
    succ = defaultdict(set)
    for b, (s, e) in enumerate(blocks):
        last = ins[e - 1]
        fall = e < len(ins)
        if last.op in ("BRA", "JMP"):
            if last.target in idx:
                succ[b].add(block_of[idx[last.target]])
            if last.guard or any(m in ("U", "DIV") for m in []) or last.srcs:
                if fall:
                    succ[b].add(block_of[e])
        elif last.op == "CALL":
            if last.target in idx:
                succ[b].add(block_of[idx[last.target]])
        elif last.op == "RET":
            for r in call_returns:
                succ[b].add(block_of[r])
        elif last.op == "EXIT":
            if last.guard and fall:
                succ[b].add(block_of[e])
        elif last.op == "BRX":
            for bb in range(len(blocks)):  # unknown targets: every block
                succ[b].add(bb)
        elif fall:
            succ[b].add(block_of[e])
    # dataflow state per block entry (Taint map); local-memory taint for
    # untracked local addresses is flow-insensitive
    state_in = [None for _ in blocks]
    state_in[0] = {}
    spill_secret = False
    changed = True
    it = 0
    while changed and it < 400:
        changed = False
        it += 1
        for b, (s, e) in enumerate(blocks):
            if state_in[b] is None:
                continue
            st = Taint(state_in[b])
            for i in range(s, e):
                x = ins[i]
                src_t = st.step(x, spill_secret)
                if x.op == "STL" and src_t and not x.dests and not spill_secret:
                    spill_secret = True
                    changed = True
            for nb in succ[b]:
                cur = state_in[nb]
                nxt = dict(st.s) if cur is None else _merge(cur, st.s)
                if nxt != cur:
                    state_in[nb] = nxt
                    changed = True
    # violations
    bad = []
    for b, (s, e) in enumerate(blocks):
        if state_in[b] is None:
            continue  # unreachable
        st = Taint(state_in[b])
        for i in range(s, e):
            x = ins[i]
            gsec = x.guard is not None and st.sec(x.guard)
            if x.op in BRANCHES or x.op == "BRX":
                if gsec or (x.op in ("BRX", "JMX", "RET") and any(st.sec(r, x.gtext) for r in x.srcs
                                                                  if r.startswith("R"))):
                    bad.append(f"0x{x.addr:04x} data-dependent branch: {x.text}")
            is_mem = x.op in LOADS or x.op in ("ST", "STG", "STS", "STL", "LDL", "RED", "REDG")
            if is_mem:
                if any(st.sec(r, x.gtext) for r in x.addr_regs):
                    bad.append(f"0x{x.addr:04x} data-dependent address: {x.text}")
                elif gsec:
                    bad.append(f"0x{x.addr:04x} data-dependent predicated access: {x.text}")
            st.step(x, spill_secret)
    return bad


def audit_lib(path: str) -> dict[str, list[str]]:
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    return {name: audit_function(ins) for name, ins in parse_functions(sass).items()}


def main(argv: list[str]) -> int:
    libs = argv or [DEFAULT_LIB]
    status = 0
    for lib in libs:
        res = audit_lib(lib)
        bad = {k: v for k, v in res.items() if v}
        print(f"{os.path.relpath(lib, ROOT)}: {len(res)} kernels audited, {len(bad)} with violations")
        for k, v in sorted(bad.items()):
            print(f"  {k}: {len(v)} violation(s)")
            for line in v[:6]:
                print("    " + line)
        status |= 1 if bad else 0
    return status


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))


def explain(lib: str, func_sub: str, addr: int, reg: str) -> None:
    """Development aid: the instructions that wrote `reg` before `addr`
    and their sources' taint at that point."""
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    for name, ins in parse_functions(sass).items():
        if func_sub in name:
            for x in ins:
                if x.addr < addr and reg in x.dests:
                    print(hex(x.addr), x.text)
            break
