#!/usr/bin/env python3
"""Count register-bank collisions in the hottest loop of a kernel's SASS.

Usage: sass_banks.py LIB_OR_OBJ FUNCTION [--loop-start HEX | --all]

The loop is the backward BRA (body <= 256 instructions) with the most FFMA2/FADD2/FFMA/FADD instructions (or
the one starting at --loop-start). For each arithmetic instruction the distinct general source
registers are mapped to a bank under two models (reg % 2 and reg % 4); an instruction whose
distinct sources share a bank counts as a collision. A diagnostic only: on B200 a C2 loop
with 8 collisions (mod 4) per 48 packed ops measured no faster than one with 24; the 3% swing
that prompted it was the point array's constant-bank offset (is_kernels.cuh kXyOffset)."""
import re
import subprocess
import sys

ARITH = re.compile(r"^(FFMA2|FADD2|FMUL2|FFMA|FADD|FMUL)\b")


def sass(lib, fn):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, lib], capture_output=True, text=True).stdout
    ins = []
    for line in out.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    return ins


def loops(ins):
    res = []
    for k, (addr, text) in enumerate(ins):
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d\s*,\s*)?0x([0-9a-f]+)", text)
        if m and int(m.group(1), 16) < addr:
            tgt = int(m.group(1), 16)
            body = [t for a, t in ins if tgt <= a <= addr]
            res.append((sum(1 for t in body if ARITH.match(t.split(" ", 1)[-1] if t.startswith("@") else t)), tgt, addr, body))
    return sorted(res, reverse=True)


def collisions(body, mod):
    n = 0
    for t in body:
        if t.startswith("@"):
            t = t.split(" ", 1)[1]
        if not ARITH.match(t):
            continue
        ops = [o.strip() for o in t.split(" ", 1)[1].split(",")]
        srcs = set()
        for o in ops[1:]:
            m = re.match(r"-?\|?R(\d+)", o)
            if m:
                srcs.add(int(m.group(1)))
        banks = [r % mod for r in srcs]
        if len(banks) != len(set(banks)):
            n += 1
    return n


def main():
    lib, fn = sys.argv[1], sys.argv[2]
    ins = sass(lib, fn)
    if "--all" in sys.argv:
        body = [t for _, t in ins]
        n2 = sum(1 for t in body if re.match(r"(@\S+ )?F(FMA|ADD|MUL)2", t))
        packed = [t for t in body if re.match(r"(@\S+ )?F(FMA|ADD|MUL)2", t)]
        print(f"whole function: {len(body)} instructions, {n2} packed fp32, "
              f"collisions mod2={collisions(body, 2)} mod4={collisions(body, 4)}; "
              f"among packed: mod4={collisions(packed, 4)}")
        return
    ls = loops(ins)
    if "--loop-start" in sys.argv:
        s = int(sys.argv[sys.argv.index("--loop-start") + 1], 16)
        ls = [l for l in ls if l[1] == s]
    inner = [l for l in ls if len(l[3]) <= 256] or ls
    narith, s, e, body = inner[0]
    print(f"loop 0x{s:x}-0x{e:x}: {len(body)} instructions, {narith} arithmetic, "
          f"collisions mod2={collisions(body, 2)} mod4={collisions(body, 4)}")


if __name__ == "__main__":
    main()
