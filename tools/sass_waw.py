"""Flag in-flight load destinations that are overwritten before being read (WAW stalls).

python tools/sass_waw.py lib.so kernel_substring
"""
import re, subprocess, sys

so, name = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
lines, on = [], False
for ln in sass.splitlines():
    if "Function :" in ln:
        on = name in ln
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if on and m:
        lines.append((m.group(1), m.group(2).strip()))
W = {"128": 4, "64": 2}
def regs(tok, width=1):
    m = re.match(r"R(\d+)", tok)
    return set(range(int(m.group(1)), int(m.group(1)) + width)) if m else set()
def parse(ins):
    ins = re.sub(r"^@!?U?P\w+\s+", "", ins)
    op, _, rest = ins.partition(" ")
    ops = [o.strip() for o in rest.split(",")] if rest else []
    return op, ops
for i, (addr, ins) in enumerate(lines):
    op, ops = parse(ins)
    if not op.startswith("LDG") or not ops:
        continue
    w = 4 if ".128" in op else 2 if ".64" in op else 1
    dst = regs(ops[0], w)
    for addr2, ins2 in lines[i + 1:]:
        op2, ops2 = parse(ins2)
        src = set().union(*[regs(o) for o in ops2[1:]]) if len(ops2) > 1 else set()
        if "STG" in op2 or "STS" in op2:
            src |= set().union(*[regs(o) for o in ops2])
        if dst & src:
            break
        if ops2 and (regs(ops2[0]) & dst) and not op2.startswith(("BRA", "BSYNC", "BSSY", "EXIT")):
            print(f"{addr} {ins}\n   overwritten at {addr2}: {ins2}")
            break
