"""Find the backward-branch loops of one kernel's SASS and count their instructions by
opcode (hot-loop instruction budget without a GPU).
usage: python scripts/sass_loops.py LIB.so SYMBOL [min_mufu]"""
import collections
import re
import subprocess
import sys

lib, sym = sys.argv[1], sys.argv[2]
min_mufu = int(sys.argv[3]) if len(sys.argv) > 3 else 8
out = subprocess.run(["cuobjdump", "-sass", "-fun", sym, lib], capture_output=True, text=True).stdout
ins = []
for line in out.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, txt) in enumerate(ins):
    m = re.search(r"BRA\s+(?:`\()?.*?0x([0-9a-f]+)", txt)
    if not m or "BRA.DIV" in txt:
        continue
    t = int(m.group(1), 16)
    if t >= a or t not in addr:
        continue
    body = ins[addr[t]:i + 1]
    ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", x).split()[0] for _, x in body)
    mufu = sum(v for k, v in ops.items() if k.startswith("MUFU"))
    if mufu < min_mufu:
        continue
    print(f"loop 0x{t:x}-0x{a:x}: {len(body)} instructions, MUFU {mufu}")
    print("   ", ", ".join(f"{k} {v}" for k, v in ops.most_common(24)))
