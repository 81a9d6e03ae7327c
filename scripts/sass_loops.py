"""List the loops (backward branches) of one kernel's SASS with their instruction mix:
python scripts/sass_loops.py <cuobjdump -sass text of one function>"""
import collections
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
ins = []
for ln in lines:
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, txt) in enumerate(ins):
    m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|)\s*0x([0-9a-f]+)", txt) or re.search(r"BRA .*?0x([0-9a-f]+)", txt)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt <= a and tgt in addr:
        body = ins[addr[tgt]:i + 1]
        ops = collections.Counter(t.split()[1 if t.startswith("@") else 0].split(".")[0] for _, t in body)
        dp = ops["DFMA"] + ops["DMUL"] + ops["DADD"]
        print(f"loop {tgt:#x}-{a:#x}: {len(body)} instr, DP {dp}, MUFU {ops['MUFU']}, LDS {ops['LDS']}, "
              f"other {len(body) - dp - ops['MUFU'] - ops['LDS']}: {dict(ops.most_common(8))}")
