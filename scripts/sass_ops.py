"""Print the opcode sequence (filtered) of one kernel from a cuobjdump -sass dump.
usage: python scripts/sass_ops.py all.sass <mangled-name-substring> [OPCODE_PREFIX ...]"""
import re
import sys

txt = open(sys.argv[1]).read()
pref = tuple(sys.argv[3:]) or ("LDG", "LDS", "DFMA", "F2F", "DMUL", "BRA", "SHF", "LOP3")
for sec in re.split(r"\n\s*Function : ", txt)[1:]:
    name = sec.split("\n", 1)[0].strip()
    if sys.argv[2] not in name:
        continue
    out = []
    for line in sec.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(.*?);", line)
        if not m:
            continue
        toks = m.group(1).split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        if op.startswith(pref):
            out.append(op)
    print(name)
    print(" ".join(out))
    break
