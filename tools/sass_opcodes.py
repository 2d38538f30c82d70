"""Opcode census of every kernel in libjunob200.so (cuobjdump -sass): the
tcgen05 / TMA / packed-FP32 instructions that prove the B200 paths, per
kernel.  usage: python tools/sass_opcodes.py [lib] > profiles/rNN_sass_opcodes.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2503_10855_b200/libjunob200.so"
KEY = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "LDTM", "STTM", "UTCATOMSWS",
       "FFMA2", "FADD2", "FMUL2", "FMNMX3", "MUFU", "SYNCS", "REDG", "ATOMG", "CCTL", "MEMBAR", "SHFL", "LDS", "LDG", "STG"]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
kern, counts = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and kern:
        counts[kern][m.group(2)] += 1
demangle = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
print(f"# static SASS opcode counts per kernel of {lib} (cuobjdump -sass, sm_100a)")
print("# columns: " + " ".join(KEY))
for (k, c), name in zip(counts.items(), demangle):
    total = sum(c.values())
    shown = {op: c[op] for op in KEY if c[op]}
    print(f"{name[:100]}\n    {total} instr: " + ", ".join(f"{op} {v}" for op, v in shown.items()))
