"""Attribute every SASS instruction of an ncu report (cuda,sass view) to the
CUDA source line listed above it, then sum warp instructions and stall
samples per line range.  usage: python tools/ncu_sass_lines.py REP FILE a-b:name ..."""
import csv, io, subprocess, sys, collections

rep, want = sys.argv[1], sys.argv[2]
ranges = []
for s in sys.argv[3:]:
    ab, name = s.split(":", 1)
    a, b = ab.split("-")
    ranges.append((int(a), int(b), name))
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, line = None, None, None
tot_i = collections.Counter(); tot_s = collections.Counter(); ops = collections.defaultdict(collections.Counter)
allI = 0
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0] != "":
        line = int(r[0]); continue
    if r[2] in ("...", "-"):
        continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        ie = float(d["Instructions Executed"]); st = float(d["Warp Stall Sampling (All Samples)"])
    except (KeyError, ValueError):
        continue
    allI += ie
    key = "other"
    if fname.endswith(want):
        for a, b, name in ranges:
            if a <= line <= b:
                key = name; break
        else:
            key = f"{want}:other"
    tot_i[key] += ie; tot_s[key] += st
    op = r[3].split()[0] if r[3].split() else "?"
    if op.startswith("@"):
        op = r[3].split()[1]
    ops[key][op.split(".")[0]] += ie
ts = sum(tot_s.values()) or 1
print(f"total warp instr {allI:.4g}")
for k, v in tot_i.most_common():
    top = ", ".join(f"{o} {100*c/v:.0f}%" for o, c in ops[k].most_common(6))
    print(f"{k:>18}: inst {100*v/allI:5.1f}%  stall {100*tot_s[k]/ts:5.1f}%   [{top}]")
