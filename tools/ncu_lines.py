"""Per-source-line instruction counts and stall samples from an ncu report
(needs -lineinfo + --import-source).  usage: python tools/ncu_lines.py rep [file-substr] [top]"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
cur_file, cur_line, cur_src = "", None, ""
inst = collections.Counter(); samp = collections.Counter(); srcs = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1]; continue
    if r and r[0] == "Line No":
        hdr = r; ie = hdr.index("Instructions Executed"); ws = hdr.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None or len(r) < len(hdr) - 2:
        continue
    if r[0]:
        cur_line = (cur_file.split("/")[-1], int(r[0])); srcs[cur_line] = r[1].strip(); continue
    if cur_line and r[2].startswith("0x"):
        try:
            inst[cur_line] += int(r[ie]); samp[cur_line] += int(r[ws])
        except ValueError:
            pass
T = sum(inst.values()) or 1; S = sum(samp.values()) or 1
print(f"total warp inst {T:.4g}, stall samples {S}")
for k, v in sorted(inst.items(), key=lambda x: -x[1])[:top]:
    if sub in k[0]:
        print(f"{k[0]:14s}{k[1]:5d} {v / T * 100:5.1f}% inst {samp[k] / S * 100:5.1f}% samples | {srcs.get(k, '')[:80]}")
