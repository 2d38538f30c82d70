"""Per-CUDA-source-line totals from an ncu report (cuda,sass source view):
instructions executed (warp level) and warp-stall samples.
usage: python tools/ncu_src_lines.py REP [top] [file-substring]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
filt = sys.argv[3] if len(sys.argv) > 3 else ""
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    d = dict(zip(hdr[4:], r[4:]))
    def num(k):
        try:
            return float(d.get(k, "0").replace(",", ""))
        except ValueError:
            return 0.0
    rows.append((fname.split("/")[-1], int(r[0]), r[1].strip()[:90], num("Instructions Executed"),
                 num("Warp Stall Sampling (All Samples)")))
rows = [x for x in rows if filt in x[0]]
ti = sum(x[3] for x in rows) or 1
ts = sum(x[4] for x in rows) or 1
print(f"total warp instr {ti:.4g}, stall samples {ts:.4g}")
for x in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{x[0]:>14}:{x[1]:<5} inst {100*x[3]/ti:5.2f}%  stall {100*x[4]/ts:5.2f}%  {x[2]}")
