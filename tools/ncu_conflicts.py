"""Shared-memory bank conflicts per CUDA source line (ncu cuda,sass view):
excessive shared wavefronts and the ideal count.  usage: REP [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    d = dict(zip(hdr[4:], r[4:]))
    def num(k):
        try:
            return float(d.get(k, "0").replace(",", ""))
        except ValueError:
            return 0.0
    rows.append((fname.split("/")[-1], int(r[0]), r[1].strip()[:80], num("L1 Wavefronts Shared Excessive"),
                 num("L1 Wavefronts Shared"), num("L1 Wavefronts Shared Ideal")))
tx = sum(x[3] for x in rows) or 1
print(f"total excessive shared wavefronts {tx:.4g}, total {sum(x[4] for x in rows):.4g}")
for x in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{x[0]:>12}:{x[1]:<5} excess {x[3]:10.4g} ({100*x[3]/tx:4.1f}%)  wavefronts {x[4]:10.4g} ideal {x[5]:10.4g}  {x[2]}")
