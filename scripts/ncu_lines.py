"""Per-source-line instruction / stall attribution of an ncu report:
python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 45
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f, out = None, []
for r in csv.reader(io.StringIO(txt)):
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No"):
        try:
            out.append((float(r[7]), float(r[4]), f, int(r[0]), r[1].strip()[:80]))
        except ValueError:
            pass
tot = sum(o[0] for o in out)
ts = sum(o[1] for o in out) or 1
print(f"total warp instructions {tot:.4e}")
for o in sorted(out, reverse=True)[:top]:
    print(f"{o[0] / tot:.3f} stall {o[1] / ts:.3f} {o[2]}:{o[3]} {o[4]}")
