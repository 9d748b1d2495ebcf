"""Stall samples and executed warp-instructions per CUDA source line of an .ncu-rep
(needs -lineinfo and --import-source on).   python tools/ncu_lines.py rep [topN]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass,cuda'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == 'Line No')
hdr = rows[hi]; ix = {}
for i, h in enumerate(hdr): ix.setdefault(h, i)
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
def f(r, k):
    try: return float(r[ix[k]])
    except Exception: return 0.0
ts = sum(f(r, '# Samples') for r in data); ti = sum(f(r, 'Instructions Executed') for r in data)
print(f"total samples {ts:.0f}  warp-instructions {ti:.0f}")
print(f"{'line':>5} {'samp%':>6} {'inst%':>6} {'long_sb':>7} {'lg':>5} {'short':>5} {'wait':>5} {'nosel':>5}  source")
cum = 0.0
for r in data:
    s = f(r, '# Samples'); cum += s
    if s / ts * 100 < 0.15 and f(r, 'Instructions Executed') / ti * 100 < 0.15: continue
    print(f"{r[0]:>5} {s/ts*100:6.2f} {f(r,'Instructions Executed')/ti*100:6.2f} {f(r,'stall_long_sb'):7.0f} "
          f"{f(r,'stall_lg'):5.0f} {f(r,'stall_short_sb'):5.0f} {f(r,'stall_wait'):5.0f} {f(r,'stall_not_selected'):5.0f}  {r[1].strip()[:80]}")
