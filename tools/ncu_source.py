"""Hot spots of the SASS/source page of an .ncu-rep: top instructions by stall samples,
and instruction-count by opcode.   python tools/ncu_source.py rep [topN]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
def f(r, k):
    try: return float(r[ix[k]])
    except Exception: return 0.0
tot_s = sum(f(r, '# Samples') for r in data); tot_i = sum(f(r, 'Instructions Executed') for r in data)
print(f"total samples {tot_s:.0f}  total warp-instructions {tot_i:.0f}  SASS lines {len(data)}")
ops = collections.Counter()
for r in data:
    op = r[ix['Source']].split()[0] if r[ix['Source']].split() else '?'
    if op.startswith('@'): op = r[ix['Source']].split()[1]
    ops[op.split('.')[0]] += f(r, 'Instructions Executed')
print("by opcode:", ", ".join(f"{k} {v/tot_i*100:.1f}%" for k, v in ops.most_common(14)))
print(f"{'idx':>5} {'samp%':>6} {'inst%':>6} {'long_sb':>8} {'wait':>6} {'short':>6} {'branch':>6}  sass")
order = sorted(range(len(data)), key=lambda i: -f(data[i], '# Samples'))[:top]
for i in sorted(order):
    r = data[i]
    print(f"{i:5d} {f(r,'# Samples')/tot_s*100:6.2f} {f(r,'Instructions Executed')/tot_i*100:6.2f} "
          f"{f(r,'stall_long_sb'):8.0f} {f(r,'stall_wait'):6.0f} {f(r,'stall_short_sb'):6.0f} {f(r,'stall_branch_resolving'):6.0f}  {r[ix['Source']][:90]}")
