"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file X.csv):
per kernel of libspmx_b200.so the launch count, average duration and share; and, for the two
kernels of the timed step, the launches over the full work list (largest grid).
    python tools/ncu_launches.py gpurun_out/launches.csv [title]"""
import collections, csv, re, sys

OURS = ("spmx_dev::", "spmm_", "carry_fixup", "validate_", "chunk_", "merge_", "exclusive_scan",
        "chain_first", "count_chunks", "ranges_from", "row_boundaries", "nnz_boundaries",
        "work_items", "boundaries_to", "next_batch", "max_rel_err")
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
per = collections.defaultdict(list)
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"^void ", "", r[ix["Kernel Name"]])
    name = re.sub(r"\(.*$", "", name).replace("spmx_dev::", "")
    if not any(k in r[ix["Kernel Name"]] for k in OURS):
        continue
    us = float(r[ix["Metric Value"]].replace(",", ""))
    us = us / 1e3 if r[ix["Metric Unit"]] in ("ns", "nsecond") else us
    grid = int(r[ix["Grid Size"]].strip("()").split(",")[0])
    per[name].append((us, grid))
tot = sum(u for v in per.values() for u, _ in v)
print(f"# {sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]}")
print(f"launches {sum(len(v) for v in per.values())}  total_us {tot:.1f}")
for name, v in sorted(per.items(), key=lambda kv: -sum(u for u, _ in kv[1])):
    s = sum(u for u, _ in v)
    print(f"{s / tot * 100:6.2f}%  n={len(v):4d}  avg_us={s / len(v):9.2f}  {name}")
step = {}
for name, v in per.items():
    if name.startswith("spmm_chunk_kernel") or name.startswith("carry_fixup_kernel"):
        g = max(gr for _, gr in v)
        full = [u for u, gr in v if gr == g]
        step[name] = (len(full), sum(full) / len(full), g)
if step:
    t = sum(a for _, a, _ in step.values())
    print("# full work-list launches (the timed step): " +
          "; ".join(f"{n} n={c} avg_us={a:.2f} (grid {g})" for n, (c, a, g) in step.items()))
    print("# share of the step: " + ", ".join(f"{n.split('<')[0]} {a / t * 100:.1f} %" for n, (c, a, g) in step.items()))
