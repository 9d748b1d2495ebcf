"""Turns the files tools/evidence_r02.sh leaves in gpurun_out/ into the tracked summaries under
profiles/ and re-ties profiles/traffic.json to the kernel source that was profiled.
    python tools/update_profiles.py"""
import hashlib
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")


def run(*cmd):
    return subprocess.run([sys.executable, *cmd], capture_output=True, text=True, cwd=ROOT).stdout


def parse(path):
    d = {}
    for line in open(path):
        m = re.match(r"\s+(\S+)\s+(\S+)\s+([\d.]+)\s*$", line)
        if m:
            d[m.group(1)] = (float(m.group(3)), m.group(2))
    return d


def to_bytes(v, u):
    return int(v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[u])


for c in ("c2", "c3", "c4", "c5", "c2_longrow"):
    open(os.path.join(P, f"r02_ncu_full_{c}_summary.txt"), "w").write(
        run("tools/ncu_summary.py", os.path.join("gpurun_out", f"r02_full_{c}.ncu-rep")))
open(os.path.join(P, "r02_launches_bench_c2.txt"), "w").write(
    run("tools/ncu_launches.py", "gpurun_out/r02_launches_bench_c2.csv",
        "python bench.py --steps 20 --warmup 3 --no-cpu-baseline (round 2)"))
for f in ("r02_launches_bench_c2.csv", "r02_exp_hot_window_c5.txt", "r02_exp_hot_window_c2.txt", "r02_widths_c2.txt",
          "r02_devbench_all.txt", "r02_bench_selfrun.json", "r02_share_c5_g8.json"):
    shutil.copyfile(os.path.join(G, f), os.path.join(P, f))
sha = hashlib.sha256(open(os.path.join(ROOT, "paper_2312_05639_b200", "csrc", "spmx_kernels.cuh"), "rb").read()).hexdigest()[:12]
tj = {}
for cfg, key in (("c2", "c2:merge:default"), ("c3", "c3:nnz:default"), ("c4", "c4:merge:default"), ("c5", "c5:nnz:default")):
    d = parse(os.path.join(P, f"r02_ncu_full_{cfg}_summary.txt"))
    rd, wr = to_bytes(*d["dram__bytes_read.sum"]), to_bytes(*d["dram__bytes_write.sum"])
    tj[key] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "kernel_sha": sha,
               "source": f"profiles/r02_ncu_full_{cfg}_summary.txt (ncu --set full --clock-control none, "
                         "spmm_chunk_kernel, one launch, round 2)"}
json.dump(tj, open(os.path.join(P, "traffic.json"), "w"), indent=1)
print("kernel source sha", sha)
for cfg in ("c2", "c3", "c4", "c5", "c2_longrow"):
    d = parse(os.path.join(P, f"r02_ncu_full_{cfg}_summary.txt"))
    print(cfg, "duration", d.get("gpu__time_duration.sum"), "dram read", d.get("dram__bytes_read.sum"),
          "write", d.get("dram__bytes_write.sum"))
