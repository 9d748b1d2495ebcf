#!/usr/bin/env python
"""bench.py — CSR SpMM (Y = A*X, fp32) throughput on B200, the metric of BASELINE.json.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N ... bench.py --gpus N ...

A step is one SpMM pass over one synthetic input (the hot path: partition already planned,
as the reference keeps partitioning and code generation outside its timed region,
src/executor.cpp:54-69). Prints ONE JSON line on rank 0.

  value      GFLOP/s = 2*nnz*d / t, inputs resident in HBM, CUDA events on the launch stream,
             max over ranks
  e2e        the same metric through the host-buffer entry point (spmx_spmm_host: the
             run_spmm-shaped call), H2D of A and X and D2H of Y inside the timed region
  roofline   algorithmic bytes 8*nnz + 4*(M+1) + 4*N*d + 4*M*d per launch / kernel time,
             against the measured HBM copy peak in MEASURED_PEAKS.json
  cpu_baseline  the reference's own CPU run_spmm (oracle/_ref, all host threads) when it was
             built, else the oracle port, on the same arrays (N=1, rank 0)

Workloads (BASELINE.json configs): N=1 -> c2 (R-MAT scale 20, d=64: the config the >=70 %
target is quoted on); N>1 -> c5 (R-MAT scale 24, d=128) sharded into nnz-balanced row
blocks, X broadcast once over NCCL, Y row-sharded ("strong" scaling). --workload overrides.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "spmm_gflops"
UNIT = "GFLOP/s"


# L2 -> SM ceiling of this pool's B200 (whole chip, any access shape, buffer resident in L2):
# 19.4-20.4 TB/s = 68-71 bytes per clock and SM (tools/microbench/l2_fill.cu)
L2_TO_SM_PEAK_TBS = 20.4


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.rows, self.proc, self.index = [], None, index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            f = [x.strip() for x in r.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0])); mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "samples": len(sm),
                "reasons": sorted(reasons)}


def gen_workload(name, device, scale=None):
    from paper_2312_05639_b200 import workloads as W
    a, x, spec = W.make_config(name, device=device, scale_override=scale)
    return a, x, spec


def describe(name, spec, a, extra=None):
    cfg = {"workload": f"{name}: " + {
        "c1": "uniform 4096x4096, 16 nnz/row",
        "c2": "R-MAT scale 20, edge factor 16, (0.57,0.19,0.19,0.05), duplicates merged",
        "c3": "banded Poisson(32) clipped [1,64], 2^22 rows, band +-65536",
        "c4": "R-MAT scale 22, edge factor 32, (0.65,0.15,0.15,0.05), duplicates merged",
        "c5": "R-MAT scale 24, edge factor 16, (0.57,0.19,0.19,0.05), duplicates merged"}[name],
        "m": a.m, "n": a.n, "nnz": a.nnz, "d": spec["d"], "seed": spec["seed"],
        "l2": "inputs exceed L2 (no flush needed)" if name != "c1" else "fits L2"}
    cfg.update(extra or {})
    return cfg


def cpu_reference_run(rp, col, vals, xn, m, n, strategy, trials, warm=1):
    """The reference's CPU run_spmm (oracle/_ref) when built, else the oracle port.
    Returns (gflops_from_mean_time, times_s, kind, cores)."""
    from oracle.pyoracle import Oracle, RefLib
    nnz, d = int(rp[m]), xn.shape[1]
    # all host threads, stated explicitly: torchrun exports OMP_NUM_THREADS=1, which would
    # otherwise make the reference's "threads = 0 -> omp_get_max_threads()" single-threaded
    host_threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    if RefLib.available():
        ref = RefLib()
        a = ref.csr(m, n, rp, col, vals)
        dyn = strategy == "row"  # the reference's default and fastest row-split mode
        _, rep = ref.run_spmm(a, xn, strategy, dyn, host_threads, "native", 128, warm + trials)
        times = rep["times_s"][warm:]
        return 2.0 * nnz * d / (sum(times) / len(times)) / 1e9, times, "reference", rep["threads"]
    orc = Oracle()
    times = []
    for i in range(warm + trials):
        t0 = time.perf_counter()
        orc.spmm_fused(m, n, rp, col, vals, xn, threads=host_threads)
        if i >= warm:
            times.append(time.perf_counter() - t0)
    return 2.0 * nnz * d / (sum(times) / len(times)) / 1e9, times, "port", orc.last_threads


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    import torch
    name = args.workload or ("c2" if world == 1 else "c5")
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    a, x, spec = gen_workload(name, dev, args.scale)
    sample = "full workload"
    if a.nnz > 80_000_000:  # bound the CPU work per step: leading row block with ~1/8 of the nnz
        cut = int(torch.searchsorted(a.row_ptr, a.nnz // 8).item())
        a = a.row_slice(0, cut)
        sample = f"rows [0,{cut}) = {a.nnz} nnz (1/8 of the nonzeros), full X"
    rp, col, vals = a.numpy()
    xn = x.cpu().numpy()
    strategy = args.strategy
    gf, times, kind, cores = cpu_reference_run(rp, col, vals, xn, a.m, a.n, strategy, args.steps,
                                               warm=args.warmup)
    ms = 1e3 * sum(times) / len(times)
    line = {"impl": "reference", "metric": METRIC, "value": gf, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": describe(name, spec, a, {"strategy": strategy + ("+dynamic" if strategy == "row" and kind == "reference" else "")}),
            "cpu_baseline": {"value": gf, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": sample + f"; {args.steps} timed run_spmm trials, mean"},
            "e2e": {"value": gf, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0, "host": {"nproc": os.cpu_count()}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=[None, "c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--scale", type=int, default=None, help="R-MAT scale override (debug only)")
    ap.add_argument("--strategy", default="merge", choices=["row", "nnz", "merge"])
    ap.add_argument("--exact", action="store_true", help="SPMX_EXACT_ORDER (bitwise) mode")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--allgather", action="store_true", help="also time the all-gather of Y (N>1)")
    ap.add_argument("--shard-by", default="nnz", choices=["nnz", "merge"],
                    help="N>1: rank-level row blocks from split_nnz(A, G) (north_star, default) or "
                         "split_merge(A, G) (rows + nonzeros balanced: see tools/shard_scaling.py)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2312_05639_b200 import workloads as W
    from paper_2312_05639_b200 import sharding
    from paper_2312_05639_b200.binding import Context, EXACT_ORDER, Lib

    assert torch.cuda.is_available(), "bench.py needs a CUDA device: there is no CPU fallback"
    # SPMX_BENCH_SHARE_GPU=1 (debug): all ranks use cuda:0 and rendezvous over gloo, to exercise
    # the N>1 code path on a one-GPU box. The ranks' kernels are independent (row shards), none
    # waits on another. Numbers from such a run are not multi-GPU numbers.
    share_gpu = os.environ.get("SPMX_BENCH_SHARE_GPU") == "1"
    if share_gpu:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    name = args.workload or ("c2" if world == 1 else "c5")
    flags = EXACT_ORDER if args.exact else 0
    lib = Lib.get()
    # everything (generation, kernels, timing events) runs on one explicit torch stream; the
    # legacy default stream has handle 0, which the C ABI reads as "create a private stream"
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = Context(local_rank, stream.cuda_stream)

    # ---- inputs: generated on the device (seeded, identical on every rank) ----------------
    a_full, x, spec = gen_workload(name, dev, args.scale)
    d = spec["d"]
    extra = {"strategy": args.strategy, "mode": "exact-order" if args.exact else "default"}
    bcast_ms = None
    if world > 1:
        # nnz-balanced row shards: split_nnz(A, G) on the device, bit-exact with the reference
        da_full = ctx.csr_wrap(a_full, validate=False)
        ranges = (ctx.split_merge if args.shard_by == "merge" else ctx.split_nnz)(da_full, world)
        da_full.close()
        a, (rb, re) = sharding.local_shard(a_full, ranges, rank)
        del a_full
        if rank != 0:
            x.zero_()  # X lives on rank 0; everyone else receives it over NVLink
        torch.cuda.synchronize(); dist.barrier()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); sharding.broadcast_x(x, 0); e1.record(); torch.cuda.synchronize()
        bcast_ms = sharding.max_over_ranks(e0.elapsed_time(e1), dev)
        extra.update({"parallelism": f"row-shard{world}", "shard_by": args.shard_by, "shard_rows": [rb, re],
                      "x_broadcast_ms": bcast_ms})
        if share_gpu:
            extra["debug"] = "SPMX_BENCH_SHARE_GPU: all ranks on one GPU over gloo (code-path check only)"
        nnz_total = int(sharding.sum_over_ranks(a.nnz, dev))
        m_total = int(sharding.sum_over_ranks(a.m, dev))
    else:
        a = a_full
        nnz_total, m_total = a.nnz, a.m
    torch.cuda.empty_cache()  # hand the generator's scratch back: the library allocates with cudaMalloc
    da = ctx.csr_wrap(a)
    y = torch.empty(a.m, d, device=dev)
    plan = ctx.plan(da, args.strategy, 0, flags=flags)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    # ---- device-resident timing ---------------------------------------------------------
    for _ in range(args.warmup):
        ctx.spmm(plan, da, x, y)
    barrier()
    sampler = ClockSampler(local_rank)
    if rank == 0:
        sampler.start()
    launches0 = lib.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        ctx.spmm(plan, da, x, y)
    ev1.record()
    barrier()
    launches = lib.launch_count() - launches0
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        ms_total = sharding.max_over_ranks(ms_total, dev)
        launches = int(sharding.sum_over_ranks(launches, dev))
    ms_step = ms_total / args.steps
    if rank == 0:
        # nvidia-smi cannot sample faster than ~20 ms: when the timed region is shorter than
        # 0.4 s keep the identical kernel running (untimed) so the sampler sees it under load
        window = "timed region"
        if ms_total < 400.0:
            extra_steps = int(min(20000, 400.0 / max(ms_step, 1e-3)))
            for _ in range(extra_steps):
                ctx.spmm(plan, da, x, y)
            torch.cuda.synchronize()
            window = f"timed region + {extra_steps} identical untimed steps (0.4 s) right after it"
        clocks = sampler.stop()
        clocks["window"] = window
    else:
        clocks = None
    if world > 1:
        dist.barrier()
    gflops = 2.0 * nnz_total * d / (ms_step * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (spmm_chunk_kernel + its carry fix-up = the step) ----
    peak, peak_src = load_peaks()
    n_cols = a.n
    bytes_alg = W.algorithmic_bytes(m_total, n_cols, nnz_total, d)
    achieved = bytes_alg / (ms_step * 1e-3) / 1e9
    traffic = None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        key = f"{name}:{args.strategy}:{'exact' if args.exact else 'default'}"
        if world == 1 and args.scale is None and key in tj:
            traffic = tj[key]["dram_bytes_per_launch"]
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak * world, "unit": "GB/s",
                "frac": achieved / (peak * world), "traffic": traffic,
                "algorithmic_bytes": bytes_alg, "peak_source": peak_src,
                "kernel": "spmm_chunk_kernel (+ carry_fixup_kernel), one launch pair per step"}
    # Second view: the kernel gathers one X row (4*d bytes) per nonzero through the L2 -> SM
    # path, whose ceiling on this GPU is measured by tools/microbench/l2_fill.cu
    # (profiles/r01_microbench_l2_fill.txt): what bounds the kernel in practice.
    gather_bytes = 4.0 * nnz_total * d
    roofline["gather"] = {"bytes": gather_bytes, "achieved_tbs": gather_bytes / (ms_step * 1e-3) / 1e12,
                          "l2_to_sm_peak_tbs": L2_TO_SM_PEAK_TBS * world,
                          "frac": gather_bytes / (ms_step * 1e-3) / 1e12 / (L2_TO_SM_PEAK_TBS * world),
                          "peak_source": "measured, tools/microbench/l2_fill.cu (L2-resident buffer, "
                                         "LDG.128, 40 warps/SM, SM clock 1.92 GHz)"}
    if world > 1:
        bytes_repl = bytes_alg + (world - 1) * 4 * n_cols * d  # X is replicated on every rank
        roofline["frac_replicated_x"] = (bytes_repl / (ms_step * 1e-3) / 1e9) / (peak * world)

    allgather_ms = None
    if world > 1 and args.allgather:
        barrier()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); yfull = sharding.allgather_rows(y, ranges); e1.record(); torch.cuda.synchronize()
        allgather_ms = sharding.max_over_ranks(e0.elapsed_time(e1), dev)
        del yfull

    # ---- end to end through the host-buffer entry point -----------------------------------------
    rp_h = a.row_ptr.cpu().pin_memory(); col_h = a.col.cpu().pin_memory()
    vals_h = a.vals.cpu().pin_memory(); x_h = x.cpu().pin_memory()
    y_h = torch.empty(a.m, d, dtype=torch.float32).pin_memory()
    rp_n, col_n = rp_h.numpy().view(np.uint64), col_h.numpy().view(np.uint32)
    vals_n, x_n, y_n = vals_h.numpy(), x_h.numpy(), y_h.numpy()
    e2e_steps = max(3, min(args.steps, 10))
    torch.cuda.empty_cache()
    ectx = Context(local_rank)  # private stream

    def e2e_once():
        ectx.spmm_host(a.m, a.n, rp_n, col_n, vals_n, x_n, y=y_n, strategy=args.strategy, flags=flags,
                       nnz=a.nnz)

    e2e_once(); e2e_once()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_once()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        e2e_s = sharding.max_over_ranks(e2e_s, dev)
    h2d = (a.m + 1) * 8 + a.nnz * 8 + a.n * d * 4
    d2h = a.m * d * 4
    if world > 1:
        h2d = int(sharding.sum_over_ranks(h2d, dev)); d2h = int(sharding.sum_over_ranks(d2h, dev))
    e2e = {"value": 2.0 * nnz_total * d / e2e_s / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
           "api": "spmx_spmm_host (run_spmm with host buffers, pinned)"}
    # the e2e result must be the same Y as the device-resident path
    same = bool(np.array_equal(y_n.view(np.uint32), y.cpu().numpy().view(np.uint32)))

    # ---- CPU baseline beside it (rank 0, N=1) ------------------------------------------------------
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        gf, times, kind, cores = cpu_reference_run(rp_n, col_n, vals_n, x_n, a.m, a.n, args.strategy,
                                                   trials=3 if a.nnz < 80_000_000 else 1)
        cpu = {"value": gf, "unit": UNIT, "cores": cores, "kind": kind,
               "sample": f"full {name} workload, {len(times)} timed trials after 1 warm-up, mean "
                         f"({sum(times)/len(times)*1e3:.1f} ms per run_spmm)"}

    if rank == 0:
        line = {"metric": METRIC, "value": gflops, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": describe(name, spec, a, extra), "roofline": roofline,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
                "e2e_matches_device_path": same, "host": {"nproc": os.cpu_count()}}
        if world > 1:
            line["config"].update({"m": m_total, "nnz": nnz_total})
            line["y_allgather_ms"] = allgather_ms
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
