#!/usr/bin/env python
"""bench.py — CSR SpMM (Y = A*X, fp32) throughput on B200, the metric of BASELINE.json.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N ... bench.py --gpus N ...

A step is one SpMM pass over one synthetic input (the hot path: partition already planned,
as the reference keeps partitioning and code generation outside its timed region,
src/executor.cpp:54-69). Prints ONE JSON line on rank 0.

  value      GFLOP/s = 2*nnz*d / t, inputs resident in HBM, CUDA events on the launch stream,
             max over ranks
  e2e        the same metric through the host-buffer entry points (N=1: spmx_spmm_host, the
             run_spmm-shaped call; N>1: spmx_mg_shard_host + spmx_mg_broadcast_x_host +
             spmx_mg_plan + spmx_mg_spmm + download), H2D of A and X and D2H of Y inside the
             timed region
  roofline   algorithmic bytes 8*nnz + 4*(M+1) + 4*N*d + 4*M*d per launch / kernel time,
             against the measured HBM copy peak in MEASURED_PEAKS.json; roofline.gather is the
             second view (4*d bytes gathered per nonzero against the L2 -> SM ceiling measured
             in this very run by spmx_probe_l2_to_sm)
  cpu_baseline  the reference's own CPU run_spmm (oracle/_ref, all host threads) when it was
             built, else the oracle port, on the same arrays (N=1, rank 0), timed BEFORE the
             GPU legs

Workloads (BASELINE.json configs): N=1 -> c2 (R-MAT scale 20, d=64: the config the >=70 %
target is quoted on); N>1 -> c5 (R-MAT scale 24, d=128) cut into nnz-balanced row blocks by the
library's multi-GPU driver (spmx_mg_*: split_nnz(A, G) on the device, ONE ncclBroadcast of X,
Y row-sharded; "strong" scaling). --workload overrides.

How N ranks come to be:
  * under torchrun (WORLD_SIZE > 1): one process per GPU; rank 0's NCCL id reaches the others
    through a gloo broadcast, every collective on the data side is the library's own NCCL call;
  * `python bench.py --gpus N` alone: ONE process drives the N GPUs (spmx_mg_create:
    ncclCommInitAll, one host thread and stream per GPU);
  * SPMX_BENCH_SHARE_GPU=1 (code-path check on a one-GPU box): the N row blocks live on
    cuda:0 and run one after the other; the "step" is the slowest block (the ranks of a real
    node never wait for each other). Such a line says so in details.debug.
"""
import argparse
import hashlib
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
KERNEL_SRC = os.path.join(ROOT, "paper_2312_05639_b200", "csrc", "spmx_kernels.cuh")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def kernel_sha():
    try:
        return hashlib.sha256(open(KERNEL_SRC, "rb").read()).hexdigest()[:12]
    except OSError:
        return None


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


WORKLOAD_TEXT = {
    "c1": "uniform 4096x4096, 16 nnz/row",
    "c2": "R-MAT scale 20, edge factor 16, (0.57,0.19,0.19,0.05), duplicates merged",
    "c3": "banded Poisson(32) clipped [1,64], 2^22 rows, band +-65536",
    "c4": "R-MAT scale 22, edge factor 32, (0.65,0.15,0.15,0.05), duplicates merged",
    "c5": "R-MAT scale 24, edge factor 16, (0.57,0.19,0.19,0.05), duplicates merged"}


def describe(name, spec, m, n, nnz, strategy):
    """The workload, identically keyed in both arms (the driver compares the dicts)."""
    return {"workload": f"{name}: " + WORKLOAD_TEXT[name], "m": m, "n": n, "nnz": nnz,
            "d": spec["d"], "seed": spec["seed"], "strategy": strategy,
            "l2": "inputs exceed L2 (no flush needed)" if name != "c1" else "fits L2"}


def host_info():
    """nproc and the CPU model (BASELINE.md section 4 asks for both with every result)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu": model}


def host_threads():
    # all host threads, stated explicitly: torchrun exports OMP_NUM_THREADS=1, which would
    # otherwise make the reference's "threads = 0 -> omp_get_max_threads()" single-threaded
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def cpu_reference_run(rp, col, vals, xn, m, n, strategy, trials, warm=1, budget_s=150.0):
    """The reference's CPU run_spmm (oracle/_ref) when built, else the oracle port, `trials`
    timed runs after `warm` untimed ones — fewer (at least 3) when they would not fit
    budget_s. Returns (times_s, kind, cores, mode)."""
    from oracle.pyoracle import Oracle, RefLib
    threads = host_threads()
    if RefLib.available():
        ref = RefLib()
        a = ref.csr(m, n, rp, col, vals)
        dyn = strategy == "row"  # the reference's default and fastest row-split mode
        _, rep = ref.run_spmm(a, xn, strategy, dyn, threads, "native", 128, max(warm, 1))
        per = rep["times_s"][-1]
        trials = max(3, min(trials, int(budget_s / max(per, 1e-6))))
        _, rep = ref.run_spmm(a, xn, strategy, dyn, threads, "native", 128, trials)
        return rep["times_s"], "reference", rep["threads"], \
            "run_spmm, Backend::Native" + (", dynamic dispatch" if dyn else ", static ranges")
    orc = Oracle()
    times = []
    i = 0
    while i < warm + trials:
        t0 = time.perf_counter()
        orc.spmm_fused(m, n, rp, col, vals, xn, threads=threads)
        dt = time.perf_counter() - t0
        if i >= warm:
            times.append(dt)
        elif i == warm - 1:
            trials = max(3, min(trials, int(budget_s / max(dt, 1e-6))))
        i += 1
    return times, "port", orc.last_threads, "oracle port (fused CSR-order loop, OpenMP over rows)"


def cpu_block(times, kind, cores, mode, nnz, d, sample):
    mean = sum(times) / len(times)
    return {"value": 2.0 * nnz * d / mean / 1e9, "unit": UNIT, "cores": cores, "kind": kind,
            "value_best": 2.0 * nnz * d / min(times) / 1e9, "ms_mean": mean * 1e3,
            "ms_min": min(times) * 1e3, "trials": len(times),
            "sample": f"{sample}; {mode}; {len(times)} timed trials after warm-up, value = mean"}


def run_reference_arm(args, rank, world):
    """The reference's own CPU implementation on the box's host cores, same config keys."""
    if rank != 0:
        return
    import torch
    name = args.workload or ("c2" if world == 1 else "c5")
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    a, x, spec = gen_workload(name, dev, args.scale)
    rp, col, vals = a.numpy()
    xn = x.cpu().numpy()
    del x
    strategy = args.strategy
    times, kind, cores, mode = cpu_reference_run(rp, col, vals, xn, a.m, a.n, strategy,
                                                 max(args.steps, 1), warm=max(args.warmup, 1))
    cpu = cpu_block(times, kind, cores, mode, a.nnz, spec["d"], f"full {name} workload")
    line = {"impl": "reference", "metric": METRIC, "value": cpu["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cpu["ms_mean"],
            "higher_is_better": True, "scaling": "strong" if world > 1 else None,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": describe(name, spec, a.m, a.n, a.nnz, strategy),
            "cpu_baseline": cpu,
            "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0, "host": host_info()}
    print(json.dumps(line), flush=True)


def roofline_block(name, args, world, m_total, n_cols, nnz_total, d, ms_step, gather_peak):
    from paper_2312_05639_b200 import workloads as W
    peak, peak_src = load_peaks()
    bytes_alg = W.algorithmic_bytes(m_total, n_cols, nnz_total, d)
    achieved = bytes_alg / (ms_step * 1e-3) / 1e9
    traffic, traffic_src = None, None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        key = f"{name}:{args.strategy}:{'exact' if args.exact else 'default'}"
        if world == 1 and args.scale is None and key in tj:
            ent = tj[key]
            if ent.get("kernel_sha") == kernel_sha():
                traffic, traffic_src = ent["dram_bytes_per_launch"], ent["source"]
            else:
                traffic_src = (f"none for this kernel: {ent['source']} profiled kernel source "
                               f"{ent.get('kernel_sha')}, running {kernel_sha()}")
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak * world, "unit": "GB/s",
                "frac": achieved / (peak * world), "frac_of_nominal_8tbs": achieved / (8000.0 * world),
                "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_bytes": bytes_alg, "peak_source": peak_src,
                "kernel": "spmm_chunk_kernel (+ carry_fixup_kernel), one launch pair per step and shard"}
    gather_bytes = 4.0 * nnz_total * d
    g = {"bytes": gather_bytes, "achieved_tbs": gather_bytes / (ms_step * 1e-3) / 1e12}
    if gather_peak:
        tbs, probe_ms = gather_peak
        g.update({"l2_to_sm_peak_tbs": tbs * world, "frac": g["achieved_tbs"] / (tbs * world),
                  "peak_source": f"measured in this run right after the timed region (spmx_probe_l2_to_sm: "
                                 f"random 256-byte rows of an L2-resident 64 MB buffer, LDG.128, best of 24/32/40/48 "
                                 f"warps per SM x 10 launches, {probe_ms * 1e3:.0f} us per launch)"})
    roofline["gather"] = g
    if world > 1:
        bytes_repl = bytes_alg + (world - 1) * 4 * n_cols * d  # X is replicated on every rank
        roofline["frac_replicated_x"] = (bytes_repl / (ms_step * 1e-3) / 1e9) / (peak * world)
    return roofline


def build_info(lib):
    bi = lib.build_info()
    return {"sass_sched_kernels": int(bi.get("SPMX_SASS_SCHED", "0")), "cuda": bi.get("cuda"),
            "kernel_sha": kernel_sha(), "lib": os.path.relpath(lib.path, ROOT)}


# ------------------------------------------------------------------------------------------
# N = 1
# ------------------------------------------------------------------------------------------
def run_single(args):
    import torch
    from paper_2312_05639_b200.binding import Context, EXACT_ORDER, Lib

    name = args.workload or "c2"
    flags = EXACT_ORDER if args.exact else 0
    # ---- CPU baseline first: before this process has touched the GPU or pinned any memory ----
    # It IS the reference arm, run as a child process (python bench.py --impl reference): the same
    # code, arrays and process conditions as the driver's own reference run. (Measured inside this
    # process after CUDA start-up and host-buffer pinning, the same run_spmm call took 31-34 ms
    # instead of 18-23 ms on c2.)
    cpu = None
    if not args.no_cpu_baseline:
        cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference", "--workload", name,
               "--strategy", args.strategy]
        # the reference speeds up over its first ten calls or so (31 -> 18 ms on c2: clocks, first
        # touches of Y): 10 untimed + 50 timed calls on the small configs (~1.5 s), so that this
        # number agrees with the reference arm's own 200-step run; 2 + 3 on the large ones
        cmd += ["--steps", "50", "--warmup", "10"] if name in ("c1", "c2") else ["--steps", "3", "--warmup", "2"]
        if args.scale is not None:
            cmd += ["--scale", str(args.scale)]
        env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
        try:
            out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env).stdout
            cpu = json.loads([l for l in out.splitlines() if l.startswith("{")][-1])["cpu_baseline"]
        except Exception as e:  # the GPU numbers do not depend on it
            cpu = {"value": None, "unit": UNIT, "error": f"reference arm child failed: {e!r}"}

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    lib = Lib.get()
    # everything (generation, kernels, timing events) runs on one explicit torch stream; the
    # legacy default stream has handle 0, which the C ABI reads as "create a private stream"
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = Context(0, stream.cuda_stream)

    a, x, spec = gen_workload(name, dev, args.scale)
    d = spec["d"]
    torch.cuda.synchronize()

    # host copies (pinned): the e2e leg's inputs and the CPU baseline's arrays
    rp_h = a.row_ptr.cpu().pin_memory(); col_h = a.col.cpu().pin_memory()
    vals_h = a.vals.cpu().pin_memory(); x_h = x.cpu().pin_memory()
    y_h = torch.empty(a.m, d, dtype=torch.float32).pin_memory()
    rp_n, col_n = rp_h.numpy().view(np.uint64), col_h.numpy().view(np.uint32)
    vals_n, x_n, y_n = vals_h.numpy(), x_h.numpy(), y_h.numpy()

    torch.cuda.empty_cache()  # hand the generator's scratch back: the library allocates with cudaMalloc
    da = ctx.csr_wrap(a)
    y = torch.empty(a.m, d, device=dev)
    plan = ctx.plan(da, args.strategy, 0, flags=flags)

    # ---- device-resident timing ---------------------------------------------------------
    for _ in range(args.warmup):
        ctx.spmm(plan, da, x, y)
    torch.cuda.synchronize()
    sampler = ClockSampler(0)
    sampler.start()
    launches0 = lib.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        ctx.spmm(plan, da, x, y)
    ev1.record()
    torch.cuda.synchronize()
    launches = lib.launch_count() - launches0
    ms_total = ev0.elapsed_time(ev1)
    ms_step = ms_total / args.steps
    # nvidia-smi cannot sample faster than ~20 ms: when the timed region is shorter than
    # 0.4 s keep the identical kernel running (untimed) so the sampler sees it under load
    window = "timed region"
    if ms_total < 400.0:
        extra_steps = int(min(20000, 400.0 / max(ms_step, 1e-3)))
        for _ in range(extra_steps):
            ctx.spmm(plan, da, x, y)
        torch.cuda.synchronize()
        window = f"timed region + {extra_steps} identical untimed steps (0.4 s) right after it"
    # the L2 -> SM ceiling at the clocks this run is at (still inside the sampled window)
    gather_peak = ctx.probe_l2_to_sm(10)  # ~15 ms
    clocks = sampler.stop()
    clocks["window"] = window
    gflops = 2.0 * a.nnz * d / (ms_step * 1e-3) / 1e9
    roofline = roofline_block(name, args, 1, a.m, a.n, a.nnz, d, ms_step, gather_peak)

    # ---- end to end through the host-buffer entry point -----------------------------------------
    e2e_steps = max(3, min(args.steps, 10))
    torch.cuda.empty_cache()
    ectx = Context(0)  # private stream

    def e2e_once():
        ectx.spmm_host(a.m, a.n, rp_n, col_n, vals_n, x_n, y=y_n, strategy=args.strategy, flags=flags,
                       nnz=a.nnz)

    e2e_once(); e2e_once()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_once()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    e2e = {"value": 2.0 * a.nnz * d / e2e_s / 1e9, "unit": UNIT,
           "h2d_bytes_per_step": (a.m + 1) * 8 + a.nnz * 8 + a.n * d * 4,
           "d2h_bytes_per_step": a.m * d * 4, "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
           "api": "spmx_spmm_host (run_spmm with host buffers, pinned)"}
    # the e2e result must be the same Y as the device-resident path
    same = bool(np.array_equal(y_n.view(np.uint32), y.cpu().numpy().view(np.uint32)))
    # The same call with PAGEABLE host arrays — what a caller of the reference's run_spmm holds
    # (std::vector): staged through pinned slots by several host threads inside the library
    # (csrc/spmx_stage.cuh). Informational; the contract's e2e above is from pinned memory.
    pg = [np.array(v) for v in (rp_n, col_n, vals_n, x_n)]
    y_pg = np.empty_like(y_n)
    def e2e_pageable():
        ectx.spmm_host(a.m, a.n, pg[0], pg[1], pg[2], pg[3], y=y_pg, strategy=args.strategy, flags=flags, nnz=a.nnz)
    e2e_pageable()
    t0 = time.perf_counter()
    for _ in range(3):
        e2e_pageable()
    e2e["pageable_host_arrays"] = {"ms_per_step": (time.perf_counter() - t0) / 3 * 1e3, "steps": 3,
                                   "matches_device_path": bool(np.array_equal(y_pg.view(np.uint32), y_n.view(np.uint32)))}
    del pg, y_pg

    line = {"metric": METRIC, "value": gflops, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": None, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": describe(name, spec, a.m, a.n, a.nnz, args.strategy),
            "details": {"mode": "exact-order" if args.exact else "default", "build": build_info(lib)},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, "e2e_matches_device_path": same, "host": host_info()}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# N > 1: the library's multi-GPU driver
# ------------------------------------------------------------------------------------------
def run_multi(args, world, rank, local_rank, under_torchrun):
    import torch
    from paper_2312_05639_b200.binding import EXACT_ORDER, Lib, MultiGpu

    share_gpu = os.environ.get("SPMX_BENCH_SHARE_GPU") == "1"
    name = args.workload or "c5"
    flags = EXACT_ORDER if args.exact else 0
    lib = Lib.get()
    dist = None
    details = {"mode": "exact-order" if args.exact else "default", "shard_by": args.shard_by,
               "parallelism": f"row-shard{world}"}

    if under_torchrun:
        if share_gpu:
            raise SystemExit("SPMX_BENCH_SHARE_GPU needs the one-process form: python bench.py --gpus N")
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")  # rendezvous only: hands the NCCL id to the other ranks
        torch.cuda.set_device(local_rank)
        box = [MultiGpu.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        stream = torch.cuda.Stream(device=local_rank)
        torch.cuda.set_stream(stream)
        mg = MultiGpu.for_rank(local_rank, rank, world, box[0], stream=stream.cuda_stream)
        local_devs = [local_rank]
        details["launch"] = "torchrun: one process per GPU, ncclCommInitRank"
    else:
        have = torch.cuda.device_count()
        if share_gpu:
            local_devs = [0]
            mg = MultiGpu([0], n_shards=world)
            details["launch"] = "one process, one GPU"
            details["debug"] = (f"SPMX_BENCH_SHARE_GPU: the {world} row blocks live on cuda:0 and run one after "
                                "the other; step = the slowest block: a code-path check / projection, not a "
                                "multi-GPU number")
        elif have >= world:
            local_devs = list(range(world))
            mg = MultiGpu(local_devs)
            details["launch"] = "one process, one host thread and stream per GPU, ncclCommInitAll"
        else:
            raise SystemExit(f"bench.py --gpus {world}: this box has {have} GPU(s) (SPMX_BENCH_SHARE_GPU=1 "
                             "runs the row blocks on one GPU as a code-path check)")
        torch.cuda.set_device(local_devs[0])
    details["nccl_version"] = mg.info()["nccl_version"]
    dev0 = torch.device("cuda", local_devs[0])

    def reduce(values, op):
        return mg.allreduce(values, op)  # the library's ncclAllReduce over all ranks

    # ---- inputs: generated on the device (seeded, identical wherever they are generated) ------
    a, x, spec = gen_workload(name, dev0, args.scale)
    d = spec["d"]
    m_total, n_cols, nnz_total = a.m, a.n, a.nnz
    torch.cuda.synchronize()
    # The same workload on ONE GPU (rank 0, the unsharded matrix, same strategy and mode), so
    # that the N-GPU number can be read against its own single-GPU time: the N = 1 bench line is
    # a different workload (c2, the configuration the metric is quoted on).
    single = None
    if rank == 0:
        from paper_2312_05639_b200.binding import Context
        sctx = Context.on_torch_stream(local_devs[0]) if not under_torchrun else \
            Context(local_devs[0], torch.cuda.current_stream().cuda_stream)
        sda = sctx.csr_wrap(a, validate=False)
        sy = torch.empty(m_total, d, device=dev0)
        splan = sctx.plan(sda, args.strategy, 0, flags=flags)
        for _ in range(2):
            sctx.spmm(splan, sda, x, sy)
        ts = [sctx.spmm(splan, sda, x, sy, timed=True) for _ in range(5)]
        single_ms = float(np.median(ts))
        single = {"ms_per_step": single_ms, "value": 2.0 * nnz_total * d / (single_ms * 1e-3) / 1e9, "unit": UNIT,
                  "what": f"{name} unsharded on one GPU (rank 0), median of 5"}
        splan.close(); sda.close(); sctx.close()
        del sy
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    ranges = mg.shard_device(a, by=args.shard_by)   # split_nnz(A, G) on the device + placement
    shards = mg.local_shards()
    # X lives on rank 0; every other rank receives it over NVLink in ONE broadcast into replicas
    # the driver owns (with them it also keeps each rank's hottest X rows compact and L2-resident)
    torch.cuda.synchronize()
    copy_ms, bcast_ms = mg.broadcast_x_from_device(x if rank == 0 else None, root=0, shape=(n_cols, d))
    bcast_ms = reduce([bcast_ms], "max")[0]
    mg.plan(args.strategy, 0, flags=flags)
    details.update({"x_broadcast_ms": bcast_ms,
                    "shard_rows": [[int(b), int(e)] for b, e in ranges],
                    "local_shards_rank0": [{k: s[k] for k in ("shard", "device", "nnz")} for s in shards]})

    # ---- device-resident timing: K steps on every rank, max over ranks ---------------------------
    mg.spmm(steps=args.warmup)
    mg.synchronize()
    reduce([0.0], "max")  # barrier
    sampler = ClockSampler(local_devs[0])
    if rank == 0:
        sampler.start()
    launches0 = lib.launch_count()
    ms_step, per_shard = mg.spmm(steps=args.steps, per_shard=True)
    launches = lib.launch_count() - launches0
    if share_gpu:
        ms_step = max(per_shard)  # the blocks ran back to back on one GPU: a node's step is its slowest rank
        details["per_shard_ms"] = per_shard
    ms_step = reduce([ms_step], "max")[0]
    launches = int(reduce([launches], "sum")[0])
    clocks = None
    if rank == 0:
        if ms_step * args.steps < 400.0:
            mg.spmm(steps=int(max(1, min(20000, 400.0 / max(ms_step, 1e-3)))))
        clocks = sampler.stop()
        clocks["window"] = "timed region (+ identical untimed steps up to 0.4 s)"
    reduce([0.0], "max")
    gflops = 2.0 * nnz_total * d / (ms_step * 1e-3) / 1e9
    roofline = roofline_block(name, args, world, m_total, n_cols, nnz_total, d, ms_step, None)

    allgather_ms = None
    if args.allgather:
        allgather_ms = reduce([mg.allgather_y()], "max")[0]

    # ---- end to end: host arrays in, host Y out, through the driver's host entry points ----------
    rows_local = sum(s["row_end"] - s["row_begin"] for s in shards)
    need_host = (m_total + 1) * 8 + nnz_total * 8 + (n_cols * d * 4 if rank == 0 else 0) + 2 * rows_local * d * 4
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = None
    procs_here = world if under_torchrun else 1
    short = avail is not None and need_host * procs_here > 0.6 * avail
    short = bool(reduce([1.0 if short else 0.0], "max")[0])
    if short:
        e2e = {"value": None, "unit": UNIT,
               "skipped": f"host memory: {need_host * procs_here >> 20} MiB of pinned buffers needed, "
                          f"{(avail or 0) >> 20} MiB available"}
    else:
        rp_h = a.row_ptr.cpu().pin_memory(); col_h = a.col.cpu().pin_memory(); vals_h = a.vals.cpu().pin_memory()
        x_h = x.cpu().pin_memory() if rank == 0 else None
        y_blocks = [torch.empty(s["row_end"] - s["row_begin"], d, dtype=torch.float32).pin_memory()
                    for s in shards]
        y_dev = [torch.empty(s["row_end"] - s["row_begin"], d, dtype=torch.float32) for s in shards]
        mg.download_y_shards(y_dev)  # the device-resident result, for the same-bits check below
        rp_n, col_n, vals_n = rp_h.numpy().view(np.uint64), col_h.numpy().view(np.uint32), vals_h.numpy()
        x_n = x_h.numpy() if x_h is not None else None
        del a, x
        torch.cuda.empty_cache()
        mg.set_x_shape(n_cols, d)

        def e2e_once():
            mg.shard_host(m_total, n_cols, rp_n, col_n, vals_n, by=args.shard_by)
            mg.broadcast_x_host(x_n, root=0)
            mg.plan(args.strategy, 0, flags=flags)
            mg.spmm(steps=1)
            mg.download_y_shards(y_blocks)

        e2e_steps = 3
        e2e_once()
        reduce([0.0], "max")
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_once()
        e2e_s = reduce([(time.perf_counter() - t0) / e2e_steps], "max")[0]
        # per process: row_ptr once (the split), every local shard's row_ptr slice, columns and values, X on the root
        h2d = (m_total + 1) * 8 + sum((s["row_end"] - s["row_begin"] + 1) * 8 + s["nnz"] * 8 for s in shards) + \
            (n_cols * d * 4 if rank == 0 else 0)
        d2h = rows_local * d * 4
        h2d, d2h = (int(v) for v in reduce([h2d, d2h], "sum"))
        same = all(bool(torch.equal(p.view(torch.int32), q.view(torch.int32))) for p, q in zip(y_blocks, y_dev))
        same = bool(reduce([0.0 if same else 1.0], "max")[0] == 0.0)
        e2e = {"value": 2.0 * nnz_total * d / e2e_s / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
               "api": "spmx_mg_shard_host + spmx_mg_broadcast_x_host + spmx_mg_plan + spmx_mg_spmm + "
                      "spmx_mg_download_y_shards (host buffers, pinned)",
               "matches_device_path": same}

    if rank == 0:
        line = {"metric": METRIC, "value": gflops, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": describe(name, spec, m_total, n_cols, nnz_total, args.strategy),
                "details": dict(details, build=build_info(lib)),
                "roofline": roofline, "cpu_baseline": None, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks, "y_allgather_ms": allgather_ms, "single_gpu_same_workload": single,
                "speedup_vs_single_gpu": (gflops / single["value"]) if single else None, "host": host_info()}
        print(json.dumps(line), flush=True)
    mg.close()
    if dist is not None:
        dist.destroy_process_group()


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
    ap.add_argument("--allgather", action="store_true", help="also time the all-gather-v of Y (N>1)")
    ap.add_argument("--shard-by", default="nnz", choices=["nnz", "merge"],
                    help="N>1: rank-level row blocks from split_nnz(A, G) (north_star, default) or "
                         "split_merge(A, G) (rows + nonzeros balanced: see tools/shard_scaling.py)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    env_world = int(os.environ.get("WORLD_SIZE", "1"))
    under_torchrun = env_world > 1
    world = env_world if under_torchrun else max(args.gpus, 1)
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    assert torch.cuda.is_available(), "bench.py needs a CUDA device: there is no CPU fallback"
    # SPMX_BENCH_MG=1 (debug): take the multi-GPU driver's path even with one rank, e.g. under
    # `torchrun --nproc-per-node 1`, to exercise the rendezvous and the rank-mode communicator
    if world == 1 and os.environ.get("SPMX_BENCH_MG") != "1":
        run_single(args)
    else:
        run_multi(args, world, rank, local_rank, under_torchrun or "RANK" in os.environ)


if __name__ == "__main__":
    main()
