#!/usr/bin/env python
"""Benchmark of the B200 SPD-solve path (BASELINE.json north_star).

Headline (N=1): CG iterations/s on the GP squared-exponential matrix
n=32768, b=128 (BASELINE.json configs[1]), FP64, one B200.

* ``value``   — iterations/s with A, rhs resident in HBM: one device-resident
  ``hs_cg_solve`` with max_iters=K (eps=1e-300, recompute every 50 as the
  reference default), timed with CUDA events on the library's stream
  (torch's current stream is handed to the context). A = 4.31 GB >> L2.
* ``e2e``     — the same metric through the reference-facing host-buffer
  entry ``hs_solve_cg_host`` (== ``hsolve::solve_cg``): every call uploads
  the packed matrix from pinned host memory, solves 50 iterations, and
  downloads x. One e2e step = one such call.
* ``roofline`` — the dominant kernel (symv_slab_kernel<128>): algorithmic
  bytes per launch (packed tiles, T*b^2*8) / its mean launch time measured
  with CUDA events around every SYMV launch of the timed solve; peak =
  MEASURED_PEAKS.json hbm_gbs.
* ``cpu_baseline`` — the compiled reference (oracle/_ref, kind "reference")
  or the C restatement (kind "port") on this host's cores, bounded sample.
* ``secondary`` — tiled Cholesky n=32768, b=512 (configs[2]) GFLOP/s
  (n^3/3 / factor time) against cuBLAS DGEMM measured live in this run;
  ``secondary.emulated_fp64`` — the same factorization with the trailing
  update on the INT8 tensor cores (Ozaki slicing, FP64-level accuracy).

``--impl reference`` times the reference CPU implementation (rank 0 only).
Multi-GPU (torchrun, N>1): row-sharded CG over NCCL, strong scaling on the
same n (override with --n).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

REASON_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    0x100: "display_clock_setting",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return json.load(open(p))
    return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int = 0):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                mask = int(parts[2], 16) if parts[2].startswith("0x") else int(parts[2])
            except ValueError:
                continue
            sm.append(s)
            mx.append(m)
            for bit, name in REASON_BITS.items():
                if mask & bit and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline / reference arm


def cpu_reference_cg(n: int, b: int, iters: int, warm: int) -> dict:
    """Reference CG on the host cores: oracle/_ref when built, else the port."""
    from oracle import Oracle, Reference
    threads = len(os.sched_getaffinity(0))
    if Reference.available():
        ref, kind = Reference(), "reference"
    else:
        ref, kind = Oracle(), "port"
    t0 = time.time()
    a = ref.generate_spd(n, b, seed=42)
    rhs = ref.generate_rhs(n, b, seed=42)
    gen_s = time.time() - t0
    if warm > 0:
        (ref.solve_cg(n, b, a, rhs, eps=1e-300, max_iters=warm, workers=threads, trace=False)
         if kind == "reference" else
         ref.solve_cg(n, b, a, rhs, eps=1e-300, max_iters=warm, threads=threads, trace=False))
    t0 = time.time()
    if kind == "reference":
        r = ref.solve_cg(n, b, a, rhs, eps=1e-300, max_iters=iters, workers=threads, trace=False)
        wall = r["wall_ms"] / 1e3
    else:
        r = ref.solve_cg(n, b, a, rhs, eps=1e-300, max_iters=iters, threads=threads, trace=False)
        wall = time.time() - t0  # includes the exit residual matvec
    del a
    return {"value": r["iterations"] / wall, "unit": "iters/s", "cores": threads,
            "kind": kind,
            "sample": f"{r['iterations']} CG iterations (after {warm} warm-up) at n={n}, "
                      f"b={b}, fraction=0, workers_a={threads}; matrix generation "
                      f"{gen_s:.1f} s untimed"}


def cpu_reference_cholesky(n: int, b: int) -> dict:
    from oracle import Oracle, Reference
    threads = len(os.sched_getaffinity(0))
    if Reference.available():
        ref, kind = Reference(), "reference"
    else:
        ref, kind = Oracle(), "port"
    a = ref.generate_spd(n, b, seed=42)
    t0 = time.time()
    if kind == "reference":
        r = ref.factorize(n, b, a, workers=threads)
        sec = r["factor_ms"] / 1e3
    else:
        ref.factorize(n, b, a, threads=threads)
        sec = time.time() - t0
    return {"value": n ** 3 / 3 / sec / 1e9, "unit": "GFLOP/s", "cores": threads,
            "kind": kind, "sample": f"factorize n={n}, b={b}, workers_a={threads}"}


def workload_config(args, world: int) -> dict:
    """The `config` dict, identical in both arms (same workload, same keys)."""
    n, b = args.n, args.b
    N = (n + b - 1) // b
    packed = N * (N + 1) // 2 * b * b * 8
    cfg_idx = "BASELINE.json configs[1]" if n == 32768 and b == 128 else (
        "BASELINE.json configs[3]" if n == 131072 and b == 128 else "not a BASELINE config")
    l2 = (f"inputs larger than L2 (packed A = {packed / 1e9:.2f} GB)" if packed > 126e6 else
          f"inputs fit in L2 (packed A = {packed / 1e6:.1f} MB, not flushed)")
    return {"workload": f"CG on GP squared-exponential SPD matrix, n={n}, b={b} ({cfg_idx})",
            "n": n, "b": b, "seed": 42, "recompute_interval": 50,
            "eps": "1e-300 (fixed iteration count)",
            "parallelism": (f"row-sharded x{world} (NCCL)" if world > 1 else "single device"),
            "l2": l2}


def run_reference_arm(args) -> None:
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    sources compiled by oracle/Makefile) on all host cores, same workload,
    steps and warm-up as our arm. Under torchrun only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    iters, warm = args.steps, args.warmup
    cb = cpu_reference_cg(args.n, args.b, iters, warm)
    line = {
        "impl": "reference", "metric": "cg_iters_per_s", "value": cb["value"],
        "unit": "iters/s", "n_gpus": args.gpus, "steps": iters, "warmup": warm,
        "ms_per_step": 1e3 / cb["value"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic GP squared-exponential matrix (generate_spd seed 42)",
        "config": workload_config(args, args.gpus),
        "device": f"host CPU, {cb['cores']} threads (reference hsolve, homogeneous "
                  f"executor A, fraction 0); rank 0 of {world}",
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": "iters/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit_json(line)


# ---------------------------------------------------------------------------
# our arm


def dgemm_peak(torch) -> float:
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn_like(a)
    c = torch.empty_like(a)
    for _ in range(2):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b, out=c)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    del a, b, c
    torch.cuda.empty_cache()
    return 2 * n ** 3 / (best * 1e-3) / 1e12


def cholesky_secondary(hs, H, rt, torch, args, peak_tf: float, world: int = 1,
                       dist=None) -> dict:
    """Tiled Cholesky GFLOP/s: single GPU, or 2D block-cyclic over `world`
    GPUs (each rank assembles and factors its own tiles; max over ranks)."""
    n, b = args.chol_n, args.chol_b
    cyclic = dist is not None
    m = hs.generate_spd_device(rt, n, b, seed=42, cyclic=cyclic)
    work = hs.DeviceMatrix(rt, n, b, cyclic=cyclic)
    times = []
    launches0 = rt.kernel_launches()
    for rep in range(1 + args.chol_reps):
        work.copy_from(m)  # fresh input each repetition (device copy, untimed)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        H.potrf_device(rt, work)
        e.record()
        e.synchronize()
        if rep > 0:
            t = s.elapsed_time(e)
            if dist is not None:
                tt = torch.tensor([t], dtype=torch.float64, device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t = float(tt.item())
            times.append(t)
        log(f"cholesky rep {rep}: {s.elapsed_time(e):.1f} ms")
    launches = (rt.kernel_launches() - launches0) // (1 + args.chol_reps)
    ms = statistics.median(times)
    gflops = n ** 3 / 3 / (ms * 1e-3) / 1e9
    out = {"metric": "cholesky_gflops", "value": gflops, "unit": "GFLOP/s",
           "ms_per_factor": ms,
           "config": {"workload": "tiled Cholesky + substitutions (configs[2])"
                                  if world == 1 else
                                  "tiled Cholesky + substitutions, 2D block-cyclic "
                                  "(configs[4] layout)",
                      "n": n, "b": b, "flops": "n^3/3", "gpus": world},
           "gpu_launches_per_factor": int(launches),
           "roofline": {"bound": "tensor", "achieved": gflops / 1e3 / world,
                        "peak": peak_tf, "unit": "TFLOP/s per GPU",
                        "frac": gflops / 1e3 / world / peak_tf,
                        "peak_source": "cuBLAS DGEMM 8192^3 measured live in this run "
                                       "(MEASURED_PEAKS.json has no FP64 entry)"}}
    if cyclic and args.chol_slices > 0:
        # 2D block-cyclic factorization with the INT8-emulated update (time only)
        rt.set_cholesky_gemm(args.chol_slices)
        et = []
        for rep in range(1 + args.chol_reps):
            work.copy_from(m)
            torch.cuda.synchronize()
            dist.barrier()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            H.potrf_device(rt, work)
            e.record()
            e.synchronize()
            if rep > 0:
                tt = torch.tensor([s.elapsed_time(e)], dtype=torch.float64, device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                et.append(float(tt.item()))
        rt.set_cholesky_gemm(0)
        ems = statistics.median(et)
        eg = n ** 3 / 3 / (ems * 1e-3) / 1e9
        out["emulated_fp64"] = {
            "value": eg, "unit": "GFLOP/s", "ms_per_factor": ems, "speedup_vs_dmma": ms / ems,
            "engine": f"trailing update on the INT8 tensor cores, {args.chol_slices} slices",
            "roofline": {"bound": "tensor", "achieved": eg / 1e3 / world, "peak": peak_tf,
                         "unit": "TFLOP/s per GPU (FP64-equivalent) vs DGEMM",
                         "frac": eg / 1e3 / world / peak_tf}}
    if not cyclic and args.chol_slices > 0:
        # the same factorization with the trailing update on the INT8 tensor
        # cores (emulated FP64, Ozaki slicing); L compared with the DMMA L
        small = n <= 65536  # both factors on the device for the comparison
        L_dmma = torch.from_numpy(work.download()).cuda() if small else None
        rt.set_cholesky_gemm(args.chol_slices)
        et = []
        for rep in range(1 + args.chol_reps):
            work.copy_from(m)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            H.potrf_device(rt, work)
            e.record()
            e.synchronize()
            if rep > 0:
                et.append(s.elapsed_time(e))
        rt.set_cholesky_gemm(0)
        ems = statistics.median(et)
        eg = n ** 3 / 3 / (ems * 1e-3) / 1e9
        diff = None
        if small:
            L_oz = torch.from_numpy(work.download()).cuda()
            diff = float((L_oz - L_dmma).abs().max() / L_dmma.abs().max())
            del L_oz, L_dmma
        # solve with the emulated factor: relative residual
        rhs_e = torch.from_numpy(hs.generate_rhs(n, b, 42).values).cuda()
        x_e = rhs_e.clone()
        H.trsv_device(rt, work, x_e.data_ptr(), upper=False)
        H.trsv_device(rt, work, x_e.data_ptr(), upper=True)
        res_e = H.true_residual_device(rt, m, x_e.data_ptr(), rhs_e.data_ptr())
        rel_e = res_e / float(torch.linalg.vector_norm(rhs_e[:n]))
        del rhs_e, x_e
        # INT8 tensor work: every FP64 MAC of the trailing update becomes
        # s(s+1)/2 INT8 MACs; nominal dense INT8 peak 4.5 POPS (no measured one)
        pairs = args.chol_slices * (args.chol_slices + 1) // 2
        i8 = eg * 1e9 * pairs / 1e15
        out["emulated_fp64"] = {
            "value": eg, "unit": "GFLOP/s", "ms_per_factor": ems,
            "speedup_vs_dmma": ms / ems,
            "engine": f"trailing update on the INT8 tensor cores (tcgen05 kind::i8), "
                      f"Ozaki slicing, {args.chol_slices} slices",
            "max_abs_L_minus_L_dmma_over_max_L": diff,
            "relative_residual": rel_e,
            "roofline": {"bound": "tensor", "achieved": eg / 1e3, "peak": peak_tf,
                         "unit": "TFLOP/s (FP64-equivalent) vs DGEMM",
                         "frac": eg / 1e3 / peak_tf,
                         "int8_pops_achieved_approx": i8, "int8_pops_nominal": 4.5,
                         "int8_frac_approx": i8 / 4.5}}
        work.copy_from(m)
        H.potrf_device(rt, work)  # DMMA factor again for the solve below
    # substitutions (single GPU, or pipelined over the block-cyclic factor)
    rhs = torch.from_numpy(hs.generate_rhs(n, b, 42).values).cuda()
    x = torch.empty_like(rhs)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.time()
    x.copy_(rhs)
    H.trsv_device(rt, work, x.data_ptr(), upper=False)
    H.trsv_device(rt, work, x.data_ptr(), upper=True)
    torch.cuda.synchronize()
    out["solve_ms"] = (time.time() - t0) * 1e3
    res = H.true_residual_device(rt, m, x.data_ptr(), rhs.data_ptr())
    out["relative_residual"] = res / float(torch.linalg.vector_norm(rhs[:n]))
    if dist is None:
        # mixed precision (beyond the reference API): a 4-slice INT8-emulated
        # factor refined in FP64 against the unmodified A to the FP64 floor
        try:
            xr = torch.empty_like(rhs)
            et = []
            for rep in range(2):
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                s0.record()
                st = H.solve_spd_refine_device(rt, m, work, rhs.data_ptr(), xr.data_ptr(),
                                               slices=4, max_iters=30, tol=0.0)
                s1.record()
                s1.synchronize()
                et.append(s0.elapsed_time(s1))
            out["mixed_precision_solve"] = {
                "engine": "factor with 4 Ozaki slices on the INT8 tensor cores, FP64 "
                          "iterative refinement (hs_solve_spd_refine)",
                "ms_total": min(et), "factor_ms": st.factor_ms,
                "refine_steps": st.iterations, "relative_residual": st.rel_residual,
                "fp64_factor_plus_solve_ms": ms + out["solve_ms"],
                "speedup_vs_fp64": (ms + out["solve_ms"]) / min(et)}
        except Exception as e:  # keep the rest of the secondary
            out["mixed_precision_solve"] = {"error": repr(e)}
    work.free()
    m.free()
    return out


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: refusing to "
                         "measure a different number of GPUs than asked for")
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local} but only "
                         f"{torch.cuda.device_count()} device(s) are visible")
    torch.cuda.set_device(local)
    import paper_2605_13209_b200 as hs
    from paper_2605_13209_b200 import hsolve as H

    stream = torch.cuda.current_stream().cuda_stream
    use_dist = world > 1 or args.dist
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(hs.Runtime.nccl_unique_id()),
                                       dtype=torch.uint8))
        dist.broadcast(idt, 0)
        rt = hs.Runtime.distributed(local, rank, world, bytes(idt.cpu().tolist()),
                                    stream=stream)
    else:
        rt = hs.Runtime(device=local, stream=stream)

    n, b = args.n, args.b
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"

    # --- inputs resident in HBM (each rank assembles its own block rows) ---
    t0 = time.time()
    m = hs.generate_spd_device(rt, n, b, seed=42)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    rhs_np = hs.generate_rhs(n, b, 42).values
    d_rhs = torch.from_numpy(rhs_np).cuda()
    d_x = torch.zeros_like(d_rhs)
    N = (n + b - 1) // b
    T = N * (N + 1) // 2
    packed_bytes = T * b * b * 8
    local_bytes = (m.row_hi * (m.row_hi + 1) // 2 - m.row_lo * (m.row_lo + 1) // 2) * b * b * 8

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local).__enter__()  # sample warm-up + timed region
    # warm-up: W iterations
    cfgw = hs.SolverConfig(block_size=b, eps=1e-300, max_iters=max(args.warmup, 1))
    hs.solve_cg_device(rt, m, d_rhs.data_ptr(), d_x.data_ptr(), cfgw)

    # timed: exactly K iterations in one solve
    cfg = hs.SolverConfig(block_size=b, eps=1e-300, max_iters=args.steps,
                          recompute_interval=50)
    rt.prof_enable(args.prof_every)
    rt.prof_reset()
    launches0 = rt.kernel_launches()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    st = hs.solve_cg_device(rt, m, d_rhs.data_ptr(), d_x.data_ptr(), cfg)
    ev1.record()
    barrier()
    clocks.__exit__(None, None, None)
    ms = ev0.elapsed_time(ev1)
    launches = rt.kernel_launches() - launches0
    n_symv, symv_ms = rt.prof_symv()
    rt.prof_enable(0)
    assert st.iterations == args.steps, (st.iterations, args.steps)
    if use_dist:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        s2 = torch.tensor([symv_ms / max(n_symv, 1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(s2, op=dist.ReduceOp.MAX)
        symv_avg = float(s2.item())
    else:
        symv_avg = symv_ms / max(n_symv, 1)
    value = args.steps / (ms * 1e-3)

    # dominant kernel roofline (per rank: local tiles per launch)
    achieved = local_bytes / (symv_avg * 1e-3) / 1e9
    traffic = None
    prof_json = os.path.join(ROOT, "profiles", "r01_symv_ncu.json")
    if os.path.exists(prof_json):
        try:
            pj = json.load(open(prof_json))
            if pj.get("n") == n and pj.get("b") == b:
                traffic = pj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic,
                "kernel": f"symv_slab_kernel<{b}>", "launches": n_symv,
                "algorithmic_bytes_per_launch": local_bytes, "peak_source": hbm_src}
    # the driver's peak is a copy (read + write); the SYMV only reads, so also
    # report the read-only roofline of this box measured now (same TMA ring)
    try:
        import ctypes as C
        g = C.c_double()
        H._check(rt._L.hs_probe_hbm_read(rt.ctx, 4 << 30, 0, 3, C.byref(g)))
        roofline["read_only_peak_gbs"] = g.value
        roofline["frac_of_read_only_peak"] = achieved / g.value
    except Exception as e:  # diagnostics only
        roofline["read_only_peak_gbs"] = repr(e)

    line = {
        "metric": "cg_iters_per_s", "value": value, "unit": "iters/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic GP squared-exponential matrix (generate_spd seed 42, median "
                "length-scale rule) assembled on the device",
        "config": workload_config(args, world),
        "matrix_assembly_s": round(gen_s, 3),
        "gpu_launches": int(launches),
        "roofline": roofline,
    }

    # ---- e2e through the host-buffer C-ABI entry (every rank; with N GPUs each
    # rank uploads its own block rows from its pinned copy of the matrix) ----
    if not args.no_e2e:
        # pinned host copy of THIS rank's block rows only (the full packed
        # array is 68.8 GB at n=131072; N ranks would pin N copies); the C
        # ABI addresses the caller's full packed array, so it gets the base
        # this buffer would have inside one (only the rank's range is touched)
        import ctypes as C
        host = torch.empty(max(local_bytes // 8, 1), dtype=torch.float64, pin_memory=True)
        tile_off = m.row_lo * (m.row_lo + 1) // 2 * b * b * 8
        base = host.data_ptr() - tile_off
        H._check(rt._L.hs_matrix_download(m.h, C.c_void_p(base)))
        rhs_pin = torch.from_numpy(rhs_np.copy()).pin_memory()
        x_pin = torch.zeros_like(rhs_pin).pin_memory()
        cfge = hs.SolverConfig(block_size=b, eps=1e-300, max_iters=args.e2e_iters)
        p = H._cg_params(cfge)
        from paper_2605_13209_b200._lib import CgStats
        ste = CgStats()
        # one untimed call (allocator / plan warm-up), then timed calls
        H._check(rt._L.hs_solve_cg_host(rt.ctx, n, b, C.c_void_p(base),
                                        C.c_void_p(rhs_pin.data_ptr()), C.byref(p),
                                        C.c_void_p(x_pin.data_ptr()), C.byref(ste), None))
        torch.cuda.synchronize()
        # per-call wall times; the metric uses the median call (the host's
        # PCIe / pinned-memory bandwidth varies between calls on shared boxes)
        call_s, xfer = [], []
        for _ in range(args.e2e_reps):
            if use_dist:
                dist.barrier()
            t0 = time.perf_counter()
            H._check(rt._L.hs_solve_cg_host(rt.ctx, n, b, C.c_void_p(base),
                                            C.c_void_p(rhs_pin.data_ptr()), C.byref(p),
                                            C.c_void_p(x_pin.data_ptr()), C.byref(ste),
                                            None))
            t = time.perf_counter() - t0
            tx = ste.transfer_ms
            if use_dist:  # the job's time is the slowest rank's
                tt = torch.tensor([t, tx], dtype=torch.float64, device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t, tx = float(tt[0]), float(tt[1])
            call_s.append(t)
            xfer.append(tx)
        med = statistics.median(call_s)
        h2d = packed_bytes + rhs_np.nbytes * world  # all ranks' uploads (rows + rhs each)
        line["e2e"] = {"value": ste.iterations / med, "unit": "iters/s",
                       "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": rhs_np.nbytes * world,
                       "step": f"one hs_solve_cg_host call ({args.e2e_iters} iterations) "
                               "from pinned host buffers; host wall clock (max over "
                               f"ranks); median of {args.e2e_reps} calls",
                       "calls_ms": [round(t * 1e3, 2) for t in call_s],
                       "transfer_ms_per_step": statistics.median(xfer),
                       "h2d_gbs": (local_bytes + rhs_np.nbytes) / 1e9 /
                                  (statistics.median(xfer) * 1e-3)}
        del host
        rt.trim()  # the host entry keeps its uploaded matrix cached
    else:
        line["e2e"] = None

    clk = clocks.summary()
    line["clocks"] = clk

    if not args.no_secondary:
        m.free()
        del d_rhs, d_x
        torch.cuda.empty_cache()
        peak_tf = dgemm_peak(torch)
        try:
            sec = cholesky_secondary(hs, H, rt, torch, args, peak_tf, world,
                                     dist if use_dist else None)
        except Exception as e:  # keep the headline line even if this fails
            sec = {"error": repr(e)}
        if rank == 0:
            line["secondary"] = sec

    if world == 1 and not args.no_anchor:
        # the north-star size on one GPU: CG at n=131072 (configs[3]'s matrix),
        # so the N>1 lines (which run that size) have a same-workload N=1 point
        try:
            line["single_gpu_n131072"] = cg_anchor(hs, rt, torch, args)
        except Exception as e:
            line["single_gpu_n131072"] = {"error": repr(e)}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_reference_cg(n, b, args.cpu_iters, 1)
            if not args.no_secondary:
                line["secondary"]["cpu_baseline"] = cpu_reference_cholesky(
                    args.cpu_chol_n, args.chol_b)
        except Exception as e:
            line["cpu_baseline"] = {"error": repr(e)}
    rt.close()
    if use_dist:
        dist.destroy_process_group()
    if rank == 0:  # last, after the communicators' teardown logging
        emit_json(line)


def cg_anchor(hs, rt, torch, args, n: int = 131072, b: int = 128, iters: int = 20) -> dict:
    """CG iterations/s at n=131072 (68.8 GB packed) on this one GPU."""
    m = hs.generate_spd_device(rt, n, b, seed=42)
    rhs = torch.from_numpy(hs.generate_rhs(n, b, 42).values).cuda()
    x = torch.zeros_like(rhs)
    hs.solve_cg_device(rt, m, rhs.data_ptr(), x.data_ptr(),
                       hs.SolverConfig(block_size=b, eps=1e-300, max_iters=3))
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    st = hs.solve_cg_device(rt, m, rhs.data_ptr(), x.data_ptr(),
                            hs.SolverConfig(block_size=b, eps=1e-300, max_iters=iters))
    ev1.record()
    ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    m.free()
    del rhs, x
    torch.cuda.empty_cache()
    N = n // b
    bytes_ = N * (N + 1) // 2 * b * b * 8
    return {"metric": "cg_iters_per_s", "value": st.iterations / (ms * 1e-3), "unit": "iters/s",
            "n": n, "b": b, "iterations": st.iterations, "warmup": 3,
            "ms_per_step": ms / st.iterations,
            "step_gbs": bytes_ / (ms / st.iterations * 1e-3) / 1e9,
            "note": "the N>1 lines run this workload (configs[3]) row-sharded; "
                    "this is its one-GPU point"}


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: launch N ranks on this node (one
    per GPU) with torch.distributed.run, refusing if fewer GPUs are visible."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        log(f"bench.py: --gpus {args.gpus} asked for but only {have} GPU(s) visible; "
            "refusing to measure fewer GPUs than asked for")
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(29500 + os.getpid() % 1000), os.path.abspath(__file__),
           *sys.argv[1:]]
    log("+ " + " ".join(cmd))
    # the ranks' fd 1 is the original stdout (this process points its own fd
    # 1 at stderr; see emit_json)
    return subprocess.call(cmd, stdout=_JSON_OUT if _JSON_OUT is not None else None)


# stdout carries only the JSON line: native libraries (NCCL prints its version
# line and, with NCCL_DEBUG=INFO, its INIT lines to stdout) write to fd 1,
# which main() points at stderr; the JSON goes to a saved copy of the
# original stdout
_JSON_OUT = None


def emit_json(line):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cg-n", "--n", dest="n", type=int, default=None,
                    help="CG size (default 32768 = configs[1] at N=1, 131072 = configs[3] "
                         "at N>1)")
    ap.add_argument("--b", type=int, default=128)
    ap.add_argument("--chol-n", type=int, default=None,
                    help="Cholesky size (default 32768 = configs[2] at N=1, 131072 = "
                         "configs[4] block-cyclic at N>1)")
    ap.add_argument("--chol-b", type=int, default=512)
    ap.add_argument("--chol-reps", type=int, default=2)
    ap.add_argument("--chol-slices", type=int, default=8,
                    help="also time the INT8-emulated FP64 Cholesky with this many "
                         "slices (0: skip)")
    ap.add_argument("--cpu-chol-n", type=int, default=4096)
    ap.add_argument("--cpu-iters", type=int, default=20)
    ap.add_argument("--ref-iters", type=int, default=50)
    ap.add_argument("--prof-every", type=int, default=8,
                    help="bracket every k-th SYMV launch of the timed solve with events")
    ap.add_argument("--e2e-iters", type=int, default=50)
    ap.add_argument("--e2e-reps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="use the NCCL (multi-GPU) code paths even on one GPU")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-anchor", action="store_true",
                    help="skip the one-GPU n=131072 CG point (N=1 only)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: --warmup < 3 violates the timing rules; using 3")
        args.warmup = 3
    if args.n is None:
        args.n = 32768 if args.gpus == 1 else 131072
    if args.chol_n is None:
        args.chol_n = 32768 if args.gpus == 1 else 131072
    if args.gpus > 1:
        # NCCL init lines (nranks per communicator) for the driver's logs
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if "WORLD_SIZE" not in os.environ and args.impl == "ours":
            sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
