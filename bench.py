#!/usr/bin/env python
"""bench.py — BSE eigensolve throughput on B200 (BASELINE.json metric, config 5).

Workload (config 5): a batch of 64 independent complex128 n=4096 BSE matrices (config-2
generator, seeds 0..63), CHOL method, partitioned across ranks by seed (rank r solves seeds
r, r+N, ...). One "step" = every rank solves one matrix of its shard (inputs resident in
HBM, distinct seed per step); NCCL only gathers the per-matrix eigenvalues to all ranks.
value = whole-job FP64 TFLOP/s under the reference flop model (160/3 n^3 real flops per
complex CHOL solve, proj/src/bench.cpp:41-50 x4 for complex).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--n 4096]
                  [--method chol|chol-svd] [--no-cpu-baseline]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

FLOP_COEFF = {"chol": 160.0 / 3.0, "chol-svd": 296.0 / 3.0}  # Table 1 x4 complex


def flops(method: str, n: int) -> float:
    return FLOP_COEFF[method] * float(n) ** 3


def load_peaks() -> dict:
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) >= 7:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for k, v in zip(names, s[3:7]):
                if v.lower() == "active":
                    reasons.add(k)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def seeds_for(rank: int, world: int, steps: int, offset: int = 0):
    """Seed partition of the 64-matrix batch: rank r owns r, r+N, ...; step k -> k-th own seed."""
    own = [s for s in range(64) if s % world == rank]
    return [own[(offset + k) % len(own)] for k in range(steps)]


def run_reference(args):
    """--impl reference: the reference's CPU path (LAPACK restatement, oracle/) on the host."""
    world, rank, _ = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0
    if rank != 0:
        return 0
    import oracle
    from paper_2008_08825_b200 import configs
    cores = os.cpu_count() or 1
    oracle.set_threads(cores)
    method = args.method
    n = args.n
    # warm-up steps: small instances page in OpenBLAS and its thread pool
    a, b = configs.config5(0, n=256)
    for _ in range(args.warmup):
        oracle.solve(method, a, b)
    times = []
    for k in range(args.steps):
        a, b = configs.config5(k % 64, n=n)
        t0 = time.perf_counter()
        oracle.solve(method, a, b)
        times.append(time.perf_counter() - t0)
    t = sum(times)
    value = flops(method, n) * args.steps / t / 1e12
    line = {
        "impl": "reference",
        "metric": f"BSE eigensolve FP64 TFLOP/s (Table-1 flop model), n={n} c128, {method}",
        "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * t / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": f"config5: batch of 64 complex128 n={n} BSE matrices, {method}; "
                               "reference arm = 1 matrix per step on the host CPU",
                   "n": n, "method": method, "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} full {method} solve(s) of config-5 matrices "
                                   f"n={n} (oracle/ LAPACK restatement, OpenBLAS "
                                   f"{oracle.blas_config().split()[1]})"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "s_per_solve": t / args.steps,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--method", default="chol", choices=["chol", "chol-svd"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--lanes", type=int, default=4, help="matrices in flight per GPU")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    world, rank, local = dist_init()
    torch.cuda.set_device(local)
    import paper_2008_08825_b200 as bse
    from paper_2008_08825_b200 import configs
    dev = torch.device("cuda", local)
    n, method = args.n, args.method
    meth = bse.Method.Chol if method == "chol" else bse.Method.CholSvd
    ctx = bse.Context(local)
    ctx.set_kernel_timing(True)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=dev)

    # ---- inputs: (W + K) x lanes distinct matrices of this rank's shard, resident in HBM.
    # One step = `lanes` matrices in flight on this GPU (bse_solve_batched_device: item i on
    # lane i % lanes, each lane's cooperative panel kernels on 1/lanes of the SMs).
    lanes = max(1, args.lanes)
    ctx.set_batch_lanes(lanes)
    total = (args.warmup + args.steps) * lanes
    # a pool of up to 8 distinct matrices per rank, item i -> pool[i % pool]: every input is
    # 512 MiB (> 126 MB L2), so cycling the pool needs no L2 flush between items
    pool = min(total, 8)
    seeds = seeds_for(rank, world, pool)
    host_pool = []
    dev_pool = []
    for sd in seeds:
        a, b = configs.config5(sd, n=n)
        ha = torch.from_numpy(a.T).pin_memory()  # same bytes, column-major complex128
        hb = torch.from_numpy(b.T).pin_memory()
        host_pool.append((ha, hb))
        dev_pool.append((ha.to(dev, non_blocking=True), hb.to(dev, non_blocking=True)))
    host = [host_pool[i % pool] for i in range(total)]
    d_in = [dev_pool[i % pool] for i in range(total)]
    torch.cuda.synchronize()
    d_lams = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(total)]
    d_vs = [torch.empty((n, 2 * n), dtype=torch.complex128, device=dev)  # 2n x n col-major
            for _ in range(lanes)]  # item i writes lane i % lanes's buffer (sequential per lane)
    lam_all = torch.empty((world, args.steps * lanes, n), dtype=torch.float64, device=dev)

    def run_items(lo, hi):
        bse.solve_batched_device(meth, n, [d_in[i][0].data_ptr() for i in range(lo, hi)],
                                 [d_in[i][1].data_ptr() for i in range(lo, hi)],
                                 [d_lams[i].data_ptr() for i in range(lo, hi)],
                                 [d_vs[i % lanes].data_ptr() for i in range(lo, hi)], ctx=ctx)

    run_items(0, args.warmup * lanes)
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    launches0 = ctx.kernel_launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        run_items(args.warmup * lanes, total)
        if world > 1:  # every matrix's eigenvalues to every rank
            with torch.cuda.stream(stream):
                dist.all_gather_into_tensor(lam_all, torch.stack(d_lams[args.warmup * lanes:]))
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = ctx.kernel_launches() - launches0
    phase_hist = [ctx.phase_times()]  # lane 0's last solve, with per-kernel event timings
    # untimed check of the last timed matrix on the device: residual / (||H||_F ||x||) and
    # ||V^H Sigma V - I||_F (verify.cpp:70-93; the same bounds as the parity tests)
    last = total - 1
    res_dev = torch.empty(n, dtype=torch.float64, device=dev)
    bse.residual_device(n, d_in[last][0].data_ptr(), d_in[last][1].data_ptr(), n,
                        d_lams[last].data_ptr(), d_vs[last % lanes].data_ptr(),
                        res_dev.data_ptr(), ctx=ctx)
    check = {"item_seed": seeds[last % pool],
             "residual_max": (res_dev / torch.linalg.vector_norm(d_vs[last % lanes], dim=1)).max().item(),
             "residual_bound": 100 * n * float(np.finfo(float).eps),
             "sigma_dev": bse.sigma_orthogonality_error_device(2 * n, n, d_vs[last % lanes].data_ptr(),
                                                               ctx=ctx)}
    check["ok"] = bool(check["residual_max"] <= check["residual_bound"])
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = world * lanes * flops(method, n) / (ms_per_step / 1e3) / 1e12
    # latency of one solve alone (whole GPU, no concurrent lane), for reference
    torch.cuda.synchronize()
    l0 = torch.cuda.Event(enable_timing=True)
    l1 = torch.cuda.Event(enable_timing=True)
    l0.record(stream)
    for i in range(2):
        bse.solve_device(meth, n, d_in[i][0].data_ptr(), d_in[i][1].data_ptr(),
                         d_lams[i].data_ptr(), d_vs[0].data_ptr(), ctx=ctx)
    l1.record(stream)
    torch.cuda.synchronize()
    single_ms = l0.elapsed_time(l1) / 2
    ph_single = ctx.phase_times()  # per-kernel event timings of a solve that owns the GPU

    # ---- end to end through the host-pointer C-ABI: every step's inputs go H2D from pinned
    # host memory and its (lambda, V) come back D2H inside the timed region. Headline: the
    # config-5 batch driver bse_solve_batched (uploads/downloads overlap the neighbouring
    # solves); also reported: one bse_solve call per step (copies serialised with the solve,
    # V streamed back in chunks during the recovery stage).
    e2e = None
    if not args.no_e2e:
        ctx.set_kernel_timing(False)  # the user-facing calls run without per-kernel events
        import ctypes
        L = bse._lib.lib()
        st = bse.Status()
        nv = lanes  # pinned outputs: item i -> i % lanes (items of one lane run in order)
        hv = [torch.empty((n, 2 * n), dtype=torch.complex128).pin_memory() for _ in range(nv)]
        hl = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(nv)]
        ns = np.zeros((total, n), dtype=np.int64)
        nn = np.zeros(total, dtype=np.int64)
        failed = ctypes.c_int64(-1)

        def arr(ts):
            return (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])

        def batched(items):
            k = len(items)
            rc = L.bse_solve_batched(ctx.handle, int(meth), n, k, arr([x[0] for x in items]), n,
                                     arr([x[1] for x in items]), n,
                                     arr([hl[i % nv] for i in range(k)]),
                                     arr([hv[i % nv] for i in range(k)]), 2 * n,
                                     ns.ctypes.data_as(ctypes.c_void_p),
                                     nn.ctypes.data_as(ctypes.c_void_p), ctypes.byref(failed),
                                     ctypes.byref(st))
            if rc != 0:
                raise RuntimeError(st.message.decode())

        def single(ha, hb):
            c64 = ctypes.c_int64(0)
            rc = L.bse_solve(ctx.handle, int(meth), n, ctypes.c_void_p(ha.data_ptr()), n,
                             ctypes.c_void_p(hb.data_ptr()), n, ctypes.c_void_p(hl[0].data_ptr()),
                             ctypes.c_void_p(hv[0].data_ptr()), 2 * n,
                             ns.ctypes.data_as(ctypes.c_void_p), ctypes.byref(c64),
                             ctypes.byref(st))
            if rc != 0:
                raise RuntimeError(st.message.decode())

        def timed(fn):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ems = e0.elapsed_time(e1)
            if world > 1:
                t = torch.tensor([ems], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ems = float(t.item())
            return ems

        batched(host[: args.warmup * lanes])  # untimed: staging buffers, lane contexts
        ems = timed(lambda: batched(host[args.warmup * lanes: total]))
        for k in range(args.warmup):
            single(*host[k])
        ems1 = timed(lambda: [single(*host[args.warmup + k]) for k in range(args.steps)])
        e2e = {"value": world * lanes * flops(method, n) / (ems / args.steps / 1e3) / 1e12,
               "unit": "TFLOP/s", "h2d_bytes_per_step": lanes * 2 * n * n * 16,
               "d2h_bytes_per_step": lanes * (2 * n * n * 16 + n * 8),
               "ms_per_step": ems / args.steps,
               "path": f"bse_solve_batched over the K x {lanes} timed matrices ({lanes} lanes; "
                       "pinned host buffers; each lane uploads its next item and downloads its "
                       "previous one while it solves)",
               "single_call": {"value": world * flops(method, n) / (ems1 / args.steps / 1e3) / 1e12,
                               "ms_per_matrix": ems1 / args.steps,
                               "path": "one bse_solve per matrix, one matrix at a time (pinned; "
                                       "V streamed back in chunks)"}}

    # ---- roofline of the dominant kernel class from the live event timings
    peaks = load_peaks()
    fp64_peak = 37.0  # DMMA m8n8k4 issue-rate probe on this pool (tools/microbench/fp64_peak.cu)

    def roofline_of(ph, where):
        panel = {"ms": ph["panel_ms"], "launches": ph["panel_launches"], "bytes": ph["panel_bytes"]}
        gemm = {"ms": ph["gemm_ms"], "launches": ph["gemm_launches"], "flops": ph["gemm_flops"]}
        if panel["ms"] >= gemm["ms"]:
            ach = panel["bytes"] / (panel["ms"] / 1e3) / 1e9
            pk = peaks.get("hbm_gbs", 6650.0)
            rf = {"bound": "hbm",
                  "kernel": ("gebrd_panel_kernel" if method == "chol-svd" else "hetrd_panel_kernel")
                  + " (cooperative, TMA tile ring)",
                  "achieved": ach, "peak": pk, "unit": "GB/s", "frac": ach / pk, "traffic": None,
                  "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback",
                  "per_launch_ms": panel["ms"] / max(panel["launches"], 1),
                  "algorithmic_bytes_per_launch": panel["bytes"] / max(panel["launches"], 1)}
        else:
            ach = gemm["flops"] / (gemm["ms"] / 1e3) / 1e12
            rf = {"bound": "tensor", "kernel": "zgemm_dmma_kernel (DMMA.8x8x4, 3M)",
                  "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s", "frac": ach / fp64_peak,
                  "traffic": None,
                  "peak_source": "measured FP64 DMMA probe (MEASURED_PEAKS.json has no FP64)",
                  "per_launch_ms": gemm["ms"] / max(gemm["launches"], 1)}
        rf["measured"] = where
        try:
            with open(os.path.join(HERE, "profiles", "traffic.json")) as f:
                tr = json.load(f).get(rf["bound"], {})
            if rf["bound"] == "hbm" and "ratio" in tr:
                # ncu dram bytes / algorithmic bytes of one captured launch, applied per launch
                trk = tr.get("gebrd", tr) if method == "chol-svd" else tr
                rf["traffic"] = trk["ratio"] * rf["algorithmic_bytes_per_launch"]
                rf["traffic_source"] = trk.get("capture")
            if rf["bound"] == "tensor" and "bytes_per_flop" in tr:
                rf["traffic"] = tr["bytes_per_flop"] * gemm["flops"] / max(gemm["launches"], 1)
                rf["traffic_unit"] = "bytes per launch (DRAM read + write)"
                rf["traffic_source"] = tr.get("capture")
        except Exception:
            pass
        return rf, panel, gemm

    ph = phase_hist[-1]
    roofline, panel, gemm = roofline_of(
        ph, f"timed region, lane 0 of {lanes}: each panel kernel runs on 1/{lanes} of the SMs "
            f"beside the other lanes' work")
    roofline_whole, _, _ = roofline_of(ph_single, "single-solve pass: the kernel owns the GPU")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        cores = os.cpu_count() or 1
        oracle.set_threads(cores)
        # bounded sample (~10-30 s of CPU work): one full solve for CHOL; for CHOL+SVD the
        # oracle's zgesvd('A','A') needs ~10-40 min at n = 4096, so the sample is n = 1024
        n_cpu = n if method == "chol" else min(n, 1024)
        a, b = configs.config5(seeds[args.warmup % pool], n=n_cpu)
        t0 = time.perf_counter()
        oracle.solve(method, a, b)
        tc = time.perf_counter() - t0
        cpu = {"value": flops(method, n_cpu) / tc / 1e12, "unit": "TFLOP/s", "cores": cores,
               "kind": "port", "s_per_solve": tc, "n": n_cpu,
               "sample": f"one {method} solve of config-5 seed {seeds[args.warmup % pool]} "
                         f"(n={n_cpu}{'' if n_cpu == n else ', reduced from ' + str(n)}) with "
                         f"the oracle/ LAPACK restatement on {cores} host threads"}

    if rank == 0:
        line = {
            "metric": f"BSE eigensolve FP64 TFLOP/s (Table-1 flop model), n={n} c128, {method}",
            "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": f"config5: batch of 64 complex128 n={n} BSE matrices "
                                   f"(config-2 generator, seeds 0..63), {method}; each step every "
                                   f"GPU solves {lanes} matrices of its seed shard concurrently "
                                   "(bse_solve_batched_device, one lane per matrix)",
                       "n": n, "method": method, "batch": 64, "matrices_per_step_per_gpu": lanes,
                       "l2": "inputs 512 MiB per solve (> 126 MB L2); a pool of up to 8 "
                             "distinct matrices per rank, cycled",
                       "parallelism": f"dp{world} (seed partition, NCCL gathers eigenvalues)"},
            "s_per_solve": ms_per_step / 1e3 / lanes,
            "single_solve_latency_ms": single_ms,
            "batch64_s": ms_per_step / 1e3 / lanes * 64 / world,
            "fp64_frac_of_peak": value / (world * fp64_peak),
            "phase_ms": {k: round(v, 3) for k, v in ph_single.items()
                         if k in ("product_pair", "triple", "reduce", "tridiag", "backtransform",
                                  "recover", "total")},  # one solve alone on the whole GPU
            "phase_ms_batch_lane0": {k: round(v, 3) for k, v in ph.items()
                                     if k in ("product_pair", "triple", "reduce", "tridiag",
                                              "backtransform", "recover", "total")},
            "kernels": {"panel": panel, "gemm": gemm,
                        "gemm_tflops": gemm["flops"] / max(gemm["ms"], 1e-9) / 1e9},
            "roofline": roofline,
            "roofline_whole_gpu": roofline_whole,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "check": check,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
