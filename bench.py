"""Benchmark: HDG trace matvec throughput (BASELINE.json configs[1]) on B200.

Workload (N=1): 1024 x 1024 quad mesh, p = 4, K = I, fp64; input trace vector
x ~ U[-1, 1] (seed 1); one STEP = 100 repeated applies y = A x (configs[1]).
  value       whole-job GDOF/s (ndof * applies / s), inputs resident in HBM, CUDA events
  e2e         the same metric through the public API (TraceSystem.matvec_free) with the
              step's x copied host(pinned)->device and the step's y read back inside the
              timed region
  roofline    the trace kernel: algorithmic bytes (16 B/DOF: x read + y written; the
              operator is the shared block held in the constant bank) / its average
              launch time, against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline the CPU oracle port of trace.py:87-94 (gather, einsum, two-owner sum)
              on a bounded sample of applies on the same system, rank 0
L2 policy: the applies rotate over 4 (x, y) pairs = 670 MB > 126 MB L2, so no apply
reads an x that a recent apply left in L2.

--impl reference: times the reference algorithm's CPU implementation (the oracle port
of trace.py:87-94; the reference is pure Python and cannot travel) with all host
threads, same metric/config; rank 0 only.
"""

from __future__ import annotations

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

N_MESH, P_ORDER, APPLIES = 1024, 4, 100
METRIC = "trace_matvec_gdof_per_s"
UNIT = "GDOF/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_init(n_gpus):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, ws, local


def barrier_max(t_ms, ws):
    if ws == 1:
        return t_ms
    import torch
    import torch.distributed as dist
    v = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(v, op=dist.ReduceOp.MAX)
    return float(v.item())


def oracle_system():
    from oracle import hdg_oracle as O
    return O.injected_shared_system(N_MESH, P_ORDER)


def cpu_matvec_threads(osys, x, threads):
    """Oracle port of trace.py:87-94 split over element row blocks (einsum releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    E = osys.grid.n_elems
    chunks = np.array_split(np.arange(E), threads)
    xe = np.where(osys.gmask, x[osys.gidx], 0.0)
    ye = np.empty_like(xe)

    def work(idx):
        ye[idx] = np.einsum("eij,ej->ei", osys.schur[idx], xe[idx])

    if threads == 1:
        work(np.arange(E))
    else:
        with ThreadPoolExecutor(threads) as pool:
            list(pool.map(work, chunks))
    return osys._sum_owners(ye)


def run_reference(args, rank, ws):
    if rank != 0:
        return
    osys = oracle_system()
    x = np.random.default_rng(1).uniform(-1.0, 1.0, osys.ndof)
    threads = os.cpu_count() or 1
    sample = 2  # applies per step (bounded sample of the 100-apply step)
    for _ in range(args.warmup):
        cpu_matvec_threads(osys, x, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for _ in range(sample):
            cpu_matvec_threads(osys, x, threads)
    dt = time.perf_counter() - t0
    val = osys.ndof * sample * args.steps / dt / 1e9
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3 * APPLIES / sample,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"configs[1]: {N_MESH}x{N_MESH} quad mesh, p={P_ORDER}, K=I, fp64, "
                                   f"{APPLIES} applies/step", "ndof": osys.ndof},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{sample} applies of the full {N_MESH}^2 p={P_ORDER} system per step "
                                       f"(oracle port of trace.py:87-94, {threads} threads)"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, ws):
    import torch
    import paper_1705_09907_b200 as P
    from paper_1705_09907_b200.mesh import build_cartesian
    from paper_1705_09907_b200.problem import constant_problem
    from paper_1705_09907_b200.trace import TraceSystem
    lib = P.lib

    sysg = TraceSystem(build_cartesian(N_MESH, N_MESH), P_ORDER, constant_problem(0.0, 1.0))
    ndof = sysg.ndof
    op = sysg.operator
    h = op.handle
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    rng = np.random.default_rng(1)
    x_host = rng.uniform(-1.0, 1.0, ndof)
    NB = 4
    xs = [torch.from_numpy(x_host).cuda()] + \
         [torch.from_numpy(np.random.default_rng(1 + k).uniform(-1, 1, ndof)).cuda() for k in range(1, NB)]
    ys = [torch.empty(ndof, dtype=torch.float64, device="cuda") for _ in range(NB)]

    def step():
        for a in range(APPLIES):
            k = a % NB
            P._lib.check(lib.hdg_matvec(h, xs[k].data_ptr(), ys[k].data_ptr(), sp))

    # ---- device-resident throughput
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    c0 = lib.hdg_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = lib.hdg_launch_count() - c0
    t_ms = barrier_max(ev0.elapsed_time(ev1), ws)
    applies = APPLIES * args.steps
    kernel_us = t_ms * 1e3 / applies
    value = ws * ndof * applies / (t_ms * 1e-3) / 1e9

    # single-launch event timing of the dominant kernel (same stream)
    e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    singles = []
    for k in range(20):
        e_a.record(stream)
        P._lib.check(lib.hdg_matvec(h, xs[k % NB].data_ptr(), ys[k % NB].data_ptr(), sp))
        e_b.record(stream)
        torch.cuda.synchronize()
        singles.append(e_a.elapsed_time(e_b) * 1e3)

    # ---- end to end through the public API, host buffers
    x_pin = torch.from_numpy(x_host).pin_memory()
    y_pin = torch.empty(ndof, dtype=torch.float64).pin_memory()

    def e2e_step():
        xd = x_pin.to("cuda", non_blocking=True)
        y = None
        for _ in range(APPLIES):
            y = sysg.matvec_free(xd)
        y_pin.copy_(y, non_blocking=True)

    for _ in range(max(args.warmup, 3)):
        e2e_step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    t_e2e = barrier_max(e0.elapsed_time(e1), ws)
    e2e_val = ws * ndof * applies / (t_e2e * 1e-3) / 1e9

    # ---- parity spot check of the timed output against the host formula (cheap, sampled)
    y_chk = ys[0].cpu().numpy()

    hbm, kind = peaks()
    alg_bytes = 16 * ndof
    achieved = alg_bytes / (kernel_us * 1e-6) / 1e9
    flops = sysg.n_blocks * (16 * (P_ORDER + 1) ** 2 - (P_ORDER + 1))   # trace.py:223
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"configs[1]: {N_MESH}x{N_MESH} quad mesh, p={P_ORDER}, K=I (shared block), "
                                   f"fp64, {APPLIES} applies/step, x~U[-1,1] seed 1",
                       "ndof": ndof, "l2": "rotating 4 (x,y) pairs = %.0f MB > 126 MB L2" % (NB * 16 * ndof / 1e6),
                       "parallelism": "replicas" if ws > 1 else "single"},
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": 8 * ndof, "d2h_bytes_per_step": 8 * ndof,
                    "path": "TraceSystem.matvec_free(cuda tensor) x100 after pinned H2D of x; D2H of y"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": None, "peak_kind": kind,
                         "kernel": "trace_apply_kernel<5,shared,EPI_Y>", "alg_bytes_per_launch": alg_bytes,
                         "kernel_us_avg": kernel_us, "kernel_us_single_median": float(np.median(singles)),
                         "fp64_tflops": flops / (kernel_us * 1e-6) / 1e12},
            "gpu_launches": int(launches),
            "clocks": clk.summary()}
    if rank == 0 and ws == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(y_chk, x_host)
    if rank == 0:
        print(json.dumps(line), flush=True)


def cpu_baseline(y_gpu, x_host):
    osys = oracle_system()
    cpu_matvec_threads(osys, x_host, 1)   # warm-up + parity reference for the timed output
    t0 = time.perf_counter()
    sample = 5
    for _ in range(sample):
        y = cpu_matvec_threads(osys, x_host, 1)
    dt = time.perf_counter() - t0
    err = float(np.abs(y - y_gpu).max() / np.abs(y).max())
    return {"value": osys.ndof * sample / dt / 1e9, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{sample} applies of the full {N_MESH}^2 p={P_ORDER} system (oracle port of "
                      f"trace.py:87-94, single-threaded numpy like the reference)",
            "parity_rel_err_vs_gpu": err}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, rank, int(os.environ.get("WORLD_SIZE", "1")))
        return
    rank, ws, _ = dist_init(args.gpus)
    run_ours(args, rank, ws)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
