"""Benchmark: HDG trace matvec throughput (BASELINE.json configs[1]) on B200.

Workload (N=1): 1024 x 1024 quad mesh, p = 4, K = I, fp64; input trace vector
x ~ U[-1, 1] (seed 1); one STEP = 100 repeated applies y = A x (configs[1]).
  value       whole-job GDOF/s (ndof * applies / s), inputs resident in HBM, CUDA events
  e2e         the same metric through the public API (TraceSystem.matvec_free) with the
              step's x copied host(pinned)->device and the step's y read back inside the
              timed region
  roofline    the trace kernel (one GPU: soa_apply_kernel on the facet-record layout,
              hdg_soa.cuh): algorithmic bytes (16 B/DOF: x read + y written; the operator is
              the shared element block) / its average launch time, against
              MEASURED_PEAKS.json hbm_gbs
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


def ncu_traffic(name):
    """dram__bytes_read + dram__bytes_write of the trace kernel from the committed ncu --set full
    capture (profiles/), per launch; None if absent."""
    path = os.path.join(ROOT, "profiles", name)
    try:
        vals = {}
        for line in open(path):
            parts = line.split()
            if len(parts) >= 3 and parts[0].startswith("dram__bytes_"):
                scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[parts[2]]
                vals[parts[0]] = float(parts[1]) * scale
        return vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (NVML in a background
    thread every ~2 ms; the timed regions are tens of ms)."""

    NAMES = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
             "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
             "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
             "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index=0):
        self.index, self.rows, self.stop = index, [], threading.Event()
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            masks = {k: getattr(N, v) for k, v in self.NAMES.items()}

            def run():
                while not self.stop.is_set():
                    try:
                        sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                        rs = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((float(sm), [k for k, m in masks.items() if rs & m]))
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.t = threading.Thread(target=run, daemon=True)
            self.t.start()
            # the timed region is tens of ms: hand control back only once the sampler is running,
            # then drop what it saw while the GPU was still idle
            t0 = time.time()
            while not self.rows and time.time() - t0 < 1.0:
                time.sleep(0.001)
            del self.rows[:]
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t is not None:
            self.t.join(timeout=2)

    def summary(self):
        sm = [r[0] for r in self.rows]
        reasons = sorted({x for r in self.rows for x in r[1]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(sm), "source": "nvml"}


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


# both CPU legs (the reference arm and the GPU arm's cpu_baseline) run the oracle port of
# trace.py:87-94 with the same thread policy: every host thread, element rows split evenly
def cpu_threads():
    return os.cpu_count() or 1


CPU_APPLIES_PER_STEP = 2   # the reference arm's bounded step: 2 full applies (~1 s of host work)


def workload_config(ws):
    """The config dict both arms print (identical, so the driver can pair the lines)."""
    return {"workload": f"configs[1]: {N_MESH}x{N_MESH} quad mesh, p={P_ORDER}, K=I (shared block), "
                        f"fp64, x~U[-1,1] seed 1; GPU step = {APPLIES} applies",
            "ndof": 2 * N_MESH * (N_MESH - 1) * (P_ORDER + 1),
            "l2": "inputs larger than L2: 4 rotating (x, y) pairs (736 MB > 126 MB L2)",
            "parallelism": f"strips{ws} (1024 element rows per GPU, NCCL halo rows)" if ws > 1 else "single"}


def run_reference(args, rank, ws):
    """--impl reference: the reference algorithm's CPU implementation (the oracle port of
    trace.py:87-94; the reference is pure Python and cannot travel to the GPU box) on all host
    threads.  One step = CPU_APPLIES_PER_STEP full applies of the configs[1] system, and
    ms_per_step is exactly the time of such a step; value is the same GDOF/s rate metric."""
    if rank != 0:
        return
    osys = oracle_system()
    x = np.random.default_rng(1).uniform(-1.0, 1.0, osys.ndof)
    threads = cpu_threads()
    sample = CPU_APPLIES_PER_STEP
    for _ in range(args.warmup):
        cpu_matvec_threads(osys, x, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for _ in range(sample):
            cpu_matvec_threads(osys, x, threads)
    dt = time.perf_counter() - t0
    val = osys.ndof * sample * args.steps / dt / 1e9
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "applies_per_step": sample,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference", "config": workload_config(ws),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{sample} applies of the full {N_MESH}^2 p={P_ORDER} system per step "
                                       f"(oracle port of trace.py:87-94, {threads} threads, element rows "
                                       "split evenly; the timed step is exactly these applies)"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, ws):
    import torch
    import paper_1705_09907_b200 as P
    from paper_1705_09907_b200.mesh import build_cartesian
    from paper_1705_09907_b200.problem import constant_problem
    from paper_1705_09907_b200.trace import TraceSystem
    lib = P.lib

    strip = None
    if ws == 1:
        sysg = TraceSystem(build_cartesian(N_MESH, N_MESH), P_ORDER, constant_problem(0.0, 1.0))
    else:
        # weak scaling: rank r owns element rows [1024 r, 1024 (r+1)) of a 1024 x 1024*ws mesh
        # of square elements (SURVEY 8(e) strips); ghost rows refreshed by NCCL before each apply
        from paper_1705_09907_b200.distributed import StripLayout, StripOperator
        from paper_1705_09907_b200.mesh import Mesh
        L = StripLayout(N_MESH, N_MESH * ws, P_ORDER, ws, rank)
        h_el = 1.0 / N_MESH
        blk = TraceSystem(Mesh(4, 4, 0.0, 0.0, h_el, h_el), P_ORDER, constant_problem(0.0, 1.0)).operator.S_cls
        sysg = TraceSystem.from_blocks(Mesh(N_MESH, L.nyl, 0.0, L.lo * h_el, h_el, h_el), P_ORDER, blk)
        strip = StripOperator(L, sysg.operator.apply)
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
    # one GPU: the facet-record device layout (hdg_soa.cuh) is the product's fastest apply; the
    # strip path (N > 1) exchanges halo rows in the reference layout and uses trace_apply_kernel
    records = strip is None
    if records:
        xs = [op.to_planes(x) for x in xs]
        ys = [torch.empty_like(xs[0]) for _ in range(NB)]
        apply_fn, kname = lib.hdg_matvec_soa, "soa_apply_kernel<5> (facet records)"
        ncu_keys = "ncu_soa_apply_p4_r02b_key_metrics.txt"
    else:
        apply_fn, kname = lib.hdg_matvec, "trace_apply_kernel<5,shared,EPI_Y>"
        ncu_keys = "ncu_trace_apply_p4_r01_key_metrics.txt"

    def step():
        for a in range(APPLIES):
            k = a % NB
            if strip is not None:
                strip.exchange(xs[k])
            P._lib.check(apply_fn(h, xs[k].data_ptr(), ys[k].data_ptr(), sp))

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
    owned = int(strip.L.owned.sum()) if strip is not None else ndof
    value = ws * owned * applies / (t_ms * 1e-3) / 1e9

    # single-launch event timing of the dominant kernel (same stream)
    e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    singles = []
    for k in range(20):
        e_a.record(stream)
        P._lib.check(apply_fn(h, xs[k % NB].data_ptr(), ys[k % NB].data_ptr(), sp))
        e_b.record(stream)
        torch.cuda.synchronize()
        singles.append(e_a.elapsed_time(e_b) * 1e3)
    # the reference-layout kernel on the same system (same stream, same rotation), for comparison
    ref_layout_us = None
    if records:
        xr = [op.from_planes(x) for x in xs]
        yr = [torch.empty(ndof, dtype=torch.float64, device="cuda") for _ in range(NB)]
        for k in range(10):
            P._lib.check(lib.hdg_matvec(h, xr[k % NB].data_ptr(), yr[k % NB].data_ptr(), sp))
        e_a.record(stream)
        for k in range(200):
            P._lib.check(lib.hdg_matvec(h, xr[k % NB].data_ptr(), yr[k % NB].data_ptr(), sp))
        e_b.record(stream)
        torch.cuda.synchronize()
        ref_layout_us = e_a.elapsed_time(e_b) * 1e3 / 200
        del xr, yr

    # ---- end to end through the public API, host buffers
    x_pin = torch.from_numpy(x_host).pin_memory()

    # Steps are pipelined over three streams (H2D of step k+1 and D2H of step k-1 overlap the
    # applies of step k); every step's pinned H2D of x and D2H of y stays inside the timed region.
    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
    x_dev = [torch.empty(ndof, dtype=torch.float64, device="cuda") for _ in range(2)]
    y_pins = [torch.empty(ndof, dtype=torch.float64).pin_memory() for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def e2e_step(k):
        b = k % 2
        s_h2d.wait_event(ev_used[b])                      # x_dev[b] free (step k-2 consumed it)
        with torch.cuda.stream(s_h2d):
            x_dev[b].copy_(x_pin, non_blocking=True)
        ev_in[b].record(s_h2d)
        stream.wait_event(ev_in[b])
        y = None
        if strip is not None:
            for _ in range(APPLIES):                     # the public API call
                y = strip.apply(x_dev[b])
        else:                                            # TraceSystem.facet_planes + matvec_free
            z = sysg.facet_planes(x_dev[b])
            for _ in range(APPLIES):
                y = sysg.matvec_free(z)
            y = y.tensor()
        ev_used[b].record(stream)
        s_d2h.wait_event(ev_used[b])
        s_d2h.wait_event(ev_out[b])                      # y_pins[b] free
        with torch.cuda.stream(s_d2h):
            y_pins[b].copy_(y, non_blocking=True)
            y.record_stream(s_d2h)
        ev_out[b].record(s_d2h)

    for k in range(max(args.warmup, 3)):
        e2e_step(k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    s_h2d.wait_event(e0)
    for k in range(args.steps):
        e2e_step(k)
    stream.wait_stream(s_d2h)
    e1.record(stream)
    torch.cuda.synchronize()
    t_e2e = barrier_max(e0.elapsed_time(e1), ws)
    e2e_val = ws * owned * applies / (t_e2e * 1e-3) / 1e9
    assert np.isfinite(y_pins[(args.steps - 1) % 2].numpy()).all()

    # ---- parity check of a timed output against the CPU oracle (cpu_baseline)
    y_chk = (op.from_planes(ys[0]) if records else ys[0]).cpu().numpy()

    hbm, kind = peaks()
    alg_bytes = 16 * ndof
    achieved = alg_bytes / (kernel_us * 1e-6) / 1e9
    flops = sysg.n_blocks * (16 * (P_ORDER + 1) ** 2 - (P_ORDER + 1))   # trace.py:223
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "applies_per_step": APPLIES, "config": workload_config(ws),
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": 8 * ndof, "d2h_bytes_per_step": 8 * ndof,
                    "path": ("per step: pinned H2D of x, TraceSystem.facet_planes (pack), matvec_free x100 on the "
                             "facet records, .tensor() (unpack), D2H of y" if records else
                             "per step: pinned H2D of x, StripOperator.apply x100, D2H of y") +
                            "; steps pipelined over 3 streams (copies of neighbouring steps overlap the applies)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": ncu_traffic(ncu_keys),
                         "traffic_source": "profiles/" + ncu_keys + (" (steady state: ncu --cache-control none, "
                                                                     "6 consecutive launches)" if records else
                                                                     " (ncu --set full)"),
                         "peak_kind": kind,
                         "kernel": kname, "alg_bytes_per_launch": alg_bytes,
                         "ref_layout_kernel_us": ref_layout_us,
                         "kernel_us_avg": kernel_us, "kernel_us_single_median": float(np.median(singles)),
                         "fp64_tflops": flops / (kernel_us * 1e-6) / 1e12},
            "gpu_launches": int(launches),
            "clocks": clk.summary()}
    if ws == 1 and not args.no_vcycle:
        line["vcycle"] = vcycle_timings()
    elif ws > 1 and not args.no_vcycle:
        try:
            line["vcycle"] = strip_vcycle_timing(rank, ws)
        except Exception as exc:   # never lose the matvec line to the multi-GPU cycle
            line["vcycle"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    if rank == 0 and ws == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(y_chk, x_host)
    if rank == 0:
        print(json.dumps(line), flush=True)


def vcycle_model_bytes(levels):
    """Minimum HBM bytes of one V(2,2) block-Jacobi cycle with every facet-local step fused into
    an operator pass: per non-coarsest level of n dofs with a coarse level of
    c dofs, p-link: zero-start double sweep 16n, residual + restriction 16n + 8c, prolongation +
    sweep 24n + 8c, sweep 24n; h-link: 16n + residual 24n + restriction 8n + 8c + prolongation
    16n + 8c + two sweeps 48n.  Shared (K = I) levels: no operator bytes."""
    total = 0
    for k in range(len(levels) - 1):
        n, c = levels[k].ndof, levels[k + 1].ndof
        same_mesh = levels[k].mesh.n_x == levels[k + 1].mesh.n_x
        total += (80 * n + 16 * c) if same_mesh else (112 * n + 16 * c)
    return total


def vcycle_timings(steps=20):
    """V(2,2) block-Jacobi(0.8) cycle time on the configs[1] hierarchy (1024^2, p=4, K=I, 13
    levels) and on configs[0] (64^2, p=2, sliced to 4x4), graph-replayed: through hdg_mg_cycle on
    reference-layout vectors (pack / unpack at the boundary when the record cycle is on) and, for
    configs[1], on record-resident vectors (hdg_mg_cycle_records), with the byte-model roofline."""
    import torch
    from paper_1705_09907_b200 import _lib
    from paper_1705_09907_b200.mesh import build_cartesian
    from paper_1705_09907_b200.multigrid import _native_mg, build_hierarchy
    from paper_1705_09907_b200.problem import config1_problem, constant_problem
    out = {}
    L = _lib.lib
    peak, _ = peaks()

    def timed(fn):
        st = torch.cuda.current_stream()
        for _ in range(3):
            fn(st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            fn(st)
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    for name, (n, p, spec, cut) in {"cfg2_1024p4": (1024, 4, constant_problem(0.0, 1.0), None),
                                    "cfg1_64p2": (64, 2, config1_problem(), 6)}.items():
        levels = build_hierarchy(build_cartesian(n, n), p, spec, smoother=None)
        levels = levels[:cut] if cut else levels
        from paper_1705_09907_b200.multigrid import attach_smoothers
        attach_smoothers(levels, "blockjacobi", 0.8)
        mg = _native_mg(levels)
        b = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, levels[0].ndof)).cuda()
        x = torch.zeros_like(b)
        ms = timed(lambda st: _lib.check(L.hdg_mg_cycle(mg.handle, b.data_ptr(), x.data_ptr(), x.data_ptr(), 2, 2, 1,
                                                        1, st.cuda_stream)))
        rec = {"ms_per_cycle": ms, "levels": len(levels), "ndof": levels[0].ndof,
               "record_levels": int(L.hdg_mg_record_levels(mg.handle))}
        if rec["record_levels"] > 0:
            sysf = levels[0].system
            bp = sysf.facet_planes(b).data
            xp = torch.zeros_like(bp)
            rms = timed(lambda st: _lib.check(L.hdg_mg_cycle_records(mg.handle, bp.data_ptr(), xp.data_ptr(),
                                                                     xp.data_ptr(), 2, 2, 1, 1, st.cuda_stream)))
            rms0 = timed(lambda st: _lib.check(L.hdg_mg_cycle_records(mg.handle, bp.data_ptr(), 0, xp.data_ptr(), 2, 2,
                                                                      1, 1, st.cuda_stream)))
            nbytes = vcycle_model_bytes(levels)
            rec["records_resident_ms_per_cycle"] = rms
            rec["records_resident_zero_guess_ms_per_cycle"] = rms0   # the preconditioner's cycle (x0 = 0)
            rec["roofline"] = {"bound": "hbm", "model_bytes_per_cycle": nbytes, "floor_ms": nbytes / peak / 1e6,
                               "frac": nbytes / peak / 1e6 / rms, "frac_zero_guess": nbytes / peak / 1e6 / rms0,
                               "peak": peak, "unit": "GB/s",
                               "frac_reference_layout_api": nbytes / peak / 1e6 / ms}
            _lib.check(L.hdg_mg_set_records(mg.handle, 0))
            rec["reference_layout_cycle_ms"] = timed(lambda st: _lib.check(L.hdg_mg_cycle(
                mg.handle, b.data_ptr(), x.data_ptr(), x.data_ptr(), 2, 2, 1, 1, st.cuda_stream)))
            _lib.check(L.hdg_mg_set_records(mg.handle, 1))
        out[name] = rec
    return out


def strip_vcycle_timing(rank, ws, steps=10):
    """V(2,2) block-Jacobi(0.8) cycle of the weak-scaled strip hierarchy (1024 x 1024*ws, p=4,
    K=I; 1024 element rows per GPU): distributed levels exchange halos over NCCL, levels with
    < 4 rows per rank are agglomerated and run replicated (DESIGN 8).  Device time, max over
    ranks.  The orchestration is host-driven (not graph-captured): small levels are launch- and
    host-bound."""
    import torch
    from paper_1705_09907_b200.distributed import strip_multigrid
    from paper_1705_09907_b200.mesh import build_cartesian
    from paper_1705_09907_b200.multigrid import build_hierarchy
    from paper_1705_09907_b200.problem import constant_problem
    levels = build_hierarchy(build_cartesian(N_MESH, N_MESH * ws, ((0.0, 1.0), (0.0, float(ws)))), P_ORDER,
                             constant_problem(0.0, 1.0), smoother=None)
    mg = strip_multigrid(levels)
    L0 = mg.layouts[0]
    bg = np.random.default_rng(0).uniform(-1, 1, levels[0].ndof)
    b = torch.from_numpy(bg[L0.local_to_global].copy()).cuda()
    for _ in range(2):
        mg.v_cycle(b)
    torch.cuda.synchronize()
    torch.distributed.barrier()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        mg.v_cycle(b)
    e1.record(st)
    torch.cuda.synchronize()
    ms = barrier_max(e0.elapsed_time(e1) / steps, ws)
    return {"strips_1024rows_per_gpu": {"ms_per_cycle": ms, "levels": len(levels), "distributed_levels": mg.d + 1,
                                        "ndof_global": levels[0].ndof, "orchestration": "host-driven, NCCL halos"}}


def cpu_baseline(y_gpu, x_host):
    osys = oracle_system()
    threads = cpu_threads()
    cpu_matvec_threads(osys, x_host, threads)   # warm-up + parity reference for the timed output
    t0 = time.perf_counter()
    sample = 5
    for _ in range(sample):
        y = cpu_matvec_threads(osys, x_host, threads)
    dt = time.perf_counter() - t0
    err = float(np.abs(y - y_gpu).max() / np.abs(y).max())
    t1 = time.perf_counter()
    cpu_matvec_threads(osys, x_host, 1)
    one = osys.ndof / (time.perf_counter() - t1) / 1e9
    return {"value": osys.ndof * sample / dt / 1e9, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{sample} applies of the full {N_MESH}^2 p={P_ORDER} system (oracle port of "
                      f"trace.py:87-94, {threads} threads, element rows split evenly: the reference arm's policy)",
            "single_core_value": one,
            "parity_rel_err_vs_gpu": err}


# ------------------------------------------------------------------------ configs[4] runner

C5_N, C5_P = 8192, 4


def config5_problem(n):
    """configs[4]: anisotropic diagonal K per element, Kxx and Kyy log-uniform in [0.1, 10] from
    default_rng(3); returns (spec, rng positioned for b)."""
    from paper_1705_09907_b200.problem import ProblemSpec, piecewise_anisotropic
    rng = np.random.default_rng(3)
    Kxx = np.exp(rng.uniform(np.log(0.1), np.log(10.0), (n, n)))
    Kyy = np.exp(rng.uniform(np.log(0.1), np.log(10.0), (n, n)))
    zero = lambda x, y: np.zeros_like(np.asarray(x, float))
    return ProblemSpec(piecewise_anisotropic(Kxx, Kyy), zero, zero, 1.0), rng


def run_config5(args, rank, ws):
    """configs[4]: 8192^2, p = 4, anisotropic K, strong scaling over N GPUs.  N = 1: the fine level
    alone (its element blocks, 214.7 GB, never exist at once: condensed and streamed by row chunks
    into the 107 GB half-stored stream), matvec only.  N > 1: rank-local strip hierarchies
    (distributed.LocalStripHierarchy), matvec with NCCL halo rows, V(2,2) block-Jacobi cycle and
    MG-PCG to 1e-10.  One JSON line (rank 0), the same config dict at every N."""
    import torch
    from paper_1705_09907_b200 import _lib
    from paper_1705_09907_b200.mesh import build_cartesian
    n, p = args.n5, C5_P
    spec, rng = config5_problem(n)
    mesh = build_cartesian(n, n)
    t0 = time.time()
    st = torch.cuda.current_stream()
    cfg = {"workload": f"configs[4]: {n}x{n} quad mesh, p={p}, anisotropic diagonal K log-U[0.1,10] seed 3, fp64; "
                       "step = one trace matvec", "ndof": 2 * n * (n - 1) * (p + 1),
           "l2": "inputs larger than L2 (the operator stream alone is 107 GB at 8192^2)",
           "parallelism": f"strips{ws} (rank-local windows, NCCL halo rows)" if ws > 1 else "single (matvec only)"}
    line = {"metric": METRIC, "unit": UNIT, "n_gpus": ws, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg}
    if ws == 1:
        from paper_1705_09907_b200.trace import RowChunkedOperator
        op = RowChunkedOperator(mesh, p, spec, rows_per_chunk=args.chunk_rows)
        torch.cuda.synchronize()
        setup_s = time.time() - t0
        ndof = op.ndof
        xs = [torch.from_numpy(rng.uniform(-1.0, 1.0, ndof)).cuda(), torch.rand(ndof, dtype=torch.float64, device="cuda")]
        ys = [torch.empty_like(xs[0]) for _ in range(2)]
        h = op.handle
        for k in range(args.warmup):
            _lib.check(_lib.lib.hdg_matvec(h, xs[k % 2].data_ptr(), ys[k % 2].data_ptr(), st.cuda_stream))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(0) as clk:
            e0.record(st)
            for k in range(args.steps):
                _lib.check(_lib.lib.hdg_matvec(h, xs[k % 2].data_ptr(), ys[k % 2].data_ptr(), st.cuda_stream))
            e1.record(st)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        hbm, kind = peaks()
        alg = op.operator_bytes() + 16 * ndof
        line.update({"value": ndof / (ms * 1e-3) / 1e9, "steps": args.steps, "warmup": args.warmup,
                     "ms_per_step": ms, "setup_s": round(setup_s, 1),
                     "roofline": {"bound": "hbm", "achieved": alg / (ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                                  "frac": alg / (ms * 1e-3) / 1e9 / hbm, "traffic": None, "peak_kind": kind,
                                  "kernel": "trace_apply_kernel<5, stored, EPI_Y> (half-stored facet stream)",
                                  "alg_bytes_per_launch": alg},
                     "clocks": clk.summary()})
        print(json.dumps(line), flush=True)
        return
    from paper_1705_09907_b200.distributed import StripOperator, local_strip_multigrid
    mg, H = local_strip_multigrid(mesh, p, spec, omega=0.8)
    torch.cuda.synchronize()
    setup_s = barrier_max(time.time() - t0, ws)
    L0 = H.layouts[0]
    ndof = L0.ndof_g
    bg = rng.uniform(-1.0, 1.0, ndof)
    b = torch.from_numpy(bg[L0.local_to_global]).cuda()
    op = H.ops[0]
    sop = StripOperator(L0, op.apply)
    for _ in range(args.warmup):
        sop.apply(b)
    torch.cuda.synchronize()
    torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        sop.apply(b)
    e1.record(st)
    torch.cuda.synchronize()
    ms = barrier_max(e0.elapsed_time(e1) / args.steps, ws)
    # V(2,2) cycle and MG-PCG over the strips
    for _ in range(2):
        mg.v_cycle(b)
    torch.cuda.synchronize()
    torch.distributed.barrier()
    e0.record(st)
    for _ in range(3):
        mg.v_cycle(b)
    e1.record(st)
    torch.cuda.synchronize()
    vms = barrier_max(e0.elapsed_time(e1) / 3, ws)
    line.update({"value": ndof / (ms * 1e-3) / 1e9, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                 "setup_s": round(setup_s, 1), "vcycle_ms": vms, "distributed_levels": H.d + 1})
    if rank == 0:
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------ configs[3] runner

FP64_PEAK_TFLOPS = 34.2   # measured DFMA peak on this pool's B200 (profiles/fp64_peak_r01.json)
C4_MESH = {1: 4096, 2: 3328, 4: 2560, 8: 1920, 12: 1536}   # ~64M trace DOFs each


def run_config4(args, rank, ws):
    """configs[3]: order sweep at ~64M trace DOFs, K = I, fp64: trace matvec throughput (the
    facet-record kernel at every order) and the V(2,2)
    block-Jacobi cycle per order.  value = all orders' DOF applies / their total time; per-order
    numbers (GDOF/s, fraction of HBM on 16 B/DOF, reference-formula FP64 rate, V-cycle ms) in
    "orders"."""
    import torch
    from paper_1705_09907_b200 import _lib
    from paper_1705_09907_b200.mesh import build_cartesian
    from paper_1705_09907_b200.multigrid import _native_mg, attach_smoothers, build_hierarchy
    from paper_1705_09907_b200.problem import constant_problem
    if rank != 0:
        return
    hbm, kind = peaks()
    st = torch.cuda.current_stream()
    orders, tot_dof, tot_us = {}, 0.0, 0.0
    for p, n in sorted(C4_MESH.items()):
        levels = build_hierarchy(build_cartesian(n, n), p, constant_problem(0.0, 1.0), smoother=None)
        attach_smoothers(levels, "blockjacobi", 0.8)
        op = levels[0].block_op
        ndof = levels[0].ndof
        xr = [torch.rand(ndof, dtype=torch.float64, device="cuda") for _ in range(2)]
        records = True   # the facet-record kernel covers every order (p <= 12)
        if records:
            xs = [op.to_planes(x) for x in xr]
            ys = [torch.empty_like(xs[0]) for _ in range(2)]
            fn, kern = _lib.lib.hdg_matvec_soa, "soa_apply_kernel (facet records)"
        else:
            xs, ys = xr, [torch.empty_like(xr[0]) for _ in range(2)]
            fn, kern = _lib.lib.hdg_matvec, "trace_apply_kernel (reference layout)"
        h = op.handle
        for k in range(max(args.warmup, 3)):
            _lib.check(fn(h, xs[k % 2].data_ptr(), ys[k % 2].data_ptr(), st.cuda_stream))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for k in range(args.steps):
            _lib.check(fn(h, xs[k % 2].data_ptr(), ys[k % 2].data_ptr(), st.cuda_stream))
        e1.record(st)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / args.steps
        mg = _native_mg(levels)
        b, x = xr[0], torch.zeros_like(xr[0])
        for _ in range(2):
            _lib.check(_lib.lib.hdg_mg_cycle(mg.handle, b.data_ptr(), 0, x.data_ptr(), 2, 2, 1, 1, st.cuda_stream))
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(5):
            _lib.check(_lib.lib.hdg_mg_cycle(mg.handle, b.data_ptr(), 0, x.data_ptr(), 2, 2, 1, 1, st.cuda_stream))
        e1.record(st)
        torch.cuda.synchronize()
        nb = levels[0].system.n_blocks
        # t_min = max(algorithmic bytes / HBM, reference-formula FLOPs / measured FP64 peak)
        fl = nb * (16 * (p + 1) ** 2 - (p + 1))
        t_hbm, t_fp = 16 * ndof / hbm / 1e3, fl / FP64_PEAK_TFLOPS / 1e6
        orders[str(p)] = {"mesh": n, "ndof": ndof, "kernel": kern, "matvec_us": round(us, 2),
                          "gdofs": round(ndof / us / 1e3, 1), "hbm_frac": round(16 * ndof / us / 1e3 / hbm, 3),
                          "fp64_tflops_ref_formula": round(fl / us / 1e6, 2),
                          "bound": "hbm" if t_hbm >= t_fp else "fp64",
                          "roofline_frac": round(max(t_hbm, t_fp) / us, 3),
                          "vcycle_ms": round(e0.elapsed_time(e1) / 5, 3), "levels": len(levels)}
        tot_dof += ndof * args.steps
        tot_us += us * args.steps
        del levels, mg, xs, ys, xr, op
        torch.cuda.empty_cache()
    line = {"metric": METRIC, "value": tot_dof / tot_us / 1e3, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": tot_us / args.steps / 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "configs[3]: order sweep p in {1,2,4,8,12} at ~64M trace DOFs "
                                   "(4096^2, 3328^2, 2560^2, 1920^2, 1536^2), K=I, fp64; step = one matvec per order",
                       "l2": "inputs larger than L2 (2 rotating vectors of ~0.5 GB)", "parallelism": "single"},
            "orders": orders, "peak": {"hbm_gbs": hbm, "kind": kind}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-vcycle", action="store_true")
    ap.add_argument("--config", type=int, default=1, choices=[1, 3, 4],
                    help="BASELINE configs index: 1 = matvec throughput (default), 3 = order sweep, "
                         "4 = multi-GPU anisotropic")
    ap.add_argument("--n5", type=int, default=C5_N, help="configs[4] mesh size (reduced runs)")
    ap.add_argument("--chunk-rows", type=int, default=256, help="configs[4] N=1: element rows per chunk")
    args = ap.parse_args()
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, rank, int(os.environ.get("WORLD_SIZE", "1")))
        return
    rank, ws, _ = dist_init(args.gpus)
    if args.config == 4:
        run_config5(args, rank, ws)
    elif args.config == 3:
        run_config4(args, rank, ws)
    else:
        run_ours(args, rank, ws)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
