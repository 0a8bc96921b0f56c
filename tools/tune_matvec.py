"""Tuning harness: time trace matvecs (cfg2 1024^2 p=4 K=I shared, stored p=4/p=8, p=1, p=8)
for each library variant given on the command line (paths to .so files)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys, json
sys.path.insert(0, %r)
import numpy as np, torch
from paper_1705_09907_b200.mesh import build_cartesian
from paper_1705_09907_b200.problem import constant_problem
from paper_1705_09907_b200.trace import TraceSystem
import paper_1705_09907_b200._lib as L
out = {"lib": os.path.basename(os.environ["HDGB200_LIB"])}
# parity spot check of this variant (host formula of trace.py:87-94 with the same blocks)
errs = []
for (n, p) in [(37, 4), (40, 1), (33, 8), (35, 2)]:
    m = build_cartesian(n, n + 3)
    s = TraceSystem(m, p, constant_problem(0.0, 1.0))
    x = np.random.default_rng(p).uniform(-1, 1, s.ndof)
    lay = s.layout
    S = s.operator.S_cls[0]
    ref = lay.sum_owners(np.einsum("ij,ej->ei", S, lay.gather(x) * np.repeat(lay.side_mask(), p + 1, axis=1)))
    errs.append(float(np.abs(s.matvec_free(x) - ref).max() / np.abs(ref).max()))
out["parity_max_rel_err"] = max(errs)
cases = [tuple(c) for c in json.loads(os.environ.get("TUNE_CASES", "null"))] if os.environ.get("TUNE_CASES") else [(1024, 4, False), (512, 4, True), (1024, 1, False), (768, 8, False), (384, 8, True)]
for (n, p, stored) in cases:
    s = TraceSystem(build_cartesian(n, n), p, constant_problem(0.0, 1.0))
    if stored:
        E = n * n
        s = TraceSystem.from_blocks(build_cartesian(n, n), p, np.repeat(s.operator.S_cls, E, axis=0), np.arange(E))
    h = s.operator.handle
    NR = int(os.environ.get("TUNE_ROT", "4"))
    xs = [torch.rand(s.ndof, dtype=torch.float64, device="cuda") for _ in range(NR)]
    ys = [torch.empty_like(xs[0]) for _ in range(NR)]
    st = torch.cuda.current_stream().cuda_stream
    for k in range(20):
        L.check(L.lib.hdg_matvec(h, xs[k %% NR].data_ptr(), ys[k %% NR].data_ptr(), st))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 200
    e0.record()
    for k in range(R):
        L.check(L.lib.hdg_matvec(h, xs[k %% NR].data_ptr(), ys[k %% NR].data_ptr(), st))
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / R
    byts = 16 * s.ndof + (s.operator.operator_bytes() if stored else 0)
    out[f"n{n}p{p}{'S' if stored else ''}"] = {"us": round(us, 2), "GBs": round(byts / us / 1e3, 1), "GDOFs": round(s.ndof / us / 1e3, 1)}
    del s, xs, ys
    torch.cuda.empty_cache()
print(json.dumps(out))
''' % ROOT

for lib in sys.argv[1:]:
    env = dict(os.environ, HDGB200_LIB=os.path.abspath(lib))
    try:
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=240)
    except subprocess.TimeoutExpired:
        print(json.dumps({"lib": lib, "error": "timeout"}), flush=True)
        continue
    print(r.stdout.strip() or r.stderr[-2000:], flush=True)
