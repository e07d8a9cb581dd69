"""Check the tensor-core fp32 path against the oracle (and the SIMT path) on a
few shapes, each in its own time-limited process.  python tools/tc_check.py"""
import os
import subprocess
import sys

CASE = r'''
import os, sys, time, numpy as np
sys.path.insert(0, ".")
import paper_1702_02241_b200 as api
from oracle import spcp_oracle as orc
m, n, k, masked = {args}
rng = np.random.default_rng(m + n + k)
x = (rng.standard_normal((m, n)) * 3).astype(np.float32).astype(np.float64)
mask = rng.random((m, n)) < 0.6 if masked else None
u = (rng.standard_normal((m, k)) / np.sqrt(k)).astype(np.float32).astype(np.float64)
v = (rng.standard_normal((n, k)) / np.sqrt(k)).astype(np.float32).astype(np.float64)
spec = api.ProblemSpec(x=x, lambda_l=1.3, lambda_s=0.5, mask=mask)
t0 = time.time()
f, gu, gv = api.split_objective(api.FactorPair(u, v), spec, precision="fp32")
t1 = time.time()
fr, gur, gvr = orc.split_objective(u, v, x, 1.3, 0.5, mask)
_, gvr_raw, gtr_raw = orc.split_raw_products(u, v, x, 0.5, mask)
def rel(a, b): return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))
print("f %.2e  grad %.2e  GV %.2e  GtU %.2e  (%.2fs)" % (abs(f - fr) / abs(fr),
      rel(np.r_[gu.ravel(), gv.ravel()], np.r_[gur.ravel(), gvr.ravel()]),
      rel(gu - 1.3 * u, gvr_raw), rel(gv - 1.3 * v, gtr_raw), t1 - t0))
'''
configs = [(128, 64, 8, False), (300, 200, 20, False), (1000, 1000, 10, False),
           (777, 1333, 20, True), (2049, 300, 3, False), (300, 2049, 32, True),
           (1500, 900, 50, False), (640, 520, 64, True)]
env = dict(os.environ, SPCP_DEBUG_SYNC=os.environ.get("SPCP_DEBUG_SYNC", "1"))
for c in configs:
    try:
        r = subprocess.run([sys.executable, "-c", CASE.replace("{args}", repr(c))], env=env,
                           capture_output=True, text=True, timeout=90)
        tail = (r.stdout + r.stderr).strip().splitlines()
        print(c, "rc", r.returncode, tail[-1] if tail else "", flush=True)
    except subprocess.TimeoutExpired:
        print(c, "TIMEOUT", flush=True)
