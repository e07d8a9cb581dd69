"""Benchmark of the Split-SPCP hot path (BASELINE.json metric):
"SPCP obj+grad evals/s & HBM GB/s; time-to-certificate at 20k x 20k r=20".

A step is one objective+gradient evaluation (one fused streaming pass over X
plus operand prep and the fixed-order reduction) of the C2 workload
(BASELINE configs[1]): the reference generator's synthetic 20000 x 20000,
rank 20, 5% outliers, noise 1e-3 (`synth.gen_low_rank_plus_sparse`, byte-
identical to the reference's, seed 0, rounded to fp32 — the reference arm
evaluates exactly this X), lambda_L = 40, lambda_S = 0.1, k = 20, fp32
tensor-core kernel.  X (1.6 GB fp32) is larger than L2 (126 MB), so no L2
flush is needed between steps.  Warm-up runs at least W steps and at least
1 s of back-to-back evaluations, so the timed steps see the sustained
(power-capped) clock, not the first-millisecond burst (reported separately).

  python bench.py [--gpus N --steps K --warmup W]       this repo (one JSON line)
  python bench.py --impl reference ...                  reference CPU path

N > 1: one rank per GPU (torchrun, or self-launched when WORLD_SIZE is unset).
The headline stays C2 per GPU (weak scaling: each rank owns a 20000 x 20000
column shard of a 20000 x 20000N problem, grad_U all-reduced every
evaluation, value = whole-job evaluations of C2-sized shards per second); the
`c5` object is the north-star strong-scaling workload (configs[4]): the
200000 x 20000, rank 50 problem split over the N ranks, evals/s and
time-to-certificate (sharded solve + sharded certificate), at every N
including the single-GPU anchor.

The reference arm times the reference's own `split_objective` (the
unmodified `spcp` package `__graft_entry__.build()` pip-installs into
baseline/_ref) on the same full C2 matrix, one evaluation per step, on all
host cores; and the reference's C1 time-to-certificate.
"""

import argparse
import json
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M = N_COLS = 20000
RANK = 20
K = 20
LAM_L, LAM_S = 40.0, 0.1
METRIC = "SPCP obj+grad evals/s (C2 20000x20000 k=20 block-evals/s)"
C5 = dict(m=200000, n=20000, rank=50, k=50, lam_l=100.0)
SUSTAIN_S = 1.0  # minimum back-to-back warm-up before the timed region



def make_config(world):
    """The workload both arms report (identical dicts: same config)."""
    return {"workload": f"C2: reference synthetic {M}x{N_COLS} (gen_low_rank_plus_sparse seed 0, "
                        f"rounded to fp32) rank {RANK}, 5% outliers, noise 1e-3, k={K}, "
                        f"lambda_L={LAM_L}, lambda_S={LAM_S}; one objective+gradient "
                        f"evaluation of each {M}x{N_COLS} column shard per step",
            "m": M, "n_per_gpu": N_COLS, "n_total": N_COLS * world, "k": K,
            "parallelism": f"column-shard dp{world}",
            "l2": "no flush: X (1.6 GB fp32 per GPU) > 126 MB L2"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per launch of the fused kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_stream_kernel.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["dram_bytes_per_launch"])
    except Exception:
        return None


def cpu_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        import threadpoolctl

        info = threadpoolctl.threadpool_info()
        blas = [{"api": i.get("internal_api"), "version": i.get("version"),
                 "threads": i.get("num_threads")} for i in info]
    except Exception:
        pass
    return {"model": model, "nproc": os.cpu_count(), "blas": blas}


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML
    in-process every 5 ms, nvidia-smi as fallback."""

    def __init__(self):
        self.samples = []  # (time, sm_mhz, max_mhz, reasons)
        self._stop = threading.Event()
        self._t = None
        self.window = (None, None)

    def start(self):
        def run_nvml(pynvml, h):
            bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
                    "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((time.perf_counter(), float(sm), float(mx),
                                         [n for n, b in bits.items() if r & b]))
                except Exception:
                    pass
                self._stop.wait(0.005)

        def run_smi():
            q = ("--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", q, "--format=csv,noheader,nounits",
                                          "-i", os.environ.get("LOCAL_RANK", "0")],
                                         capture_output=True, text=True, timeout=5).stdout
                    parts = [x.strip() for x in out.strip().split(",")]
                    self.samples.append((time.perf_counter(), float(parts[0]), float(parts[1]),
                                         [n for n, v in zip(names, parts[2:6])
                                          if v.lower().startswith("active")]))
                except Exception:
                    pass
                self._stop.wait(0.05)

        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("LOCAL_RANK", "0")))
            target, args = run_nvml, (pynvml, h)
        except Exception:
            target, args = run_smi, ()
        self._t = threading.Thread(target=target, args=args, daemon=True)
        self._t.start()

    def mark(self, begin):
        t = time.perf_counter()
        self.window = (t, None) if begin else (self.window[0], t)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        t0, t1 = self.window
        inside = [x for x in self.samples
                  if (t0 is None or x[0] >= t0) and (t1 is None or x[0] <= t1)]
        if not inside and self.samples:  # region shorter than the sampling period
            inside = [min(self.samples, key=lambda x: abs(x[0] - (t0 or 0.0)))]
        sm = [x[1] for x in inside]
        mx = inside[-1][2] if inside else None
        reasons = sorted({r for x in inside for r in x[3]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "sm_mhz_min": float(np.min(sm)) if sm else None,
                "reasons": reasons, "samples": len(sm)}


def alg_bytes(m, n, k, masked=False):
    """B_alg per evaluation: X once, mask bits, U/V in, grads out."""
    return 4 * m * n + (((m * n + 7) // 8) if masked else 0) + 2 * 4 * (m + n) * k


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_pkg():
    """The unmodified reference package (`spcp`, pure Python) installed into
    baseline/_ref by `__graft_entry__.build()` (pip --target), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "spcp")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import spcp
    except Exception:
        return None
    if not os.path.abspath(spcp.__file__).startswith(REF_DIR):
        return None
    return spcp


def c2_host_x():
    """The C2 matrix from the reference's own generator law (byte-identical
    restatement, tested against the reference in tests/test_oracle_golden.py),
    rounded to fp32 exactly as the device receives it."""
    from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse

    x, _, _ = gen_low_rank_plus_sparse(M, N_COLS, RANK, 0.05, 1e-3, seed=0)
    return x.astype(np.float32)


def c2_iterate(n_cols=N_COLS, col0=0):
    """A representative iterate: U, V ~ N(0, 2) (the scale of the rank-20
    factors), from one host stream shared by every rank (U is replicated)."""
    rng = np.random.default_rng(1)
    u = rng.standard_normal((M, K)) * np.sqrt(2.0)
    v_all = rng.standard_normal((N_COLS, K)) * np.sqrt(2.0)
    return u, v_all[col0 % N_COLS:col0 % N_COLS + n_cols]


def reference_c1_ttc(ref):
    """The reference's time-to-certificate at C1: solve_split_spcp + certificate
    (solver.py:255, certificate.py:77) on configs[0], host cores."""
    x, _, _ = ref.gen_low_rank_plus_sparse(1000, 1000, 10, 0.05, 1e-3, seed=0)
    x = x.astype(np.float32).astype(np.float64)
    spec = ref.ProblemSpec(x=x, lambda_l=10.0, lambda_s=0.1)
    t0 = time.perf_counter()
    rep = ref.solve_split_spcp(spec, 10, ref.SolverConfig())
    t1 = time.perf_counter()
    cert = ref.certificate(rep.factors, spec, f_bound_hint=rep.best_objective)
    t2 = time.perf_counter()
    return {"seconds": t2 - t0, "solve_s": t1 - t0, "certificate_s": t2 - t1,
            "termination": rep.termination, "iterations": len(rep.iterations) - 1,
            "objective": rep.objective, "e_norm": cert.e_norm, "r": cert.r}


def reference_c3_ttc(ref, ks=(3,)):
    """The reference's time-to-certificate at C3 (110592 x 2000, lambda_L 30):
    minutes of CPU, so only with --ref-c3."""
    x, _, _ = ref.gen_low_rank_plus_sparse(110592, 2000, 3, 0.05, 1e-3, seed=0)
    x = x.astype(np.float32).astype(np.float64)
    spec = ref.ProblemSpec(x=x, lambda_l=30.0, lambda_s=0.1)
    out = {}
    for k in ks:
        t0 = time.perf_counter()
        rep = ref.solve_split_spcp(spec, k, ref.SolverConfig())
        t1 = time.perf_counter()
        cert = ref.certificate(rep.factors, spec, f_bound_hint=rep.best_objective)
        t2 = time.perf_counter()
        out[f"k{k}"] = {"seconds": t2 - t0, "solve_s": t1 - t0, "certificate_s": t2 - t1,
                        "termination": rep.termination, "iterations": len(rep.iterations) - 1,
                        "objective": rep.objective, "e_norm": cert.e_norm, "r": cert.r}
    return out


def run_reference(args, rank, world):
    """--impl reference: the unmodified reference on the box's host cores,
    rank 0 only.  One full C2 split_objective per step (the same X and
    config as this repo's arm)."""
    if rank != 0:
        return
    ref = reference_pkg()
    kind = "reference"
    if ref is None:  # the oracle port stands in (kind "port")
        from oracle import spcp_oracle as orc
        kind = "port"
    x = c2_host_x().astype(np.float64)
    u, v = c2_iterate()
    if ref is not None:
        spec = ref.ProblemSpec(x=x, lambda_l=LAM_L, lambda_s=LAM_S)
        fp = ref.FactorPair(u, v)

        def call():
            ref.split_objective(fp, spec)
    else:
        def call():
            orc.split_objective(u, v, x, LAM_L, LAM_S)
    for _ in range(args.warmup):
        call()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    per = float(np.mean(times))
    val = 1.0 / per
    ttc = reference_c1_ttc(ref) if ref is not None else None
    ttc3 = reference_c3_ttc(ref) if (ref is not None and args.ref_c3) else None
    info = cpu_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": make_config(world),
        "cpu_baseline": {"value": val, "unit": "evals/s", "cores": info["nproc"], "kind": kind,
                         "sample": f"{'reference spcp' if ref else 'oracle port'}."
                                   f"split_objective on the full C2 matrix ({M}x{N_COLS}, "
                                   f"float64 numpy/OpenBLAS, all host threads), one evaluation "
                                   f"per step, {args.steps} timed steps",
                         "cpu": info, "ttc_c1": ttc, "ttc_c3": ttc3},
        "e2e": {"value": val, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- this repo's arm
def _dist_setup(world, backend):
    import torch

    if world == 1:
        torch.cuda.set_device(0)
        return None
    import torch.distributed as dist

    from paper_1702_02241_b200.dist import pin_nccl

    local = int(os.environ.get("LOCAL_RANK", os.environ.get("RANK", 0)))
    torch.cuda.set_device(local % torch.cuda.device_count())
    pin_nccl()
    dist.init_process_group(backend)
    return dist


def _time_evals(dp, step, steps, warmup, dist, stream):
    """W warm-up steps (and at least SUSTAIN_S seconds of them), then exactly
    `steps` timed steps between barriers; returns (ms per step, fused-kernel
    ms, launches, burst dict, clocks)."""
    import torch

    clocks = ClockSampler()
    clocks.start()  # NVML up before the timed region; samples kept only inside it
    # burst: 20 steps on a cold clock (after 3 that absorb first-call setup)
    for i in range(3):
        step(i)
    torch.cuda.synchronize()
    dp.prof_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nb = 20
    e0.record(stream)
    for i in range(nb):
        step(i)
    e1.record(stream)
    torch.cuda.synchronize()
    k_ms, k_cnt, _ = dp.prof_read()
    burst = {"steps": nb, "ms_per_step": e0.elapsed_time(e1) / nb,
             "kernel_ms": k_ms / max(k_cnt, 1)}
    dp.prof_enable(False)
    # then at least SUSTAIN_S seconds back to back (the same count on every
    # rank: the sharded step holds a collective)
    extra = max(warmup - nb - 3, int(np.ceil(SUSTAIN_S * 1e3 / max(burst["ms_per_step"], 1e-3))))
    if dist:
        t = torch.tensor([float(extra)], device=torch.device("cuda"), dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        extra = int(t[0])
    for i in range(extra):
        step(nb + i)
    done = 3 + nb + extra
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    dp.prof_read()  # reset the launch counter: gpu_launches counts the timed steps only
    dp.prof_enable(True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    clocks.mark(True)
    ev0.record(stream)
    for i in range(steps):
        step(i)
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks.mark(False)
    clk = clocks.stop()
    ms_total = ev0.elapsed_time(ev1)
    k1_ms, k1_count, launches = dp.prof_read()
    dp.prof_enable(False)
    t_step = ms_total / steps
    k1_avg = k1_ms / max(k1_count, 1)
    if dist:
        t = torch.tensor([t_step, k1_avg], device=torch.device("cuda"), dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_step, k1_avg = float(t[0]), float(t[1])
    return t_step, k1_avg, launches, burst, clk, done


def run_b200(args, rank, world):
    import torch

    from paper_1702_02241_b200._lib import SPCP_F32
    from paper_1702_02241_b200.device import DeviceProblem

    dist = _dist_setup(world, args.backend)
    dev = torch.device("cuda", torch.cuda.current_device())
    n_total = N_COLS * world
    col0 = N_COLS * rank
    xh = c2_host_x() if (rank == 0 or world == 1) else None
    if world > 1:  # every rank's shard is a copy of the C2 block (weak scaling)
        xt = torch.empty((M, N_COLS), dtype=torch.float32, device=dev)
        if rank == 0:
            xt.copy_(torch.from_numpy(xh))
        dist.broadcast(xt, 0)
        xsrc = xt
    else:
        xsrc = xh
    dp = DeviceProblem(xsrc, LAM_L, LAM_S, store=("f32",), n_total=n_total, col0=col0)
    if world > 1:
        del xt, xsrc
    torch.cuda.empty_cache()
    u, v = c2_iterate(N_COLS, col0)
    z = torch.from_numpy(np.r_[u.ravel(), v.ravel()]).to(dev)
    dz = torch.from_numpy(np.random.default_rng(2).standard_normal(z.numel()) * 1e-3).to(dev)
    g = torch.empty_like(z)
    if world > 1:
        from paper_1702_02241_b200.dist import ShardedSpace

        space = ShardedSpace(dp, K, M, N_COLS)

        def step(i):
            space.eval(z, dz, 1e-3 * (i % 50 + 1), g, "fp32")
    else:
        out_dev = torch.empty(8, device=dev, dtype=torch.float64)

        def step(i):
            # stream-ordered: the scalars stay on the device (the solver's
            # synchronous call, with its host round trip, is what e2e times)
            dp.eval_async(K, SPCP_F32, z, dz, 1e-3 * (i % 50 + 1), g, out_dev)

    t_step, k1_avg, launches, burst, clk, warm_done = _time_evals(
        dp, step, args.steps, args.warmup, dist, dp.stream)
    value = world * 1e3 / t_step  # whole-job C2-block evaluations per second

    # ---- e2e: the reference-facing host API (split_objective with host buffers)
    e2e = None
    if world == 1 and not args.skip_e2e:
        uh = torch.empty((M, K), dtype=torch.float64).pin_memory().numpy()
        vh = torch.empty((N_COLS, K), dtype=torch.float64).pin_memory().numpy()
        uh[:] = u
        vh[:] = v
        gu_h = torch.empty((M, K), dtype=torch.float64).pin_memory().numpy()
        gv_h = torch.empty((N_COLS, K), dtype=torch.float64).pin_memory().numpy()
        for _ in range(3):
            dp.split_objective_host(uh, vh, SPCP_F32, out=(gu_h, gv_h))
        torch.cuda.synchronize()
        n_e2e = max(3, args.steps // 2)
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            dp.split_objective_host(uh, vh, SPCP_F32, out=(gu_h, gv_h))
        te = (time.perf_counter() - t0) / n_e2e
        nz = (M + N_COLS) * K
        e2e = {"value": 1.0 / te, "unit": "evals/s", "h2d_bytes_per_step": 8 * nz,
               "d2h_bytes_per_step": 8 * nz + 8, "steps": n_e2e,
               "path": "spcp_split_objective_host (C ABI, pinned host float64 U,V in, "
                       "grads out to pinned host buffers, one sync per call)"}
    dp.close()
    del dp, z, dz, g
    torch.cuda.empty_cache()

    ttc = None
    if world == 1 and not args.skip_ttc:
        ttc = _guard(lambda: time_to_certificate(dev, xh))
    c5 = None
    if not args.skip_c5:
        c5 = _guard(lambda: c5_bench(dev, rank, world, dist, ttc=not args.skip_ttc))
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        cpu = _guard(lambda: cpu_baseline(xh))

    line = None
    if rank == 0:
        b_alg = alg_bytes(M, N_COLS, K)
        achieved = b_alg / (k1_avg * 1e-3) / 1e9
        peak, peak_src = peaks()
        cfg = make_config(world)
        step_desc = ("one objective+gradient evaluation at z + alpha dz: max, operand images, "
                     "fused pass, fixed-order reduction (stream-ordered, scalars left on the "
                     "device)" + ("; grad_U + scalars all-reduced (one NCCL group)"
                                  if world > 1 else ""))
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": warm_done, "ms_per_step": t_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": cfg, "step": step_desc,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(),
                         "kernel": "tc_eval_kernel<16,false,20> (tcgen05 fused pass, "
                                   "K-concatenated operand images)",
                         "kernel_ms": k1_avg, "alg_bytes": b_alg, "peak_source": peak_src,
                         "sustained": f"timed after >= {SUSTAIN_S} s of back-to-back "
                                      f"evaluations ({warm_done} warm-up steps)",
                         "burst": dict(burst, frac=b_alg / (burst["kernel_ms"] * 1e-3) / 1e9
                                       / peak)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "time_to_certificate": ttc,
            "c5": c5,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return line


def _guard(fn):
    """A sub-measurement failure must not void the bench line."""
    try:
        return fn()
    except Exception as exc:  # noqa: BLE001
        return {"error": f"{type(exc).__name__}: {exc}"[:500]}


def cpu_baseline(xh):
    """The reference on the box's host cores (rank 0, N=1): one full C2
    split_objective on the same X and iterate, and the C1 time-to-certificate
    (~10-20 s of CPU in total)."""
    ref = reference_pkg()
    u, v = c2_iterate()
    x = xh.astype(np.float64)
    info = cpu_info()
    if ref is not None:
        spec = ref.ProblemSpec(x=x, lambda_l=LAM_L, lambda_s=LAM_S)
        fp = ref.FactorPair(u, v)
        t0 = time.perf_counter()
        ref.split_objective(fp, spec)
        t = time.perf_counter() - t0
        kind, what = "reference", "reference spcp.split_objective (baseline/_ref)"
        ttc = reference_c1_ttc(ref)
    else:
        from oracle import spcp_oracle as orc

        t0 = time.perf_counter()
        orc.split_objective(u, v, x, LAM_L, LAM_S)
        t = time.perf_counter() - t0
        kind, what, ttc = "port", "oracle split_objective (numpy port)", None
    return {"value": 1.0 / t, "unit": "evals/s", "cores": info["nproc"], "kind": kind,
            "sample": f"{what}, float64 numpy/OpenBLAS on all host threads, one evaluation "
                      f"of the full C2 matrix at the bench iterate",
            "cpu": info, "ttc_c1": ttc}


def time_to_certificate(dev, xh):
    """C2 end to end with X resident: rSVD init, L-BFGS (fp32 bulk, fp64
    finish), certificate; wall clock (synchronous API).  Also C1 (k=10) and
    C3 (k=3, 5) on the reference generator's matrices."""
    import torch

    from paper_1702_02241_b200 import ProblemSpec, SolverConfig, certificate, solve_split_spcp
    from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse, \
        gen_low_rank_plus_sparse_device

    # one-time library/workspace initialisation on a separate small problem
    # that still takes the mixed-precision solve and certificate paths; the
    # C2 problem itself is not touched before the clock starts
    xw = gen_low_rank_plus_sparse_device(4200, 4200, 5, 0.05, 1e-3, seed=1)
    sw = ProblemSpec(x=xw, lambda_l=4.0, lambda_s=LAM_S)
    rw = solve_split_spcp(sw, 5, SolverConfig(max_iter=20))
    certificate(rw.factors, sw, f_bound_hint=rw.best_objective)
    sw.release_device()
    del xw, sw, rw
    x = torch.from_numpy(xh).to(dev)
    spec = ProblemSpec(x=x, lambda_l=LAM_L, lambda_s=LAM_S)
    spec.device("mixed")
    runs = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = solve_split_spcp(spec, K, SolverConfig())
        t1 = time.perf_counter()
        cert = certificate(rep.factors, spec, f_bound_hint=rep.best_objective)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        runs.append((t2 - t0, t1 - t0, t2 - t1, rep, cert))
    best = min(runs, key=lambda r: r[0])
    _, _, _, rep, cert = best
    out = {"seconds": best[0], "solve_s": best[1], "certificate_s": best[2],
           "runs_s": [round(r[0], 4) for r in runs],
           "termination": rep.termination, "iterations": len(rep.iterations) - 1,
           "n_evals": rep.extra["n_evals"], "objective": rep.objective,
           "e_norm": cert.e_norm, "gap_bound": cert.gap_bound, "r": cert.r,
           "verdict": "certified" if cert.gap_bound <= 1e-2 * max(1.0, abs(rep.objective))
           else "flagged", "t4": cert.info, "fp64_switch_iter": rep.extra.get("fp64_switch_iter")}
    gold = os.path.join(ROOT, "tests", "golden", "c2.npz")
    if os.path.exists(gold):
        d = np.load(gold)
        out["reference"] = {"objective": float(d["k20_obj"]), "termination": str(d["k20_term"]),
                            "iterations": int(len(d["k20_recobj"]) - 1),
                            "n_evals": int(d["k20_evals"]), "e_norm": float(d["k20_cert"][0]),
                            "solve_s_8cores": float(d["k20_solve_s"]),
                            "certificate_s_8cores": float(d["k20_cert_s"])}
        out["objective_rel_vs_reference"] = abs(rep.objective - float(d["k20_obj"])) / abs(
            float(d["k20_obj"]))
    out["first_certified"] = first_certified(spec)
    spec.release_device()
    out["from_file"] = ttc_from_file(xh)
    del x
    torch.cuda.empty_cache()
    out["c1"] = _guard(lambda: small_ttc(dev, "c1", 1000, 1000, 10, 10.0, (10,)))
    out["c3"] = _guard(lambda: small_ttc(dev, "c3", 110592, 2000, 3, 30.0, (3, 5)))
    return out


def small_ttc(dev, tag, m, n, rank, lam_l, ks):
    """Time to certificate on a reference-generator matrix (X resident)."""
    import torch

    from paper_1702_02241_b200 import ProblemSpec, SolverConfig, certificate, solve_split_spcp
    from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse

    xh, _, _ = gen_low_rank_plus_sparse(m, n, rank, 0.05, 1e-3, seed=0)
    x = torch.from_numpy(xh.astype(np.float32)).to(dev)
    spec = ProblemSpec(x=x, lambda_l=lam_l, lambda_s=LAM_S)
    spec.device("mixed")
    res = {}
    gold = os.path.join(ROOT, "tests", "golden", f"{tag}.npz")
    d = np.load(gold) if os.path.exists(gold) else None
    for k in ks:
        best = None
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = solve_split_spcp(spec, k, SolverConfig())
            t1 = time.perf_counter()
            cert = certificate(rep.factors, spec, f_bound_hint=rep.best_objective)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            if best is None or t2 - t0 < best["seconds"]:
                best = {"seconds": t2 - t0, "solve_s": t1 - t0, "certificate_s": t2 - t1,
                        "termination": rep.termination,
                        "iterations": len(rep.iterations) - 1,
                        "n_evals": rep.extra["n_evals"], "objective": rep.objective,
                        "e_norm": cert.e_norm, "r": cert.r,
                        "verdict": "certified" if cert.gap_bound <= 1e-2 * max(
                            1.0, abs(rep.objective)) else "flagged"}
        if d is not None and f"k{k}_obj" in d:
            best["reference"] = {"objective": float(d[f"k{k}_obj"]),
                                 "termination": str(d[f"k{k}_term"]),
                                 "e_norm": float(d[f"k{k}_cert"][0])}
            if f"k{k}_solve_s" in d:
                best["reference"]["seconds_8cores"] = float(d[f"k{k}_solve_s"]) + float(
                    d[f"k{k}_cert_s"])
        res[f"k{k}"] = best
    spec.release_device()
    return res


def c5_bench(dev, rank, world, dist, ttc=True, steps=20):
    """configs[4]: 200000 x 20000, rank 50, k=50, column-sharded over the
    `world` ranks (strong scaling; world = 1 is the single-GPU anchor).  The
    shard is generated on each GPU (column-block counter streams: the same
    matrix at every N).  Evals/s of the whole problem (max over ranks) and
    time-to-certificate (sharded solve + sharded certificate)."""
    import torch

    from paper_1702_02241_b200._lib import SPCP_F32
    from paper_1702_02241_b200.device import DeviceProblem
    from paper_1702_02241_b200.dist import shard_bounds
    from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse_device

    m, n, rk, k, lam = C5["m"], C5["n"], C5["rank"], C5["k"], C5["lam_l"]
    c0, nl = shard_bounds(n, world, rank)
    x = gen_low_rank_plus_sparse_device(m, nl, rk, 0.05, 1e-3, seed=0, col0=c0, n_total=n)
    dp = DeviceProblem(x, lam, LAM_S, store=("f32",), n_total=n, col0=c0)
    rng = np.random.default_rng(5)
    u = rng.standard_normal((m, k))
    v = rng.standard_normal((n, k))[c0:c0 + nl]
    z = torch.from_numpy(np.r_[u.ravel(), v.ravel()]).to(dev)
    g = torch.empty_like(z)
    if world > 1:
        from paper_1702_02241_b200.dist import ShardedSpace

        space = ShardedSpace(dp, k, m, nl)

        def step(i):
            space.eval(z, None, 0.0, g, "fp32")
    else:
        out_dev = torch.empty(8, device=dev, dtype=torch.float64)

        def step(i):
            dp.eval_async(k, SPCP_F32, z, None, 0.0, g, out_dev)

    t_step, k1_avg, _, _, _, _ = _time_evals(dp, step, steps, 3, dist, dp.stream)
    out = {"workload": f"{m}x{n} rank {rk}, k={k}, lambda_L={lam}, column-sharded over "
                       f"{world} GPU(s) ({nl} columns per rank)", "n_gpus": world,
           "evals_per_s": 1e3 / t_step, "ms_per_eval": t_step, "kernel_ms": k1_avg,
           "roofline_frac_per_gpu": alg_bytes(m, nl, k) / (k1_avg * 1e-3) / 1e9 / peaks()[0],
           "scaling": "strong"}
    del g, z
    if ttc:
        out["time_to_certificate"] = _guard(lambda: c5_ttc(x, dp, rank, world, dist))
    dp.close()
    del x, dp
    torch.cuda.empty_cache()
    return out


def c5_ttc(x, dp_eval, rank, world, dist):
    import torch

    from paper_1702_02241_b200.dist import certificate_sharded, shard_bounds, \
        solve_split_spcp_sharded
    from paper_1702_02241_b200.solver import SolverConfig

    m, n, k, lam = C5["m"], C5["n"], C5["k"], C5["lam_l"]
    c0, nl = shard_bounds(n, world, rank)
    dp_eval.close()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    if world > 1:
        rep = solve_split_spcp_sharded(x, lam, LAM_S, k, n, c0, SolverConfig())
        t1 = time.perf_counter()
        cert = certificate_sharded(rep)
    else:
        from paper_1702_02241_b200 import ProblemSpec, certificate, solve_split_spcp

        spec = ProblemSpec(x=x, lambda_l=lam, lambda_s=LAM_S)
        rep = solve_split_spcp(spec, k, SolverConfig())
        t1 = time.perf_counter()
        cert = certificate(rep.factors, spec, f_bound_hint=rep.best_objective)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    tt = torch.tensor([t2 - t0, t1 - t0], dtype=torch.float64, device=x.device)
    if dist:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    res = {"seconds": float(tt[0]), "solve_s": float(tt[1]),
           "certificate_s": float(tt[0] - tt[1]), "termination": rep.termination,
           "iterations": len(rep.iterations) - 1, "n_evals": rep.extra["n_evals"],
           "objective": rep.objective, "e_norm": cert.e_norm, "r": cert.r,
           "verdict": "certified" if cert.gap_bound <= 1e-2 * max(1.0, abs(rep.objective))
           else "flagged", "t4": cert.info}
    if world > 1:
        res["allreduce_calls"] = rep.extra.get("allreduce_calls")
        res["allreduce_bytes"] = rep.extra.get("allreduce_bytes")
    else:
        spec.release_device()  # the problem's workspaces (outside the timed region)
    return res


def ttc_from_file(xh):
    """SURVEY §8(d) 'also reported including H2D': the same C2 solve and
    certificate, with the clock started before X is read from an SLRM file
    (float64, 3.2 GB, page cache warm) and streamed into HBM as float32
    (exact: X is fp32-rounded) by the native reader."""
    import shutil
    import tempfile

    import torch

    from paper_1702_02241_b200 import ProblemSpec, SolverConfig, certificate, solve_split_spcp
    from paper_1702_02241_b200.matrixio import read_matrix, write_matrix

    tmp = tempfile.mkdtemp(prefix="spcp_ttc_")
    try:
        path = os.path.join(tmp, "x.bin")
        write_matrix(xh.astype(np.float64), path)  # untimed: the file exists before the run
        torch.cuda.empty_cache()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        xd = read_matrix(path, device="cuda", dtype=torch.float32)
        spec = ProblemSpec(x=xd, lambda_l=LAM_L, lambda_s=LAM_S)
        spec.device("mixed")
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        rep = solve_split_spcp(spec, K, SolverConfig())
        cert = certificate(rep.factors, spec, f_bound_hint=rep.best_objective)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        res = {"seconds": t2 - t0, "ingest_s": t1 - t0, "file_bytes": os.path.getsize(path),
               "objective": rep.objective, "e_norm": cert.e_norm,
               "path": "read_matrix(device=cuda) -> ProblemSpec -> solve -> certificate"}
        spec.release_device()
        return res
    except Exception as exc:  # disk trouble must not void the bench line
        return {"error": f"{type(exc).__name__}: {exc}"}
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


class _Certified(Exception):
    pass


def first_certified(spec, every=5):
    """SURVEY §8(d) time-to-certificate (ii): the CLI's `--certificate every:N`
    mode (cli.py:229-236) — certify every N iterations, stop the clock at the
    first iterate with no under-rank warning (gap <= 1e-2 max(1, |f|),
    cli.py:27,246-251) and no sigma(P) > 1.  Wall clock from solve entry,
    including the certificates computed along the way."""
    import torch

    from paper_1702_02241_b200 import SolverConfig, certificate, solve_split_spcp, split_objective

    found = {}
    t0 = time.perf_counter()

    def hook(it, st):
        if it == 0 or it % every:
            return None
        f, _, _ = split_objective(st.factors, spec)
        cert = certificate(st.factors, spec, f_bound_hint=f)
        ok = cert.gap_bound <= 1e-2 * max(1.0, abs(f)) and cert.info.get("n_sigma_over_1", 0) == 0
        if ok:
            torch.cuda.synchronize()
            found.update(seconds=time.perf_counter() - t0, iteration=it, objective=f,
                         e_norm=cert.e_norm, gap_bound=cert.gap_bound, every=every)
            raise _Certified()
        return None

    try:
        solve_split_spcp(spec, K, SolverConfig(), iter_hook=hook)
    except _Certified:
        pass
    return found or None


def _spawned(local_rank, world, port, argv):
    os.environ.update({"RANK": str(local_rank), "LOCAL_RANK": str(local_rank),
                       "WORLD_SIZE": str(world), "MASTER_ADDR": "127.0.0.1",
                       "MASTER_PORT": str(port)})
    sys.argv = [sys.argv[0]] + argv
    main()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--backend", default="nccl", help="torch.distributed backend for N > 1")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-ttc", action="store_true")
    ap.add_argument("--skip-c5", action="store_true")
    ap.add_argument("--ref-c3", action="store_true",
                    help="reference arm: also time the reference's C3 solve + certificate")
    args, _ = ap.parse_known_args()
    if args.impl == "b200":
        args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # self-launch one process per GPU (what torchrun would do)
        import socket

        import torch.multiprocessing as mp

        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        mp.start_processes(_spawned, args=(args.gpus, port, sys.argv[1:]), nprocs=args.gpus,
                           start_method="spawn")
        return
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_b200(args, rank, world)


if __name__ == "__main__":
    main()
