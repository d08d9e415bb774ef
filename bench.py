"""MF-WQ B200 benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], "cfg2"): unit-cube Poisson, identity
geometry, n_el = 128 per direction, maximal-regularity splines p = 2..6,
fp64.  One step = one MF-WQ stiffness matvec at every degree of the sweep on
x ~ N(0,1) (seed 0).  value = DoFs processed / second over the whole sweep.
The coefficient grids (0.4-0.9 GB per degree) exceed the 126 MB L2, so no
explicit flush is needed between iterations.

Extra keys: per-degree times, roofline of the matvec kernel (HBM bound per
BASELINE; fp64 fraction alongside), e2e through the public API with pinned
host buffers (and through the drop-in numpy call), the CPU baseline (oracle
port on the host cores), the cfg-3 matvec / FD-PCG, the cfg-4 per-phase
k-sweep and cfg 1 (--pcg), and the cfg-5 FD-PCG on one GPU (--slab).

With N > 1 (torchrun, or --gpus N, which spawns the ranks itself) the headline
is the cfg-5 FD-PCG split into N xi3 slabs, one rank per GPU (strong scaling,
native comm-aware solver over NCCL); the N = 1 line carries the same solve on
one GPU under "slab_pcg" as its baseline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--pcg 0|1] [--slab 0|1]
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SWEEP = (2, 3, 4, 5, 6)
N_EL = 128
METRIC = "MF-WQ fp64 matvec DoF/s (cfg2 sweep p=2-6, n_el=128)"
UNIT = "DoF/s"
# the workload both arms run (identical dict in both JSON lines); arm-specific detail goes to "execution"
CONFIG = {"workload": "cfg2 unit-cube MF-WQ matvec sweep: one matvec per degree p=2..6 per step, n_el=128",
          "sweep": list(SWEEP), "n_el": N_EL, "geometry": "identity", "x": "N(0,1) seed 0"}
ANCHORS = os.path.join(ROOT, "tests", "golden", "full_vectors.json")  # reference-run anchors (make_anchors.py)


def anchors():
    try:
        with open(ANCHORS) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pcg", type=int, default=1)
    ap.add_argument("--cpu-baseline", type=int, default=1)
    ap.add_argument("--path", default="auto", choices=["auto", "generic", "fused"])
    ap.add_argument("--slab", type=int, default=1, help="cfg5 slab PCG (1-GPU baseline / N-GPU headline)")
    return ap.parse_args()


def dist_info():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ----------------------------------------------------------------------------- clocks
# NVML clocks-event-reason bits (nvml.h nvmlClocksEventReason*)
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    """Polls NVML (SM clock, clocks-event reasons) every ~2 ms while the timed region runs."""

    def __init__(self, index, period=0.002):
        self.index, self.period = index, period
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((sm, rs))
                    except pynvml.NVMLError:
                        pass
                    time.sleep(self.period)

            self.t = threading.Thread(target=run, daemon=True)
            self.t.start()
        except Exception:  # NVML unavailable: report no samples
            self.t = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.t is not None:
            self.t.join(timeout=1)

    def summary(self):
        sm = [s for s, _ in self.samples]
        reasons = set()
        for _, rs in self.samples:
            for bit, name in REASONS.items():
                if rs & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm), "source": "NVML polled every 2 ms in the timed region"}


# ----------------------------------------------------------------------------- peaks
def peaks():
    out = {"hbm_gbs": 6650.0, "hbm_src": "fallback (B200_PROFILING.md)", "fp64_tflops": 37.1,
           "fp64_src": "DMMA probe tools/fp64_peak (profiles/fp64_peak_r01.json)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            m = json.load(fh)
        out["hbm_gbs"] = float(m["hbm_gbs"])
        out["hbm_src"] = "measured (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        pass
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")) as fh:
            f = json.load(fh)
        out["fp64_tflops"] = max(float(f["dmma_tflops"]), float(f["dfma_tflops"]))
    except (OSError, KeyError, ValueError):
        pass
    return out


def traffic_from_profile():
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return None


# ----------------------------------------------------------------------------- CPU baseline
def cpu_sample(steps=None, threads=None):
    """Oracle port (oracle/mfwq_oracle.py) on the host: one matvec per degree.

    Coefficient grids for identity geometry are the exact constants the
    reference computes there (C = I; operators.py:64-84 gives det = 1 and
    J^-1 = I exactly), built directly so the sample times the matvec only.
    """
    from oracle import mfwq_oracle as O

    degs = SWEEP if steps is None else [SWEEP[i % len(SWEEP)] for i in range(steps)]
    built = {}
    total_n, total_t = 0, 0.0
    per = {}
    for p in degs:
        if p not in built:
            kv = O.uniform_knots(p, N_EL)
            rule = O.rule_1d(kv)
            nq = len(rule.pts) ** 3
            C = {k: (np.ones(nq) if k[0] == k[1] else np.zeros(nq)) for k in O.COEFF_KEYS}
            built[p] = O.Stiffness([rule] * 3, C)
        A = built[p]
        x = np.random.default_rng(0).standard_normal(A.N)
        t0 = time.perf_counter()
        A.apply(x)
        dt = time.perf_counter() - t0
        total_n += A.N
        total_t += dt
        per.setdefault(p, []).append(dt)
    return total_n / total_t, per, total_t


# ----------------------------------------------------------------------------- reference arm
def _ref_worker(widx, p, warmup, steps, start_evt, q):
    """One host core: the oracle matvec (scipy CSR sum-factorisation, single-threaded like the
    reference's csr_matvecs path) at degree p, `warmup` untimed then `steps` timed applies."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import mfwq_oracle as O

    kv = O.uniform_knots(p, N_EL)
    rule = O.rule_1d(kv)
    nq = len(rule.pts) ** 3
    C = {k: (np.ones(nq) if k[0] == k[1] else np.zeros(nq)) for k in O.COEFF_KEYS}
    A = O.Stiffness([rule] * 3, C)
    x = np.random.default_rng(0).standard_normal(A.N)
    for _ in range(warmup):
        A.apply(x)
    q.put(("ready", widx))
    start_evt.wait()
    t0 = time.perf_counter()
    for _ in range(steps):
        A.apply(x)
    q.put(("done", widx, p, A.N * steps, time.perf_counter() - t0))


def _ref_workers():
    """Independent single-threaded matvec processes: one per host core, bounded by ~2 GB each."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    try:
        with open("/proc/meminfo") as fh:
            avail_kb = next(int(l.split()[1]) for l in fh if l.startswith("MemAvailable:"))
        by_mem = max(1, int(avail_kb / 1e6 * 0.6 / 2.0))
    except (OSError, StopIteration, ValueError):
        by_mem = cores
    cap = int(os.environ.get("MFWQ_REF_WORKERS", "0")) or cores
    return max(1, min(cores, by_mem, cap)), cores


def run_reference_slab(args, rank, world):
    """Reference arm of the N > 1 headline (cfg5 slab PCG): the oracle port's PCG iteration (one MF-WQ
    matvec, one FD apply, the vector updates; solvers.py:154-172) on a bounded sample of the cfg5
    problem -- the quarter ring at p = 6 with the full 512 x 512 element cross-section and a z-extent
    of SLAB_SAMPLE_EL elements -- timed on rank 0's host cores; value = sample DoFs x iterations / s."""
    if rank != 0:
        return
    from oracle import mfwq_oracle as O
    p, n_el = CFG5
    ez = int(os.environ.get("MFWQ_SLAB_SAMPLE_EL", "4"))
    nxy = int(os.environ.get("MFWQ_SLAB_SAMPLE_NXY", str(n_el)))  # tests shrink the cross-section
    kxy, kz = O.uniform_knots(p, nxy), O.uniform_knots(p, ez)
    rules = [O.rule_1d(kxy), O.rule_1d(kxy), O.rule_1d(kz)]
    A = O.Stiffness(rules, O.stiffness_coeffs(rules, O.jac_ring))
    P = O.FD([kxy, kxy, kz])
    r = np.random.default_rng(1).standard_normal(A.N)
    pv = r.copy()
    x = np.zeros(A.N)

    def it():
        Ap = A.apply(pv)
        alpha = float(r @ r) / float(pv @ Ap)
        x.__iadd__(alpha * pv)
        rn = r - alpha * Ap
        z = P.apply(rn)
        return float(rn @ z)

    for _ in range(max(1, min(args.warmup, 1))):
        it()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        it()
    dt = (time.perf_counter() - t0) / args.steps
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    val = A.N / dt
    line = {"metric": SLAB_METRIC, "value": val, "unit": "DoF-iterations/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"cfg5 quarter ring p={p} n_el={n_el}, xi3 slabs x{world}",
                       "parallelism": f"xi3 slabs x{world} (NCCL)"},
            "cpu_baseline": {"value": val, "unit": "DoF-iterations/s", "cores": cores, "kind": "port",
                             "sample": f"one oracle PCG iteration (MF-WQ matvec + FD apply + updates) per step on a "
                                       f"{nxy} x {nxy} x {ez}-element z-slab of the cfg5 quarter ring (p={p}), "
                                       f"{A.N} DoFs; scipy CSR single-threaded, FD dgemm on the host BLAS threads"},
            "e2e": {"value": val, "unit": "DoF-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_reference(args, rank, world):
    """The reference's CPU path on every host core the box gives us.

    The reference matvec (operators.py:185-204 via scipy csr_matvecs) is single-threaded, so the
    host's throughput comes from independent applies in parallel processes: worker w runs degree
    SWEEP[w % 5] (so the sweep is covered evenly), each step = one apply per worker, all workers
    released together after their warm-up; value = all DoFs / wall time of the timed region.
    The reference itself cannot travel to the GPU box, so its oracle port stands in (pinned to the
    reference's outputs by tests/test_oracle_golden.py)."""
    if rank != 0:
        return
    import multiprocessing as mp

    nw, cores = _ref_workers()
    ctx = mp.get_context("fork")
    start, q = ctx.Event(), ctx.Queue()
    warm = max(1, min(args.warmup, 2))
    procs = [ctx.Process(target=_ref_worker, args=(w, SWEEP[w % len(SWEEP)], warm, args.steps, start, q))
             for w in range(nw)]
    for pr in procs:
        pr.start()
    for _ in range(nw):
        assert q.get()[0] == "ready"
    t0 = time.perf_counter()
    start.set()
    done = [q.get() for _ in range(nw)]
    wall = time.perf_counter() - t0
    for pr in procs:
        pr.join()
    dofs = sum(d[3] for d in done)
    val = dofs / wall
    per = {}
    for d in done:
        per.setdefault(str(d[2]), []).append(d[4] / args.steps)
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": dict(CONFIG),
            "execution": {"parallelism": f"host: {nw} single-threaded processes"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": nw, "kind": "port",
                             "host_cores": cores,
                             "sample": f"{nw} worker processes (one per core, degree p = 2..6 round-robin), each "
                                       f"{args.steps} timed oracle matvecs at n_el=128 after {warm} warm-up; "
                                       "scipy CSR sum-factorisation, single-threaded per apply like the reference"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "per_degree_s": {k: statistics.median(v) for k, v in sorted(per.items())}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_1712_08565_b200 as M
    from paper_1712_08565_b200 import _lib

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ops = {}
    for p in SWEEP:
        space = M.tensor_space(p, N_EL)
        rule = M.build_tensor_rule(space)
        A = M.setup_stiffness(space, rule, M.identity_map(3))
        if args.path != "auto":
            A.set_path(args.path)
        x = torch.from_numpy(np.random.default_rng(0).standard_normal(space.n_dofs)).to(dev)
        y = torch.empty_like(x)
        info = A.info()
        ngrids = len({(min(a, b), max(a, b)) for a in range(3) for b in range(3)
                      if info["term_mask"] >> (3 * a + b) & 1})
        ops[p] = dict(A=A, x=x, y=y, N=space.n_dofs, Nq=A.n_points, grids=ngrids,
                      bytes=8 * (2 * space.n_dofs + ngrids * A.n_points), flops=A.apply_flops,
                      flops_active=A.apply_flops_active)
    stream = torch.cuda.current_stream()

    def step(evs=None):
        for p in SWEEP:
            o = ops[p]
            if evs is not None:
                evs[p][0].record(stream)
            o["A"].apply(o["x"], out=o["y"])
            if evs is not None:
                evs[p][1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = _lib.lib().mfwq_launch_count()
    per_p = {p: [] for p in SWEEP}
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        all_evs = []
        for _ in range(args.steps):
            evs = {p: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for p in SWEEP}
            step(evs)
            all_evs.append(evs)
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = _lib.lib().mfwq_launch_count() - launches0
    ms = t0.elapsed_time(t1)
    for evs in all_evs:
        for p in SWEEP:
            per_p[p].append(evs[p][0].elapsed_time(evs[p][1]))
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t)
    dofs_step = sum(ops[p]["N"] for p in SWEEP)
    value = dofs_step * args.steps * world / (ms * 1e-3)

    # e2e through the public API: pinned host x -> device -> matvec -> pinned host y
    hx = {p: torch.from_numpy(ops[p]["x"].cpu().numpy()).pin_memory() for p in SWEEP}
    hy = {p: torch.empty(ops[p]["N"], dtype=torch.float64, pin_memory=True) for p in SWEEP}
    for p in SWEEP:
        ops[p]["A"].apply_pipelined(hx[p], out=hy[p])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e2e_steps = max(1, min(args.steps, 20))  # long enough to amortise the pipeline fill and drain
    e0.record(stream)
    last = {}
    for _ in range(e2e_steps):
        for p in SWEEP:
            # pinned host x -> H2D (side stream) -> kernel -> D2H (side stream) into pinned host y:
            # consecutive calls overlap the two copy directions and the kernels
            _, last[p] = ops[p]["A"].apply_pipelined(hx[p], out=hy[p])
    for p in SWEEP:  # the timed region ends when the last result has landed in host memory
        stream.wait_event(last[p])
    e1.record(stream)
    torch.cuda.synchronize()
    for p in SWEEP:  # the host results are the device results
        yd = ops[p]["y"].cpu()  # equal up to the atomics' summation order
        assert float(torch.linalg.vector_norm(hy[p] - yd)) <= 1e-12 * float(torch.linalg.vector_norm(yd)), \
            "e2e host result differs from the device result"
    e2e_ms = e0.elapsed_time(e1)
    e2e_t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = dofs_step * e2e_steps * world / (float(e2e_t) * 1e-3)
    pcie = pcie_probe(torch, hx, ops, stream)
    dropin = dropin_e2e(torch, ops, dofs_step, e2e_steps)

    # on-the-fly coefficients (reference on_the_fly=True, operators.py:171-183): same sweep with C
    # evaluated in-kernel from C(xi1) instead of read from the N_q grids (secondary figure)
    otf_us = {}
    for p in SWEEP:
        o = ops[p]
        o["A"].set_on_the_fly(True)
        for _ in range(2):
            o["A"].apply(o["x"], out=o["y"])
        ts = []
        for _ in range(max(3, min(args.steps, 10))):
            e0.record(stream)
            o["A"].apply(o["x"], out=o["y"])
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        otf_us[p] = statistics.median(ts)
        o["A"].set_on_the_fly(False)
    otf = {"value": dofs_step / (sum(otf_us.values()) * 1e-6), "unit": UNIT, "per_degree_us": otf_us,
           "note": "on_the_fly=True: C evaluated in-kernel from C(xi1), no N_q coefficient grids stored or read"}

    # roofline of the matvec kernel, aggregated over the sweep
    pk = peaks()
    med = {p: statistics.median(per_p[p]) for p in SWEEP}
    tot_ms = sum(med.values())
    bytes_tot = sum(ops[p]["bytes"] for p in SWEEP)
    flops_act = sum(ops[p]["flops_active"] for p in SWEEP)
    achieved = bytes_tot / (tot_ms * 1e-3) / 1e9
    fp64 = flops_act / (tot_ms * 1e-3) / 1e12
    trf = traffic_from_profile()
    roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / pk["hbm_gbs"], "peak_src": pk["hbm_src"],
            "traffic": trf.get("bytes_per_launch") if trf else None,
            "traffic_src": trf.get("source") if trf else None,
            "fp64_achieved_tflops": fp64, "fp64_peak_tflops": pk["fp64_tflops"],
            "fp64_frac": fp64 / pk["fp64_tflops"], "fp64_src": pk["fp64_src"],
            "algorithmic_bytes": "8*(2N + G*Nq) per matvec, G = non-zero coefficient grids (3 on identity)"}

    pcg = cfg4 = cfg1 = None
    if args.pcg and world == 1:
        pcg = run_pcg(M, torch, dev)
        pcg["on_the_fly_variant"] = {k: v for k, v in run_pcg(M, torch, dev, otf=True).items()
                                     if k in ("iterations", "converged", "solve_s", "u_norm", "device_memory_used_gb",
                                              "matvec", "anchor")}
        cfg4 = run_cfg4(M, torch, dev)
        cfg1 = run_cfg1(M, torch, dev)
    slab = None
    if args.slab:  # cfg 5 strong scaling: the 1-GPU baseline here, the N-GPU headline in run_slab_headline
        slab = run_slab_pcg(M, torch, dev, rank, world)

    if rank == 0:
        cpu = None
        if args.cpu_baseline and world == 1:
            v, per, tot = cpu_sample()
            cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": "one oracle matvec per degree p=2..6 at n_el=128 (identical workload to one step; "
                             f"{tot:.1f} s of single-threaded scipy CSR sum-factorisation)",
                   "per_degree_s": {str(k): v2[0] for k, v2 in per.items()}}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": dict(CONFIG),
                "execution": {"l2": "coefficient grids 0.4-0.9 GB per degree > 126 MB L2 (no flush)",
                              "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                              "path": args.path},
                "per_degree_us": {str(p): 1e3 * med[p] for p in SWEEP},
                "per_degree_dofs": {str(p): ops[p]["N"] for p in SWEEP},
                "roofline": roof,
                "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": UNIT, "pcie": pcie,
                        "h2d_bytes_per_step": 8 * dofs_step, "d2h_bytes_per_step": 8 * dofs_step,
                        "api": "StiffnessOperator.apply_pipelined on pinned host tensors (H2D / kernel / D2H "
                               "overlapped across calls)",
                        "dropin": dropin},
                "gpu_launches": int(launches),
                "clocks": clk.summary(),
                "on_the_fly": otf,
                "pcg": pcg,
                "cfg4": cfg4,
                "cfg1": cfg1,
                "slab_pcg": slab}
        print(json.dumps(line), flush=True)


SLAB_METRIC = "MF-WQ cfg5 slab FD-PCG DoF-iterations/s (quarter ring p=6, n_el=512, xi3 slabs, to 1e-8)"
CFG5 = (6, 512)


def run_slab_pcg(M, torch, dev, rank, world, steps=1, warmup=1):
    """BASELINE configs[4]: the quarter ring at p=6, n_el=512 (137 M DoFs), FD-PCG to 1e-8 on
    b = default_rng(1), split into `world` xi3 slabs, one rank per GPU: the native comm-aware solver
    (mfwq_pcg_solve_comm; halo exchanges, FD all-to-all and allreduced scalars over NCCL).  world = 1
    is the single-GPU device PCG (the strong-scaling baseline).  Time = max over ranks (CUDA events)."""
    import torch.distributed as dist
    p, n_el = CFG5
    b_full = np.random.default_rng(1).standard_normal(M.tensor_space(p, n_el).n_dofs)
    t0 = time.perf_counter()
    space = M.tensor_space(p, n_el)
    rule = M.build_tensor_rule(space)
    geom = M.quarter_ring_map()
    t1 = time.perf_counter()
    if world > 1:
        from paper_1712_08565_b200.dist import Communicator, SlabSolver
        S = SlabSolver(space, rule, geom, Communicator.nccl())
        b = [torch.from_numpy(v.copy()).to(dev) for v in S.owned_slices(b_full)]
        solve = lambda: S.cg(b, tol=1e-8)  # noqa: E731
    else:
        A = M.setup_stiffness(space, rule, geom)
        P = M.FDPreconditioner(space)
        b1 = torch.from_numpy(b_full).to(dev)
        solve = lambda: M.cg(A.apply, b1, P.apply, tol=1e-8)  # noqa: E731
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t1
    for _ in range(warmup):
        solve()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        u, rep = solve()
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1) * 1e-3 / steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        u = u[0]
    nrm = torch.stack([(u * u).sum()])
    if world > 1:
        dist.all_reduce(nrm)
    secs = float(t)
    free, total = torch.cuda.mem_get_info()
    return {"metric": SLAB_METRIC, "value": space.n_dofs * rep.iterations / secs, "unit": "DoF-iterations/s",
            "scaling": "strong", "config": f"cfg5 quarter ring p={p} n_el={n_el}, xi3 slabs x{world}",
            "N": space.n_dofs, "iterations": rep.iterations, "converged": rep.converged,
            "final_rel_residual": rep.residuals[-1], "solve_s": secs, "setup_s": setup_s,
            "rule_s": t1 - t0, "u_norm": float(nrm[0]) ** 0.5, "device_memory_used_gb": (total - free) / 1e9,
            "solver": "mfwq_pcg_solve_comm (NCCL)" if world > 1 else "mfwq_pcg_solve (single GPU)"}


def solve_case(M, torch, dev, p, n_el, geom="ring", reps=1, otf=False):
    """Setup phases + FD-PCG to 1e-8 on b ~ N(0,1) seed 1, each phase timed (SURVEY §8(d) cfg 3-5)."""
    t0 = time.perf_counter()
    space = M.tensor_space(p, n_el)
    rule = M.build_tensor_rule(space)
    t1 = time.perf_counter()
    A = M.setup_stiffness(space, rule, M.quarter_ring_map() if geom == "ring" else M.identity_map(3),
                          on_the_fly=otf)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    P = M.FDPreconditioner(space)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    b = torch.from_numpy(np.random.default_rng(1).standard_normal(space.n_dofs)).to(dev)
    M.cg(A.apply, b, P.apply, tol=1e-8, maxit=2)  # warm-up
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    secs = []
    for _ in range(reps):
        e0.record()
        u, rep = M.cg(A.apply, b, P.apply, tol=1e-8)
        e1.record()
        torch.cuda.synchronize()
        secs.append(e0.elapsed_time(e1) * 1e-3)
    sec = sorted(secs)[len(secs) // 2]
    # FD apply alone (six modal DMMA GEMMs): 12 n^4 + N flops against the DMMA peak
    z = torch.empty_like(b)
    fts = []
    for _ in range(7):
        e0.record()
        P.apply(b, out=z)
        e1.record()
        torch.cuda.synchronize()
        fts.append(e0.elapsed_time(e1) * 1e-3)
    fsec = sorted(fts)[len(fts) // 2]
    # the matvec alone on x ~ N(0,1) seed 0, with its roofline (stored grids: 8 (2N + G Nq) bytes,
    # G = non-zero grids; on the fly: 16 N bytes, so the fp64 roof is the binding one)
    x = torch.from_numpy(np.random.default_rng(0).standard_normal(space.n_dofs)).to(dev)
    y = torch.empty_like(x)
    A.apply(x, out=y)
    mts = []
    for _ in range(9):
        e0.record()
        A.apply(x, out=y)
        e1.record()
        torch.cuda.synchronize()
        mts.append(e0.elapsed_time(e1) * 1e-3)
    msec = sorted(mts)[len(mts) // 2]
    tm = A.info()["term_mask"]
    grids = 0 if otf else len({(min(a, b), max(a, b)) for a in range(3) for b in range(3) if tm >> (3 * a + b) & 1})
    mbytes = 8 * (2 * space.n_dofs + grids * A.n_points)
    pk = peaks()
    mv = {"us": msec * 1e6, "dofs_per_s": space.n_dofs / msec, "grids_read": grids, "bytes": mbytes,
          "kernel_terms": A.info()["kernel_terms"],
          "roofline": {"bound": "hbm" if not otf else "fp64", "achieved_gbs": mbytes / msec / 1e9,
                       "peak_gbs": pk["hbm_gbs"], "hbm_frac": mbytes / msec / 1e9 / pk["hbm_gbs"],
                       "fp64_achieved_tflops": A.kernel_flops / msec / 1e12,
                       "fp64_frac": A.kernel_flops / msec / 1e12 / pk["fp64_tflops"],
                       "flops": "reference CostMeter count of the active terms (no on-the-fly coefficient charge)"}}
    fd_flops = sum(2 * 2 * n * n * space.n_dofs // n for n in space.n_per_dir) + space.n_dofs
    fd = {"apply_s": fsec, "flops": fd_flops, "tflops": fd_flops / fsec / 1e12, "peak_tflops": pk["fp64_tflops"],
          "frac": fd_flops / fsec / 1e12 / pk["fp64_tflops"], "bound": "tensor (fp64 DMMA)", "peak_src": pk["fp64_src"]}
    free, total = torch.cuda.mem_get_info()
    return {"device_memory_used_gb": (total - free) / 1e9, "on_the_fly": otf, "config": f"quarter ring p={p} n_el={n_el}" if geom == "ring" else f"cube p={p} n_el={n_el}",
            "N": space.n_dofs, "iterations": rep.iterations, "converged": rep.converged,
            "final_rel_residual": rep.residuals[-1], "solve_s": sec,
            "dof_iters_per_s": space.n_dofs * rep.iterations / sec,
            "setup_s": {"wq_rule": t1 - t0, "coeff_grids": t2 - t1, "fd": t3 - t2},
            "fd_apply": fd, "matvec": mv,
            "u_norm": float(torch.linalg.vector_norm(u)),
            "_u": u}


def anchor_check(r, key):
    """Iterations and ||u|| against the reference's own run at this configuration (make_anchors.py)."""
    a = anchors().get(key)
    u = r.pop("_u")
    if not a:
        return None
    return {"ref_iterations": a["iterations"], "iter_diff": r["iterations"] - a["iterations"],
            "u_norm_rel_diff": abs(float(torch_norm(u)) - a["norm"]) / a["norm"]}


def torch_norm(u):
    import torch
    return torch.linalg.vector_norm(u)


def pcie_probe(torch, hx, ops, stream):
    """Host<->device copy bandwidth with the e2e step's own pinned buffers: one direction alone and
    both at once (the ceiling of the pipelined e2e figure, which moves 2 x 88 MB per step)."""
    dx = {p: ops[p]["x"] for p in SWEEP}
    hy = {p: torch.empty_like(hx[p]).pin_memory() for p in SWEEP}
    nbytes = sum(hx[p].numel() * 8 for p in SWEEP)
    s2 = torch.cuda.Stream()
    res = {}
    for mode in ("h2d", "d2h", "both"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        s2.wait_stream(stream)
        for p in SWEEP:
            if mode in ("h2d", "both"):
                with torch.cuda.stream(stream):
                    dx[p].copy_(hx[p], non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    hy[p].copy_(ops[p]["y"], non_blocking=True)
        stream.wait_stream(s2)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        res[mode + "_gbs"] = (2 if mode == "both" else 1) * nbytes / (ms * 1e-3) / 1e9
    return res


def run_pcg(M, torch, dev, otf=False):
    """cfg 3: quarter ring, p=4, n_el=256 (17.2 M DoFs), FD-PCG to 1e-8 on b ~ N(0,1) seed 1."""
    r = solve_case(M, torch, dev, 4, 256, otf=otf)
    r["config"] = "cfg3 quarter ring p=4 n_el=256"
    r["anchor"] = anchor_check(r, "cfg3_u")
    return r


CFG4 = ((2, 128), (4, 126), (6, 124), (8, 122), (10, 120))


def run_cfg4(M, torch, dev):
    """BASELINE configs[3]: k-method sweep on the quarter ring, N = 128^3 at every degree; per-phase
    setup times (WQ rule, coefficient grids, FD eigendecomposition), FD-PCG to 1e-8, matvec roofline,
    iterations / ||u|| against the reference's run."""
    out = {}
    for p, n_el in CFG4:
        r = solve_case(M, torch, dev, p, n_el)
        r["anchor"] = anchor_check(r, f"cfg4_p{p}_u")
        out[str(p)] = {k: r[k] for k in ("N", "iterations", "converged", "solve_s", "setup_s", "matvec", "anchor")}
        out[str(p)]["n_el"] = n_el
        out[str(p)]["fd_apply_s"] = r["fd_apply"]["apply_s"]
    return out


def run_cfg1(M, torch, dev):
    """BASELINE configs[0] on the GPU: p=3, n_el=16 unit cube; one matvec on x = default_rng(0) (median of
    100, CUDA events) and FD-PCG to 1e-8 on the cube-sine load vector (host wall clock per solve)."""
    space = M.tensor_space(3, 16)
    geom = M.identity_map(3)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), geom)
    P = M.FDPreconditioner(space)
    x = torch.from_numpy(np.random.default_rng(0).standard_normal(space.n_dofs)).to(dev)
    b = M.assemble_rhs(space, geom, M.cube_sine_case().f)
    b = (b if torch.is_tensor(b) else torch.as_tensor(b)).to(dev)
    y = torch.empty_like(x)
    for _ in range(5):
        A.apply(x, out=y)
        u, rep = M.cg(A.apply, b, P.apply, tol=1e-8)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    mts = []
    for _ in range(100):
        e0.record()
        A.apply(x, out=y)
        e1.record()
        torch.cuda.synchronize()
        mts.append(e0.elapsed_time(e1) * 1e3)
    walls = []
    for _ in range(50):
        t0 = time.perf_counter()
        u, rep = M.cg(A.apply, b, P.apply, tol=1e-8)
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t0) * 1e6)
    return {"N": space.n_dofs, "matvec_us": statistics.median(mts), "pcg_wall_us": statistics.median(walls),
            "iterations": rep.iterations, "u_norm": float(torch.linalg.vector_norm(u)),
            "matvec_norm": float(torch.linalg.vector_norm(y))}


def dropin_e2e(torch, ops, dofs_step, steps):
    """The reference user's call: A.apply(numpy x) -> numpy y (pageable host memory, synchronous like
    the reference's numpy semantics), over the cfg2 sweep; host wall clock."""
    hx = {p: ops[p]["x"].cpu().numpy() for p in SWEEP}
    for p in SWEEP:
        ops[p]["A"].apply(hx[p])
    torch.cuda.synchronize()
    n = max(1, min(steps, 10))
    t0 = time.perf_counter()
    for _ in range(n):
        for p in SWEEP:
            yh = ops[p]["A"].apply(hx[p])
    dt = time.perf_counter() - t0
    assert isinstance(yh, np.ndarray)
    return {"value": dofs_step * n / dt, "unit": UNIT, "api": "StiffnessOperator.apply(np.ndarray) -> np.ndarray",
            "h2d_bytes_per_step": 8 * dofs_step, "d2h_bytes_per_step": 8 * dofs_step, "steps": n}


def run_slab_headline(args, rank, world, local):
    """N > 1: the headline is the cfg5 slab PCG on N GPUs (strong scaling; one rank per GPU, NCCL)."""
    import torch

    import paper_1712_08565_b200 as M
    from paper_1712_08565_b200 import _lib
    dev = torch.device("cuda", local)
    launches0 = _lib.lib().mfwq_launch_count()
    with ClockSampler(local) as clk:
        r = run_slab_pcg(M, torch, dev, rank, world, steps=args.steps, warmup=args.warmup)
    launches = _lib.lib().mfwq_launch_count() - launches0
    if rank == 0:
        line = {"metric": SLAB_METRIC, "value": r["value"], "unit": r["unit"], "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * r["solve_s"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": r["config"], "parallelism": f"xi3 slabs x{world} (NCCL)"},
                "slab_pcg": r, "gpu_launches": int(launches), "clocks": clk.summary(),
                "note": "N=1 lines carry the same cfg5 solve on one GPU under 'slab_pcg' (the strong-scaling "
                        "baseline); the single-GPU headline is the cfg2 matvec sweep"}
        print(json.dumps(line), flush=True)


def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: launch N ranks (one per GPU) through torch.distributed.run."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    rank, world, local = dist_info()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        if world > 1 and args.slab:
            run_reference_slab(args, rank, world)
        else:
            run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        run_slab_headline(args, rank, world, local)
        dist.destroy_process_group()
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
