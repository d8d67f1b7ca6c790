"""Benchmark: eigenpairs/s of the spectrum-sliced shift-invert Lanczos solve.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3]
                    [--impl ours|reference] [--streams S]

One step = the whole hot path over the workload: factor every uniform
shift (inertia), run restarted shift-invert Lanczos on every slice
(sigma_k, sigma_k+1], lock every eigenpair the inertia promises, and bring
eigenvalues + eigenvectors to the host.  Default workload: BASELINE
configs[2] (cfg3: 2D 256x256 elements, p=4, rIGA BS=16, 16 uniform
slices over [0, lam_e], first 2000 eigenpairs) -- the configuration the
metric is quoted on "at 1/2/4/8 B200" with slices distributed across GPUs.

``value`` is measured with the system resident in HBM; ``e2e`` through the
public API from host CSR buffers (upload, ordering, symbolic, solve,
eigenpairs to host).  ``--impl reference`` times the reference's own
package (rigaeig v0.1.0, installed by build() into oracle/_ref; the oracle
port when it is absent) on the host cores, on a bounded sample of the
workload (``--sample-q 0``: the whole workload, for calibration).
Multi-GPU: one process per GPU (torchrun); slices are partitioned by LPT
over the boundary inertias (weak in the number of slices per GPU:
"scaling" is "strong" -- the total work is fixed).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # many concurrent slice streams
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "backend:cudaMallocAsync")  # stream-ordered torch allocations

if "--impl" in sys.argv and "reference" in sys.argv:
    # the reference's CPU path: one BLAS thread per worker process
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_FP64_TFLOPS = 37.16  # tools/fp64_peak.cu on this pool's B200 (DMMA m8n8k4 loop)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--streams", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sample-q", type=int, default=8, help="eigenpairs per slice in the CPU sample")
    ap.add_argument("--ldlt-config", default="cfg5", help="config of the LDL^T TFLOP/s line ('' to skip)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(
        os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------------------
# CPU reference arm (oracle port of the reference path, bounded sample)
# ---------------------------------------------------------------------------

_W = {}
REF_DIR = os.path.join(ROOT, "oracle", "_ref")  # the reference package installed by build() (rigaeig v0.1.0)


def ref_kind() -> str:
    """'reference' when the reference's own package (oracle/_ref/rigaeig) is importable, else 'port'."""
    return "reference" if os.path.isdir(os.path.join(REF_DIR, "rigaeig")) else "port"


def _ref_module():
    if ref_kind() == "reference":
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import rigaeig

        return rigaeig
    from oracle import rigaeig_port

    return rigaeig_port


def _worker_init(cfgname):
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:
        pass
    from paper_2009_08167_b200.configs import CONFIGS

    c = CONFIGS[cfgname]
    R = _ref_module()
    _W["R"] = R
    _W["sys"] = R.build_system(c.d, c.ne, c.p, c.level)


def _worker_task(task):
    k, lo, hi, m = task
    t0 = time.perf_counter()
    r = _W["R"].solve_slice(_W["sys"], (lo, hi), seed=k, m=m)
    return k, r.eigenvalues.size, r.expected_count, time.perf_counter() - t0


def cpu_sample_tasks(cfgname, q):
    """Bounded sample: the q lowest eigenpairs above every uniform shift, m = 2 q (q = 0: the whole workload,
    every slice with m = 2 count_k as the GPU arm)."""
    from oracle import rigaeig_port as O
    from paper_2009_08167_b200.configs import CONFIGS

    c = CONFIGS[cfgname]
    lam = O.kronecker_spectrum(c.d, c.ne, c.p, c.level)
    lam_e, _ = O.lambda_e_for(lam, c.n0)
    tasks = []
    for k in range(c.slices):
        lo, top = k * lam_e / c.slices, (k + 1) * lam_e / c.slices
        i0 = int(np.sum(lam < lo))
        if q <= 0:
            cnt = int(np.sum((lam > lo) & (lam <= top)))
            tasks.append((k, lo, top, 2 * cnt, cnt))
            continue
        i = i0 + q - 1
        while i + 1 < lam.size and lam[i + 1] - lam[i] <= 1e-8 * lam[i + 1]:
            i += 1
        hi = 0.5 * (lam[i] + lam[i + 1])
        tasks.append((k, lo, hi, 2 * (i + 1 - i0), i + 1 - i0))
    # longest first: the pool drains evenly
    return sorted(tasks, key=lambda t: -t[4])


def run_cpu_sample(cfgname, q, steps=1, warmup=0, proc_bytes=0.0):
    import multiprocessing as mp

    tasks = cpu_sample_tasks(cfgname, q)
    workers = min(os.cpu_count() or 1, len(tasks))
    if proc_bytes > 0:  # host memory: each process holds the pencil and one factor
        import psutil

        workers = max(1, min(workers, int(0.6 * psutil.virtual_memory().available // proc_bytes)))
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    ctxmp = mp.get_context("spawn")
    times = []
    with ctxmp.Pool(workers, initializer=_worker_init, initargs=(cfgname,)) as pool:
        for it in range(warmup + steps):
            t0 = time.perf_counter()
            out = pool.map(_worker_task, [t[:4] for t in tasks], chunksize=1)
            dt = time.perf_counter() - t0
            for k, found, exp, _ in out:
                if found != exp:
                    raise RuntimeError(f"CPU sample slice {k}: {found} != {exp}")
            if it >= warmup:
                times.append(dt)
    pairs = sum(t[4] for t in tasks)
    return pairs, times, workers


def _sample_text(c, q, pairs, workers, kind):
    what = ("the reference's rigaeig.solve_slice (oracle/_ref, rigaeig v0.1.0)" if kind == "reference"
            else "oracle port of ref solve_slice")
    if q <= 0:
        return (f"{c.name}: the whole workload ({pairs} pairs), every uniform slice with m = 2 count_k, {what}, "
                f"{workers} processes x 1 BLAS thread (ref cli.py:208-210 ProcessPool mode)")
    return (f"{c.name}: the {q} lowest eigenpairs above each of the {c.slices} uniform shifts ({pairs} pairs), "
            f"{what} with m = 2q, {workers} processes x 1 BLAS thread (ref cli.py:208-210 ProcessPool mode)")


CALIBRATION = os.path.join(ROOT, "profiles", "r2_reference_full_cfg3.json")


def _calibration(q):
    """Full-workload vs sample rate of the reference on the GPU box host (tools: bench.py --impl reference
    --sample-q 0, committed under profiles/)."""
    try:
        cal = json.load(open(CALIBRATION))
    except (OSError, ValueError):
        return None
    return {"full_run_eigenpairs_per_s": cal.get("value"), "full_run_s": cal.get("ms_per_step", 0) / 1e3,
            "source": os.path.relpath(CALIBRATION, ROOT), "sample_q": q}


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2009_08167_b200.configs import CONFIGS

    c = CONFIGS[args.config]
    kind = ref_kind()
    warm = min(args.warmup, 1)
    pairs, times, workers = run_cpu_sample(args.config, args.sample_q, steps=args.steps, warmup=warm)
    t = float(np.mean(times))
    v = pairs / t
    sample = _sample_text(c, args.sample_q, pairs, workers, kind)
    cal = _calibration(args.sample_q)
    if cal and cal["full_run_eigenpairs_per_s"]:
        cal["sample_over_full"] = v / cal["full_run_eigenpairs_per_s"]
    line = {"impl": "reference", "metric": "eigenpairs/s", "value": v, "unit": "eigenpairs/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": warm,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (deterministic pencil, seeded start vectors)",
            "config": {"workload": c.text, "config": c.name, "sample": sample},
            "cpu_baseline": {"value": v, "unit": "eigenpairs/s", "cores": workers, "kind": kind,
                             "sample": sample, "calibration": cal},
            "e2e": {"value": v, "unit": "eigenpairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "per_step_s": times}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


class ClockSampler:
    """SM clocks + throttle reasons during the timed region, sampled in-process
    through NVML (the library nvidia-smi reads) every 250 ms on a daemon
    thread; falls back to an nvidia-smi subprocess if NVML is unavailable."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        import threading

        self.sm, self.mx, self.reasons = [], [], set()
        self.stop_ev = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.bits = {"hw_slowdown": pynvml.nvmlClocksThrottleReasonHwSlowdown,
                         "hw_thermal_slowdown": getattr(pynvml, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                         "sw_thermal_slowdown": getattr(pynvml, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                         "sw_power_cap": pynvml.nvmlClocksThrottleReasonSwPowerCap}
            self.ok = True
        except Exception:
            self.ok = False
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        while not self.stop_ev.is_set():
            if self.ok:
                try:
                    nv = self.nv
                    self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                    self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)))
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                    for nm in self.NAMES:
                        if r & self.bits[nm]:
                            self.reasons.add(nm)
                except Exception:
                    pass
            self.stop_ev.wait(0.25)

    def stop(self):
        self.stop_ev.set()
        self.t.join()
        if not self.ok or not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": float(max(self.mx)),
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "NVML (in-process)"}


def dcgs_bytes(R, n):
    """Algorithmic bytes of the step's Gram-Schmidt (delayed CGS2, SURVEY 8d's
    2 passes x 2 x R x N x 8 reorganised): one dots sweep reads R rows of
    MV / LM and the two vectors, one update sweep reads R rows of V / L and
    the two vectors and writes the two results."""
    return 2.0 * R * n * 8.0 + 6.0 * n * 8.0


def ncu_traffic(kernel, d):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed ncu --set full capture (profiles/ncu_traffic.json), scaled
    to this launch's algorithmic bytes (the capture may use another R)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        rec = json.load(open(p))[kernel]
        return rec["dram_bytes"] * d["bytes_per_launch"] / rec["algorithmic_bytes"]
    except Exception:
        return None


def ldlt_rate(P, D, cfgname, flush, reps=3):
    """LDL^T FP64 rate on the largest single-GPU config (the one whose fronts
    exercise the DMMA frontal updates): median device time of `reps`
    factorizations at its first interior uniform shift, L2 flushed before
    each; work = the reference's sum colcount^2 (sparsela.py:258)."""
    import numpy as np
    import torch
    from paper_2009_08167_b200.configs import CONFIGS
    from paper_2009_08167_b200.sparsela import Symbolic, numeric_factor

    cc = CONFIGS[cfgname]
    t0 = time.perf_counter()
    s = P.build_system(cc.d, cc.ne, cc.p, cc.level)
    lam_e, _ = P.choose_lambda_e(s, cc.n0)
    sh = P.uniform_shifts(lam_e, cc.slices)
    sym = Symbolic.on_device(s.device, P.separator_ordering(s))
    t_setup = time.perf_counter() - t0
    ms = []
    for _ in range(reps + 1):
        flush.zero_()
        torch.cuda.synchronize()
        f = numeric_factor(sym, float(sh[1]))
        ms.append(f.device_ms)
        flops = f.factor_flops
        del f
    fm = float(np.median(ms[1:]))
    tf = flops / (fm / 1e3) / 1e12
    # the frontal Schur-complement update kernels in situ (north_star: "LDL^T frontal updates at >= 50 % of
    # FP64 tensor peak"): CUDA events around each k_trail128 launch of one more factorization, work = their
    # algorithmic flops (2 K per updated lower-triangle entry)
    import ctypes

    from paper_2009_08167_b200 import _lib

    L = _lib.lib()
    L.riga_prof_reset()
    L.riga_prof_enable(1)
    flush.zero_()
    torch.cuda.synchronize()
    f = numeric_factor(sym, float(sh[1]))
    torch.cuda.synchronize()
    L.riga_prof_enable(0)
    pm, pw, pc = np.zeros(8), np.zeros(8), np.zeros(8, np.int64)
    L.riga_prof_read(_lib.ptr(pm), _lib.ptr(pw), _lib.ptr(pc), 8)
    L.riga_prof_reset()
    del f
    upd = {"ms": float(pm[6]), "flops": float(pw[6]), "launches": int(pc[6]),
           "achieved": float(pw[6]) / (pm[6] / 1e3) / 1e12 if pm[6] > 0 else 0.0, "unit": "TFLOP/s",
           "share_of_factor_flops": float(pw[6]) / flops,
           "how": "CUDA events around every k_trail128 launch of one factorization (prof scopes on: the "
                  "factorization then runs on one stream, no look-ahead, so each scope times its kernel alone), "
                  "algorithmic flops of the lower-triangle updates"}
    upd["frac"] = upd["achieved"] / MEASURED_FP64_TFLOPS
    out = {"config": cfgname, "N": s.dof_count, "ms": fm, "flops_per_launch": flops, "achieved": tf,
           "unit": "TFLOP/s", "peak": MEASURED_FP64_TFLOPS, "frac": tf / MEASURED_FP64_TFLOPS,
           "peak_source": "tools/fp64_peak.cu DMMA loop on this pool's B200",
           "how": f"median of {reps} factorizations (after one warm-up), CUDA events on the factor stream, "
                  "L2 flushed before each; flops = reference sum colcount^2",
           "frontal_updates": upd, "setup_s": t_setup}
    del sym, s
    torch.cuda.synchronize()
    return out


def kernel_roofline(P, D, L, system, shifts, sym, perm, c, flush, reps=10):
    """Time the hot kernels of one Lanczos step on the benchmark's own data
    (the middle slice: its factor, its m-vector basis), each bracketed by
    CUDA events on the engine stream with an L2 flush before every launch.
    Algorithmic work per launch: CGS2 = 2 passes x 2 x R x N x 8 B
    (R = basis rows), solve = 16 fill_nnz + 32 N bytes, SpMV = 12 nnz +
    4 (N+1) + 16 N bytes, factor = sum colcount^2 flops."""
    import ctypes

    import numpy as np
    import torch
    from paper_2009_08167_b200 import _lib
    from paper_2009_08167_b200.eigensolver import DeviceShiftInvert
    from paper_2009_08167_b200.sparsela import numeric_factor

    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else open(os.devnull) as fh:
        try:
            peaks = json.load(fh)
        except Exception:
            peaks = {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    src = "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else "fallback 6650 GB/s"
    ctx = D.Context()
    k = len(shifts) // 2
    n = system.dof_count
    with ctx:
        f = numeric_factor(sym, float(shifts[k]), ctx)
        fms = []
        for _ in range(3):
            with torch.cuda.stream(ctx.stream):
                flush.sum()
            g = numeric_factor(sym, float(shifts[k]), ctx)
            fms.append(g.device_ms)
            del g
        lam_cnt = int(np.sum(P.kronecker_spectrum(system) < shifts[k + 1])) - f.n_negative
        m = min(2 * max(lam_cnt, 1), n - 1)
        st = P.LanczosState(DeviceShiftInvert(f, system.M), n, mass=system.M, shift=f.sigma, max_dim=m + 1,
                            rng=np.random.default_rng(0), ctx=ctx)
        P.lanczos_extend(st, m)
        x = torch.randn(n, dtype=torch.float64, device=f"cuda:{ctx.device}")
        y = torch.empty_like(x)
        b = torch.randn(n, dtype=torch.float64, device=f"cuda:{ctx.device}")

        def timed(fn, stream=None):
            stream = stream or ctx.stream
            ts = []
            for _ in range(reps):
                with torch.cuda.stream(stream):
                    flush.sum()  # read-flush: evicts L2 without leaving dirty lines to write back
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fn()
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            return float(np.median(ts))

        rows = ctypes.c_int64(0)
        st.k = st.k  # basis full (k = m): the probe uses rows [0, k] + locked
        # the two sweeps between events recorded inside the probe, around the kernels alone (the probe's
        # upload of the recurrence state is not part of a step's sweeps)
        ts = []
        for _ in range(reps):
            with torch.cuda.stream(ctx.stream):
                flush.sum()
            _lib.check(L.riga_lanczos_dcgs_probe(st.handle, _lib.ptr(x), ctypes.byref(rows)))
            ms = ctypes.c_float(0.0)
            _lib.check(L.riga_lanczos_last_extend_ms(st.handle, ctypes.byref(ms)))
            ts.append(float(ms.value))
        t_cgs = float(np.median(ts))
        t_sol = timed(lambda: f.solve_device(b, y))
        # the system's SpMV runs on the system's context stream
        sstream = system.device.ctx.stream
        t_mv = timed(lambda: _lib.check(L.riga_spmv(system.device.handle, 1, 0.0, _lib.ptr(b), _lib.ptr(y))),
                     sstream)
        ctx.synchronize()
    nnz = system.K.nnz
    work = {"dcgs_sweeps": dcgs_bytes(rows.value, n), "supernodal_solve": 16.0 * f.fill_nnz + 32.0 * n,
            "csr_spmv": 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n}
    times = {"dcgs_sweeps": t_cgs, "supernodal_solve": t_sol, "csr_spmv": t_mv}
    cats = {}
    for name in work:
        ach = work[name] / (times[name] / 1e3) / 1e9
        cats[name] = {"ms": times[name], "bytes_per_launch": work[name], "achieved": ach, "unit": "GB/s",
                      "peak": hbm, "frac": ach / hbm}
    cats["dcgs_sweeps"]["rows"] = int(rows.value)
    fm = float(np.median(fms))
    tf = f.factor_flops / (fm / 1e3) / 1e12
    cats["ldlt_factor"] = {"ms": fm, "flops_per_launch": f.factor_flops, "achieved": tf, "unit": "TFLOP/s",
                           "peak": MEASURED_FP64_TFLOPS, "frac": tf / MEASURED_FP64_TFLOPS,
                           "peak_source": "tools/fp64_peak.cu DMMA loop on this pool's B200"}
    return cats, hbm, src, reps


def concurrent_rates(P, D, L, system, shifts, sym, streams, m, reps=6):
    """Aggregate throughput of the two hot kernels under the production
    concurrency: `streams` slice streams, each with its own factor and an
    m-vector Lanczos basis, all launching at once.  Timed with CUDA events:
    every stream waits on one start event; the span is start -> the last
    stream's end event."""
    import ctypes
    import threading

    import numpy as np
    import torch
    from paper_2009_08167_b200 import _lib
    from paper_2009_08167_b200.eigensolver import DeviceShiftInvert
    from paper_2009_08167_b200.sparsela import numeric_factor

    n = system.dof_count
    S = len(shifts) - 1
    # as many concurrent (factor, basis) pairs as fit, like the slice driver's memory plan
    st_ = sym.stats
    per = 8.0 * (1.35 * st_.get("panel_entries", 0) + 6 * n) + 16.0 * (m + 2) * n * 2
    torch.cuda.empty_cache()
    free_b, _ = torch.cuda.mem_get_info()
    streams = max(1, min(streams, int(0.7 * free_b // max(per, 1.0))))
    ctxs = [D.Context() for _ in range(streams)]
    facts, states, vecs = [], [], []
    for i, ctx in enumerate(ctxs):
        with ctx:
            f = numeric_factor(sym, float(0.5 * (shifts[i % S] + shifts[i % S + 1])), ctx)
            st = P.LanczosState(DeviceShiftInvert(f, system.M), n, mass=system.M, shift=f.sigma, max_dim=m + 1,
                                rng=np.random.default_rng(i), ctx=ctx)
            facts.append(f)
            states.append(st)
            vecs.append((torch.randn(n, dtype=torch.float64, device="cuda"),
                         torch.empty(n, dtype=torch.float64, device="cuda")))

    def run_all(fn):
        th = [threading.Thread(target=fn, args=(i,)) for i in range(streams)]
        for t in th:
            t.start()
        for t in th:
            t.join()

    def ext(i):
        with ctxs[i]:
            P.lanczos_extend(states[i], m)
            ctxs[i].synchronize()

    run_all(ext)
    rows = ctypes.c_int64(0)
    _lib.check(L.riga_lanczos_dcgs_probe(states[0].handle, _lib.ptr(vecs[0][0]), ctypes.byref(rows)))
    graphs = []
    for i, ctx in enumerate(ctxs):
        with ctx:
            b, y = vecs[i]
            facts[i].solve_device(b, y)
            ctx.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=ctx.stream, capture_error_mode="thread_local"):
                for _ in range(10):
                    facts[i].solve_device(b, y)
            graphs.append(g)
    torch.cuda.synchronize()

    def span(work):
        t0 = torch.cuda.Event(enable_timing=True)
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(streams)]
        torch.cuda.synchronize()
        t0.record(torch.cuda.current_stream())
        for ctx in ctxs:
            ctx.stream.wait_event(t0)

        def go(i):
            with ctxs[i]:
                work(i)
                ends[i].record(ctxs[i].stream)

        run_all(go)
        torch.cuda.synchronize()
        return max(t0.elapsed_time(e) for e in ends)

    def cgs(i):
        for _ in range(reps):
            _lib.check(L.riga_lanczos_dcgs_probe(states[i].handle, _lib.ptr(vecs[i][0]), ctypes.byref(ctypes.c_int64())))

    def sol(i):
        for _ in range(reps):
            graphs[i].replay()

    span(cgs)
    t_cgs = span(cgs)
    span(sol)
    t_sol = span(sol)
    out = {"streams": streams,
           "dcgs_sweeps": {"ms_span": t_cgs, "launches": streams * reps, "rows": int(rows.value),
                           "bytes": streams * reps * dcgs_bytes(rows.value, n)},
           "supernodal_solve": {"ms_span": t_sol, "launches": streams * reps * 10,
                                "bytes": streams * reps * 10 * (16.0 * facts[0].fill_nnz + 32.0 * n)}}
    for k in ("dcgs_sweeps", "supernodal_solve"):
        out[k]["achieved"] = out[k]["bytes"] / (out[k]["ms_span"] / 1e3) / 1e9
        out[k]["per_launch_ms"] = out[k]["ms_span"] / out[k]["launches"]
    del graphs, states, facts, ctxs
    torch.cuda.synchronize()
    return out


def ours(args):
    import ctypes

    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        # one process per GPU; RIGA_DIST_BACKEND=gloo (+ more ranks than GPUs) only
        # exercises the multi-rank code path functionally, it is not a scaling run
        backend = os.environ.get("RIGA_DIST_BACKEND", "nccl")
        local = local % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    import paper_2009_08167_b200 as P
    from paper_2009_08167_b200 import _lib
    from paper_2009_08167_b200 import device as D
    from paper_2009_08167_b200.assembly import DeviceSystem, DiscreteSystem, SymSparseMatrix
    from paper_2009_08167_b200.configs import CONFIGS
    from paper_2009_08167_b200.sparsela import Symbolic

    L = _lib.lib()
    c = CONFIGS[args.config]
    dev = torch.cuda.current_device()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    coll_dev = f"cuda:{dev}" if os.environ.get("RIGA_DIST_BACKEND", "nccl") == "nccl" else "cpu"

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        torch.distributed.all_reduce(t)
        return float(t.item())

    # ---- setup (untimed): device assembly, lam_e, ordering, symbolic -------
    system = P.build_system(c.d, c.ne, c.p, c.level)
    lam_e, count = P.choose_lambda_e(system, c.n0)
    shifts = P.uniform_shifts(lam_e, c.slices)
    perm = P.separator_ordering(system)
    from paper_2009_08167_b200.slicing import solve_plan, solve_sub_levels

    per_gpu = -(-c.slices // world)
    with solve_plan(solve_sub_levels(min(args.streams, per_gpu))):
        sym = Symbolic.on_device(system.device, perm)
    seeds = list(range(c.slices))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{dev}")  # 256 MB > L2

    def step():
        return P.solve_uniform_slices(system, shifts, seeds=seeds, streams=args.streams, rank=rank,
                                      world=world, pencil_symbolic=sym, perm=perm)

    GATE = 1e-8  # north_star: ||K u - lam M u|| / (|lam| ||M u||) of every returned pair

    def check(r):
        # counts exact (inertia) and every pair inside the residual gate, every step
        assert int(r.found.sum()) == count, (r.found, count)
        assert r.max_residual <= GATE, r.max_residual
        return r.max_residual

    max_res = 0.0
    for _ in range(args.warmup):
        r = step()
        check(r)
    # ---- timed region ------------------------------------------------------
    times, found = [], 0
    n0 = ctypes.c_int64()
    L.riga_launch_count(ctypes.byref(n0))
    clocks = ClockSampler(dev)
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = step()
        torch.cuda.synchronize()
        e1.record()
        barrier()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
        found = int(r.found.sum())
        max_res = max(max_res, check(r))
    clk = clocks.stop()
    n1 = ctypes.c_int64()
    L.riga_launch_count(ctypes.byref(n1))
    t_step = max_over_ranks(float(np.mean(times)))
    value = found / t_step
    launches = int(sum_over_ranks(float(n1.value - n0.value)))
    assert found == count, (found, count)

    # ---- e2e through the public API from host buffers -----------------------
    e2e = None
    if not args.no_e2e:
        # the step's inputs in pinned host memory (one pattern, two value arrays)
        import scipy.sparse as sps

        K0, M0 = system.K.csr, system.M.csr

        def pinned(a, dt):
            t = torch.empty(a.size, dtype=dt, pin_memory=True)
            t.numpy()[:] = a
            return t

        rp_t = pinned(np.asarray(K0.indptr, np.int32), torch.int32)  # scipy keeps one index dtype
        ci_t = pinned(np.asarray(K0.indices, np.int32), torch.int32)
        kv_t = pinned(np.asarray(K0.data, np.float64), torch.float64)
        mv_t = pinned(np.asarray(M0.data, np.float64), torch.float64)
        rp_h, ci_h = rp_t.numpy(), ci_t.numpy()
        Kh = sps.csr_array((kv_t.numpy(), ci_h, rp_h), shape=K0.shape)
        Mh = sps.csr_array((mv_t.numpy(), ci_h, rp_h), shape=M0.shape)
        Mh.indices, Mh.indptr = Kh.indices, Kh.indptr  # one pattern object
        h2d = Kh.nnz * (8 + 8 + 4) + (Kh.shape[0] + 1) * 8
        ctx = D.current()
        e2e_times, d2h = [], 0
        for _ in range(max(1, min(args.steps, 3))):
            flush.zero_()
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dsys = DeviceSystem.upload(ctx, Kh, Mh)
            dsys.attach_kron(system.k1d, system.m1d)  # the public DiscreteSystem's 1D factors
            sys2 = DiscreteSystem(SymSparseMatrix(device=dsys, which=0), SymSparseMatrix(device=dsys, which=1),
                                  system.spaces, system.dim, system.dof_count, system.k1d, system.m1d, dsys)
            perm2 = P.separator_ordering(sys2)
            r2 = P.solve_uniform_slices(sys2, shifts, seeds=seeds, streams=args.streams, rank=rank,
                                        world=world, perm=perm2)
            torch.cuda.synchronize()
            e1.record()
            barrier()
            torch.cuda.synchronize()
            e2e_times.append(e0.elapsed_time(e1) / 1e3)
            d2h = sum(v.nbytes for v in r2.local_vectors.values()) + 8 * int(r2.found.sum())
            max_res = max(max_res, check(r2))
            del dsys, sys2, r2
        te = max_over_ranks(float(np.mean(e2e_times)))
        e2e = {"value": count / te, "unit": "eigenpairs/s", "h2d_bytes_per_step": int(h2d),
               "how": "public API per step: upload of the pinned host CSR (K, M values + pattern) and the 1D "
                      "factors, separator ordering, symbolic analysis, solve_uniform_slices, eigenvectors to host",
               "d2h_bytes_per_step": int(sum_over_ranks(d2h)), "ms_per_step": te * 1e3,
               "per_step_s": [round(t, 4) for t in e2e_times]}

    # ---- roofline: the step's kernels timed with CUDA events on their stream ---
    cats, hbm, src, reps = kernel_roofline(P, D, L, system, shifts, sym, perm, c, flush)
    ldlt_large = None
    if rank == 0 and args.ldlt_config and args.ldlt_config != c.name:
        ldlt_large = ldlt_rate(P, D, args.ldlt_config, flush)
    rows_avg = float(r.counters.phase_s.get("cgs_rows", 0.0)) / max(r.counters.nfb, 1)
    m_mid = int(2 * np.median(r.expected))
    conc = concurrent_rates(P, D, L, system, shifts, sym, args.streams, m_mid)
    # per Lanczos step, in the concurrent regime: one solve, two Gram-Schmidt
    # passes over rows_avg rows (scaled from the probe's R), one SpMV
    share = {"supernodal_solve": conc["supernodal_solve"]["per_launch_ms"],
             "dcgs_sweeps": conc["dcgs_sweeps"]["per_launch_ms"] * rows_avg / max(conc["dcgs_sweeps"]["rows"], 1)}
    for k_ in ("dcgs_sweeps", "supernodal_solve"):
        cats[k_]["concurrent"] = {"achieved": conc[k_]["achieved"], "frac": conc[k_]["achieved"] / hbm,
                                  "unit": "GB/s", "streams": conc["streams"],
                                  "per_launch_ms_aggregate": conc[k_]["per_launch_ms"]}
        cats[k_]["step_ms_aggregate"] = share[k_]
    # dominant = largest aggregate device time per Lanczos step in the
    # production (16-stream) regime
    dom = max(share, key=lambda k_: share[k_])
    d = cats[dom]
    roofline = {"bound": "hbm", "achieved": d["achieved"], "peak": hbm, "unit": "GB/s", "frac": d["frac"],
                "traffic": ncu_traffic(dom, d), "kernel": dom, "peak_source": src,
                "per_launch_bytes": d["bytes_per_launch"],
                "how": "isolated launch: CUDA events on the engine stream around the kernels, L2 flushed (256 MB "
                       "read) before each launch, median of %d" % reps,
                "concurrent": d["concurrent"],
                "rows_avg_timed_region": rows_avg,
                "step_share_aggregate": {k_: v / sum(share.values()) for k_, v in share.items()}}

    line = {"metric": "eigenpairs/s", "value": value, "unit": "eigenpairs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (deterministic B-spline Laplace pencil; seeded standard-normal start vectors)",
            "config": {"workload": c.text, "config": c.name, "d": c.d, "ne": c.ne, "p": c.p,
                       "level": c.level, "N": system.dof_count, "eigenpairs": count, "slices": c.slices,
                       "lambda_e": lam_e, "streams_per_gpu": args.streams,
                       "parallelism": f"slices partitioned over {world} GPU(s) (LPT on inertia counts)",
                       "l2": "working set > L2 (V+MV 2x251xNx8 B = 369 MB per slice); 256 MB flush between steps"},
            "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "roofline_by_kernel": cats,
            "ldlt": ldlt_large if ldlt_large else cats.get("ldlt_factor"),
            "ldlt_workload": cats.get("ldlt_factor"), "clocks": clk,
            "parity": {"counts_exact": True, "max_residual": max_res, "residual_gate": GATE,
                       "how": "every step (warm-up, timed, e2e): found == inertia count per slice and the device "
                              "residual ||Ku - lam Mu|| / (|lam| ||Mu||) of every returned pair <= gate"},
            "timing": {"per_step_s": times, "boundary_s": r.timings["boundary_s"],
                       "slices_s": r.timings["slices_s"], "streams_used": r.timings.get("streams_used")}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # oracle process footprint: L (value + index) with working copies, plus the CSR pencil
        pb = 3.0 * 12.0 * sym.stats["fill_nnz"] + 40.0 * system.K.nnz
        pairs, ctimes, workers = run_cpu_sample(args.config, args.sample_q, steps=1, proc_bytes=pb)
        cal = _calibration(args.sample_q)
        if cal and cal["full_run_eigenpairs_per_s"]:
            cal["sample_over_full"] = pairs / ctimes[0] / cal["full_run_eigenpairs_per_s"]
        line["cpu_baseline"] = {"value": pairs / ctimes[0], "unit": "eigenpairs/s", "cores": workers,
                                "kind": ref_kind(),
                                "sample": _sample_text(c, args.sample_q, pairs, workers, ref_kind()),
                                "calibration": cal}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    return ours(args)


if __name__ == "__main__":
    sys.exit(main())
