"""SSsNAL time-to-KKT benchmark (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 1]

Workload (BASELINE.json configs[1]): linear C-SVC dual, dense fp64 A of
n = 50,000 samples x q = 300 features drawn as a two-class Gaussian mixture
(means +-0.5*1, identity covariance, balanced labels), C = 1, cold start
(x0 = w0 = 0), solved to relative KKT residual 1e-6.  One "step" is one full
solve.  Synthetic data (the reference's LIBSVM files are not available offline).

  value    device time of the solve with A already resident in HBM (CUDA events on
           the solver's stream), max over ranks; L2 (126 MB) is flushed with a
           256 MB write before every timed step.
  e2e      the same solve through the public API from HOST buffers: upload of A, y
           (pinned), problem construction, solve, and the read-back of x.
  roofline the dominant kernel by device time inside the timed region, algorithmic
           bytes per launch / mean launch time, against MEASURED_PEAKS.json.
  cpu_baseline  the numpy oracle (tests' CPU restatement of the reference) solving the
           same problem on the host cores, rank 0, N = 1.

--impl reference times that CPU restatement alone (the reference package itself is
pure Python and cannot be run on the GPU box).  N > 1 runs N
independent replicas (one per GPU) of the single-GPU solve.
"""

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

METRIC = "SSNAL time-to-KKT 1e-6 (C-SVC dense fp64, config 1: n=50000 x q=300)"
TOL = 1e-6


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML inside the
    timed region -- between solves, after each step's closing event, so the query
    never lands inside a latency-bound solve (an nvidia-smi process polling every
    200 ms did, adding ms-scale stalls to the host syncs).  Falls back to a single
    nvidia-smi query per sample when NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index):
        self.index = index
        self.sm, self.smax, self.reasons = [], [], set()
        self.nv = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self.nv = None

    def start(self):
        self.sample()

    def sample(self):
        try:
            if self.nv is not None:
                nv = self.nv
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                self.smax.append(float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, attr in self.REASONS:
                    if mask & getattr(nv, attr, 0):
                        self.reasons.add(name)
                return
            out = subprocess.run(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10).stdout
            r = [c.strip() for c in out.split(",")]
            self.sm.append(float(r[0]))
            self.smax.append(float(r[1]))
            for name, val in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                  "sw_power_cap"], r[2:6]):
                if val.lower() == "active":
                    self.reasons.add(name)
        except Exception:
            pass

    def stop(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock query unavailable"]}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.smax),
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml" if self.nv is not None else "nvidia-smi"}


def _sweep_bytes(problem):
    """Algorithmic HBM bytes of one sweep of A (X d or X^T v): A, labels, in/out vectors."""
    op = problem.q_op
    return 8 * op.n_phys * op.q + 8 * op.n_phys + 8 * (problem.n + op.q)


def _ncu_traffic():
    """DRAM read + write bytes per launch of the committed ncu --set full capture of
    the per-Newton-step sweep stream_xd_kernel<2> (X [t, r]; profiles/r1_ncu_stream_xd_kernel.txt),
    or None."""
    try:
        vals = {}
        with open(os.path.join(ROOT, "profiles", "r1_ncu_stream_xd_kernel.txt")) as fh:
            for line in fh:
                parts = line.split()
                if parts and parts[0] == "raw" and parts[1].startswith("dram__bytes_"):
                    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}[parts[2]]
                    vals[parts[1]] = float(parts[3]) * scale
        return vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    except Exception:
        return None


def cpu_oracle_solve(cfg):
    """Numpy restatement of the reference path (oracle/), stable psi evaluation."""
    import oracle as O

    O.set_psi_mode("delta")  # the product's default line search
    op, c, bl = O.csvc_problem(cfg["A"], cfg["y"], cfg["C"])
    t0 = time.perf_counter()
    rep = O.alm_solve(op, c, bl, O.AlmOpts(tol_kkt=TOL))
    return time.perf_counter() - t0, rep


def _threads():
    try:
        from threadpoolctl import threadpool_info

        return max(int(i.get("num_threads", 1)) for i in threadpool_info()) or 1
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_1910_01312_b200 import datagen

    cfg = datagen.make_config(args.config)
    for _ in range(args.warmup):
        cpu_oracle_solve(cfg)
    times = []
    rep = None
    for _ in range(args.steps):
        t, rep = cpu_oracle_solve(cfg)
        times.append(t)
    v = float(np.mean(times))
    cores = _threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Gaussian mixture, BASELINE config 1 shapes)",
        "config": {"workload": f"config{args.config}", "tol_kkt": TOL, "cold_start": True},
        "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "port",
                         "sample": "full solve of the workload per step (numpy oracle, OpenBLAS)"},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "result": {"kkt": rep["kkt_residual"], "objective": rep["objective"],
                   "outer": rep["outer_iters"], "inner": rep["total_inner_iters"],
                   "converged": rep["converged"]},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_1910_01312_b200 as P
    from paper_1910_01312_b200 import datagen

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    be = P.default_backend()
    cfg = datagen.make_config(args.config)
    A_host = torch.from_numpy(cfg["A"]).pin_memory()
    y_host = cfg["y"]
    A_dev = A_host.to("cuda")
    problem = P.build_csvc_dual(A_dev, y_host, cfg["C"])
    opts = P.AlmOptions(tol_kkt=TOL)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        rep = P.alm_solve(problem, opts)
    barrier()
    stream = torch.cuda.current_stream()
    sampler = ClockSampler(local_rank)
    sampler.start()
    launches0 = be.launch_count()
    step_s = []
    reps = []
    for _ in range(args.steps):
        flush.fill_(1)  # evict L2 between timed iterations
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rep = P.alm_solve(problem, opts, return_device=True)
        e1.record(stream)
        e1.synchronize()
        step_s.append(e0.elapsed_time(e1) * 1e-3)
        reps.append(rep)
        sampler.sample()
    launches = (be.launch_count() - launches0) // max(args.steps, 1)
    # per-op-class device time: the same K solves again with CUDA events around every
    # op on the solver stream (kept out of the timed region above: event records cost
    # host time the latency-bound solve would otherwise not pay)
    kern = {}
    prof_opts = P.SsnOptions(profile=True)
    prof_wall = []
    for _ in range(args.steps):
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        P.alm_solve(problem, opts, prof_opts, return_device=True)
        e1.record(stream)
        e1.synchronize()
        prof_wall.append(e0.elapsed_time(e1) * 1e-3)
        sampler.sample()
        for name, v in getattr(problem, "op_profile", {}).items():
            c, s, b = kern.get(name, (0, 0.0, 0.0))
            kern[name] = (c + v["calls"], s + v["seconds"], b + v["bytes"])
    clocks = sampler.stop()
    barrier()
    t_local = float(np.sum(step_s))
    t = torch.tensor([t_local], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total = float(t[0])
    value = total / args.steps

    # ---- end to end through the public API from host buffers
    e2e_times = []
    h2d = A_host.numel() * 8 + 3 * y_host.size * 8  # A, labels, box a; c
    d2h = y_host.size * 8
    for i in range(args.warmup + args.steps):
        flush.fill_(1)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        pb = P.build_csvc_dual(A_host, y_host, cfg["C"])
        r = P.alm_solve(pb, opts)  # x_opt copied to a host numpy array
        e1.record(stream)
        e1.synchronize()
        if i >= args.warmup:
            e2e_times.append(e0.elapsed_time(e1) * 1e-3)
        del pb
    te = torch.tensor([float(np.sum(e2e_times))], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = float(te[0]) / args.steps

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    peak, peak_kind = _peaks()
    # dominant op class by device time; roofline = its algorithmic bytes / its time
    roof = None
    ptotal = float(np.sum(prof_wall)) if prof_wall else 0.0
    if kern:
        # dominant HBM-bound kernel of the launch list (profiles/r1_launches_config1_solve.txt):
        # the streaming sweeps of A -- per Newton step ONE stream_xd<2> (X [t, r]: Qd and the
        # gradient), plus the inner-solve start (X^T s) and the KKT/refresh sweeps.
        # achieved = their algorithmic bytes / their device time, measured live here over
        # the K profiled solves (op classes dense_xt and dense_x hold exactly the sweeps);
        # traffic = DRAM bytes per launch of one ncu --set full capture of stream_xd<2>
        sweeps = [kern[k] for k in ("dense_xt", "dense_x") if k in kern]
        cnt = sum(v[0] for v in sweeps)
        secs = sum(v[1] for v in sweeps)
        nbytes = sum(v[2] for v in sweeps)
        achieved = (nbytes / secs) / 1e9 if secs > 0 and nbytes > 0 else 0.0
        roof = {"bound": "hbm",
                "kernel": "stream_xd_kernel<2> / stream_xd / stream_xt (sweeps of A)",
                "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak if peak else None,
                "traffic": _ncu_traffic(), "peak_kind": peak_kind, "op_calls": cnt,
                "algorithmic_bytes_per_sweep": _sweep_bytes(problem),
                "share_of_step": secs / ptotal if ptotal else None,
                "measured": "CUDA events on the solver stream, K extra profiled solves",
                "ops": {k: {"calls": v[0], "s": v[1], "share": v[1] / ptotal if ptotal else None,
                            "GBps": v[2] / v[1] / 1e9 if v[1] else None}
                        for k, v in kern.items()}}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        secs, ref = cpu_oracle_solve(cfg)
        cpu = {"value": secs, "unit": "s", "cores": _threads(), "kind": "port",
               "sample": "one full solve of the workload (numpy oracle, stable psi, OpenBLAS)",
               "kkt": ref["kkt_residual"], "objective": ref["objective"]}
    last = reps[-1]
    line = {
        "metric": METRIC, "value": value, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Gaussian mixture, BASELINE config 1 shapes)",
        "config": {"workload": f"config{args.config}", "n": problem.n, "q": problem.q_op.q,
                   "C": cfg["C"], "tol_kkt": TOL, "cold_start": True,
                   "l2": "flushed (256 MB write) before every timed step",
                   "parallelism": "replicas" if world > 1 else "single"},
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "result": {"kkt": last.kkt_residual, "objective": last.objective,
                   "outer": last.outer_iters, "inner": last.total_inner_iters,
                   "p": last.unbounded_support_count, "converged": last.converged},
        "counters": getattr(problem, "native_counters", None),
        "step_ms": [round(t * 1e3, 3) for t in step_s],
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import __graft_entry__

    __graft_entry__.build()
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
