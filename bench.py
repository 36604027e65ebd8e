#!/usr/bin/env python
"""TT-rounding benchmark (BASELINE.json metric "TT-rounding core GB/s").

Workload (BASELINE.json configs[2], the 2 GB-class tensor the metric and the
north-star target are quoted on): Y random TT, d=10, n=8000 per mode,
ranks 30, fp64 N(0,1) (the reference's random_tt seed 0, drawn on the device); X = Y + Y (ranks
60, 1.85 GB of cores, built by our add kernel outside the timed region);
one step = round_tt(X, RoundingOptions(1e-10, "LRLI")) -> ranks 30.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched with torchrun; every rank holds its block_bounds slices of
every core (the paper's 1 x P x 1 distribution) and the value is the whole
tensor's algorithmic bytes over the max-over-ranks step time.

value       = B_alg / t_step, B_alg = 8 (2|X| + |Y_out|)
e2e         = same metric through the public host API (round_tt_host) from
              page-locked host cores into page-locked output buffers: H2D of
              X and D2H of the result inside every timed step, overlapped
              with the sweeps by the library
roofline    = dominant kernel class (TSQR leaf factorization), fp64-bound:
              reference Householder flops / its CUDA-event time, against the
              measured fp64 peak of this device (ttb_fp64_peak)
cpu_baseline= the CPU restatement of the reference (oracle/, numpy + scipy
              LAPACK, all host threads) on the same X, rank 0 only
--impl reference: that CPU path alone, on the same full workload
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

HBM_PEAK_FALLBACK = 6545.6  # GB/s, MEASURED_PEAKS.json hbm_gbs at round start

CONFIGS = {
    # name: (dims, Y ranks, how X is formed, eps0, max_rank)
    "cfg1": ((2000,) * 8, 10, "y+y", 1e-10, None),
    "cfg3": ((8000,) * 10, 30, "y+y", 1e-10, None),
}


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_PEAK_FALLBACK, "fallback"


def chain(cfg):
    dims, r, _, _, _ = CONFIGS[cfg]
    N = len(dims)
    ry = (1,) + (r,) * (N - 1) + (1,)
    rx = (1,) + (2 * r,) * (N - 1) + (1,)
    return dims, ry, rx


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index, enabled=True):
        self.index = index
        self.enabled = enabled
        self.lines = []
        self.proc = None
        self.window = None

    def __enter__(self):
        """Start nvidia-smi (20 ms sampling) and wait until it delivers its
        first sample, so the timed region that follows is covered."""
        if not self.enabled:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 10.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def start(self):
        """Mark the start of the timed region (samples before it are dropped)."""
        self.window = [time.time(), None]

    def stop(self):
        if self.window is not None:
            self.window[1] = time.time()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.window is not None and self.window[1] is not None:
            inside = [ln for t, ln in lines if self.window[0] <= t <= self.window[1]]
            lines = inside if inside else [ln for _, ln in lines[:1]]  # region shorter than one sample
        else:
            lines = [ln for _, ln in lines]
        for ln in lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def make_input(T, comm, cfg, seed=0):
    """Y = the reference's random_tt(dims, ranks, seed) restricted to this
    rank's slices, generated on the device bitwise equal to the host
    generator (ttb_fill_random; core.py:250-282), and X = Y + Y."""
    dims, ry, _ = chain(cfg)
    y = T.DistTTTensor.random(comm, dims, ry, seed)
    return y, T.add(y, y)


def leaf_traffic():
    """DRAM bytes (read + write) of one leaf launch from the committed ncu
    --set full capture (profiles/*_leaf_ncu.json, newest round), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r*_leaf_ncu.json")))
    if not files:
        return None
    try:
        d = json.load(open(files[-1]))
        return {"bytes_per_launch": (d["dram_read_MB"] + d["dram_write_MB"]) * 1e6,
                "algorithmic_bytes_per_launch": d["algorithmic_MB"] * 1e6,
                "launch": d["launch"], "source": os.path.relpath(files[-1], os.path.dirname(os.path.abspath(__file__)))}
    except Exception:
        return None


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2011_06532_b200 as T
    from paper_2011_06532_b200 import _lib, cost

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
        comm = T.DistComm()
    else:
        comm = T.SerialComm(torch.device("cuda", local))
    cfg = args.config
    dims, ry, rx = chain(cfg)
    eps0, maxr = CONFIGS[cfg][3], CONFIGS[cfg][4]
    opts = T.RoundingOptions(eps0, "LRLI", maxr)
    y, x = make_input(T, comm, cfg)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=comm.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # warm-up (also validates the result ranks)
    out = None
    for _ in range(max(args.warmup, 1)):
        out = T.round_tt(x, opts)
    torch.cuda.synchronize()
    out_ranks = out.ranks
    assert out_ranks == ry, f"rounding returned ranks {out_ranks}, expected {ry}"
    del out

    # timed region: inputs resident in HBM (1.85 GB of cores > 126 MB L2)
    barrier()
    torch.cuda.synchronize()
    l0 = _lib.launch_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local, enabled=os.environ.get("TTB_BENCH_NO_SMI") is None) as clk:
        clk.start()
        e0.record(stream)
        for _ in range(args.steps):
            out = T.round_tt(x, opts)
        e1.record(stream)
        torch.cuda.synchronize()
        clk.stop()
    launches = _lib.launch_counter() - l0
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    del out
    B = cost.rounding_bytes(dims, rx, ry)
    F = cost.rounding_flops(dims, rx, ry, "LRLI")
    value = B / (ms * 1e-3) / 1e9

    # end-to-end through the public host API (round_tt_host: the drop-in for
    # the reference's numpy-level call) from page-locked host cores into
    # page-locked output buffers: every step uploads all input cores and
    # downloads all output cores inside the timed region (the transfers
    # overlap the sweeps inside the call)
    host_cores = [s.detach().permute(2, 1, 0).contiguous().permute(2, 1, 0).cpu().pin_memory() for s in x.local]
    host_out = [torch.empty(c.numel(), dtype=torch.float64).pin_memory() for c in host_cores]
    h2d = sum(c.numel() * 8 for c in host_cores)
    e2e_ms = []
    d2h = 0
    for it in range(args.warmup + args.steps):
        barrier()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        bev = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        res, md = T.round_tt_host(host_cores, opts, comm=comm, out=host_out)
        bev.record(stream)
        torch.cuda.synchronize()
        assert md["output_ranks"] == ry, md
        d2h = sum(r.numel() * 8 for r in res)
        if it >= args.warmup:
            e2e_ms.append(a.elapsed_time(bev))
        del res
    e2e_t = max_over_ranks(float(np.mean(e2e_ms)))
    e2e = {"value": B / (e2e_t * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_t,
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
           "api": "round_tt_host (ttb_round_host), page-locked host cores in and out"}
    # the plain drop-in call a reference user makes: pageable numpy cores in,
    # freshly allocated numpy cores out (the library registers / pins per call)
    np_cores = [np.array(c.numpy(), order="F", copy=True) for c in host_cores]  # pageable copies
    pg_ms = []
    for it in range(1 + min(args.steps, 3)):
        barrier()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        bev = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        res, md = T.round_tt_host(np_cores, opts, comm=comm)
        bev.record(stream)
        torch.cuda.synchronize()
        assert md["output_ranks"] == ry, md
        if it >= 1:
            pg_ms.append(a.elapsed_time(bev))
        del res
    pg_t = max_over_ranks(float(np.mean(pg_ms)))
    e2e["pageable"] = {"value": B / (pg_t * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": pg_t, "steps": len(pg_ms),
                       "api": "round_tt_host(numpy cores) -- pageable input, output allocated per call"}
    del np_cores

    # dominant-kernel roofline from one instrumented (event-timed) step
    dfma, dmma = _lib.fp64_peak(stream.cuda_stream)
    _lib.prof_enable(True)
    o = T.round_tt(x, opts)
    torch.cuda.synchronize()
    prof = _lib.prof_dump()
    _lib.prof_enable(False)
    del o
    leaf_ms = prof.get("tsqr_leaf", (1, float("nan")))[1]
    leaf_launch = prof.get("tsqr_leaf", (1, 0))[0]
    leaf_f = cost.tsqr_leaf_flops(dims, rx, ry, "LRLI") / max(world, 1)
    fp64_peak = max(dfma, dmma)
    achieved = leaf_f / (leaf_ms * 1e-3) / 1e12
    peak_hbm, peak_src = hbm_peak()
    roofline = {"bound": "fp64", "kernel": "tsqr_leaf (Householder TSQR leaf chains)",
                "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                "traffic": (leaf_traffic() or {}).get("bytes_per_launch"), "traffic_detail": leaf_traffic(),
                "peak_source": "measured fp64 (ttb_fp64_peak: DFMA %.1f, DMMA %.1f TF/s)" % (dfma, dmma),
                "launches": leaf_launch, "ms_per_step": leaf_ms,
                "share_of_step": leaf_ms / ms if ms else None}
    step_roofline = {"hbm_frac": value / peak_hbm, "hbm_peak_gbs": peak_hbm, "hbm_peak_source": peak_src,
                     "fp64_frac": (F / (ms * 1e-3) / 1e12) / fp64_peak,
                     "kernel_ms": {k: round(v[1], 3) for k, v in prof.items()}}

    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        o = T.round_tt(x, opts)
        torch.cuda.synchronize()
        cpu, parity = cpu_baseline_same_input(x, o, dims, rx, ry, eps0, maxr)
        del o
    norms = None
    if not args.no_norm:
        del x, y
        torch.cuda.synchronize()
        norms = measure_norms(T, comm)

    clocks = clk.summary()
    line = {
        "metric": "TT-rounding core GB/s",
        "value": value,
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: the reference generator's seeded N(0,1) cores (random_tt, seed 0), drawn on the device bitwise",
        "config": {"workload": f"{cfg}: round_tt(X = Y + Y) d={len(dims)} n={dims[0]} ranks {rx[1]}->{ry[1]}, "
                               f"tol {eps0}, LRLI", "dims": list(dims), "in_ranks": list(rx),
                   "out_ranks": list(ry), "parallelism": f"mode-sliced P={world}",
                   "l2": "inputs larger than L2 (X = %.2f GB of cores)" % (sum(cost.core_sizes(dims, rx)) * 8 / 1e9),
                   "algorithmic_bytes": B, "algorithmic_flops": F},
        "e2e": e2e,
        "gpu_launches": int(launches // max(args.steps, 1)) if args.steps else 0,
        "gpu_launches_total": int(launches),
        "roofline": roofline,
        "step_roofline": step_roofline,
        "cpu_baseline": cpu,
        "parity": parity,
        "norm": norms,
        "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def threadpool_desc():
    try:
        from threadpoolctl import threadpool_info
        return [{k: d.get(k) for k in ("internal_api", "num_threads", "version")} for d in threadpool_info()]
    except Exception:
        return None


def cpu_baseline_same_input(x, out, dims, rx, ry, eps0, maxr):
    """The reference on the same X, all host threads; one step (~6 s on 16
    cores for cfg3): the unmodified package staged under baseline/_ref
    (ttpar.round_tt(serial_tt(X)), kind "reference") when present, else its
    CPU restatement (oracle/, kind "port").  Its result is also the full-size
    parity check of the GPU output ``out``:
    ranks identical, TT-form relative difference by the ortho route (computed
    with the oracle's error routine), and the norm."""
    from oracle import tt_oracle as O

    cores = [np.asfortranarray(s.detach().cpu().numpy()) for s in x.local]
    threads = os.cpu_count() or 1
    ttpar = _load_ttpar()
    t0 = time.perf_counter()
    if ttpar is not None:
        ro = ttpar.round_tt(ttpar.serial_tt(ttpar.TTTensor(cores)), ttpar.RoundingOptions(eps0, "LRLI", maxr))
        dt = time.perf_counter() - t0
        ref, meta = [np.asfortranarray(c.array) for c in ttpar.gather(ro).cores], ro.meta
        kind, what = "reference", "ttpar.round_tt(serial_tt(X)) from baseline/_ref (the unmodified reference package"
    else:
        ref, meta = O.round_tt(cores, eps0, "LRLI", maxr)
        dt = time.perf_counter() - t0
        kind, what = "port", "oracle.round_tt (the oracle port: baseline/_ref is absent"
    from paper_2011_06532_b200 import cost

    B = cost.rounding_bytes(dims, rx, ry)
    got = [np.asfortranarray(s.detach().cpu().numpy()) for s in out.local]
    rel = O.rel_diff(got, ref)
    parity = {"against": kind, "ranks_equal": tuple(out.ranks) == O.ranks_of(ref), "rel_err_ortho": rel,
              "norm_rel": abs(out.meta["norm"] - meta["norm"]) / meta["norm"],
              "bar": "ranks identical, rel_err_ortho <= 1e-10, norm_rel <= 1e-12",
              "pass": bool(tuple(out.ranks) == O.ranks_of(ref) and rel <= 1e-10
                           and abs(out.meta["norm"] - meta["norm"]) <= 1e-12 * meta["norm"])}
    cpu = {"value": B / dt / 1e9, "unit": "GB/s", "cores": threads, "kind": kind,
           "sample": f"the full workload, 1 step ({dt:.1f} s): {what}; numpy + scipy LAPACK/OpenBLAS, "
                     f"{threads} threads) on the same X copied to host",
           "threadpools": threadpool_desc()}
    return cpu, parity


def measure_norms(T, comm, reps=5):
    """BASELINE's second metric, "norm GB/s": the Gram sweep on cfg2 (d=16,
    n=100000, ranks 16; X, Z the reference's random_tt seeds 0 / 1, drawn on
    the device).  GB/s = algorithmic bytes (8 |X| (+ 8 |Z|)) / device time,
    CUDA events around each call (each returns a host scalar)."""
    import torch

    from paper_2011_06532_b200 import cost

    dims, r = (100_000,) * 16, (1,) + (16,) * 15 + (1,)
    x = T.DistTTTensor.random(comm, dims, r, 0)
    z = T.DistTTTensor.random(comm, dims, r, 1)
    bx = 8.0 * sum(cost.core_sizes(dims, r))
    calls = {"inner_xz": (lambda: T.inner_product(x, z), 2 * bx),
             "norm_innerprod": (lambda: T.norm(x, "innerprod"), bx),
             "norm_innerprod_sym": (lambda: T.norm(x, "innerprod_sym"), bx),
             "norm_ortho": (lambda: T.norm(x, "ortho"), bx)}
    res = {"workload": "cfg2: d=16, n=100000, ranks 16 (X, Z: random_tt seeds 0, 1)", "unit": "GB/s"}
    stream = torch.cuda.current_stream()
    for name, (fn, nbytes) in calls.items():
        for _ in range(2):
            fn()
        ts = []
        for _ in range(reps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        gbs = nbytes / (ms * 1e-3) / 1e9
        # the Gram sweep is HBM-bound: fraction of the measured copy bandwidth
        res[name] = {"value": gbs, "ms": ms, "bytes": nbytes, "hbm_frac": gbs / hbm_peak()[0]}
    res["hbm_peak_gbs"], res["hbm_peak_source"] = hbm_peak()
    del x, z
    torch.cuda.synchronize()
    return res


# ---------------------------------------------------------------------------
# reference arm: the CPU path alone
# ---------------------------------------------------------------------------
def _load_ttpar():
    """The UNMODIFIED reference package staged under baseline/_ref (pip install
    --target of /root/reference/pkg), or None."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "ttpar")):
        return None
    sys.path.insert(0, ref)
    try:
        import ttpar  # noqa: F401
        return ttpar
    except Exception:
        sys.path.remove(ref)
        return None


def run_reference(args):
    rank, world, local = env_rank()
    if rank != 0:
        return
    from paper_2011_06532_b200 import cost

    cfg = args.config
    dims, ry, rx = chain(cfg)
    eps0, maxr = CONFIGS[cfg][3], CONFIGS[cfg][4]
    # the full workload (same config as our arm): ~6 s per step on 16 host
    # cores, so the default --steps/--warmup run takes a few minutes
    n = dims[0]
    sdims = dims
    ttpar = _load_ttpar()
    t0 = time.perf_counter()
    if ttpar is not None:
        # the reference's own public API and stock code path:
        # round_tt(serial_tt(X), RoundingOptions(...)), parallel.py:293
        y = ttpar.random_tt(sdims, ry, 0)
        t_gen = time.perf_counter() - t0
        x = ttpar.serial_tt(ttpar.add(y, y))
        opts = ttpar.RoundingOptions(eps0, "LRLI", maxr)
        step = lambda: ttpar.round_tt(x, opts)  # noqa: E731
        ranks_of = lambda o: tuple(o.ranks)  # noqa: E731
        kind, what = "reference", "ttpar.round_tt(serial_tt(X)) from baseline/_ref (the unmodified reference package"
    else:
        from oracle import tt_oracle as O

        y = O.random_cores(sdims, ry, 0)
        t_gen = time.perf_counter() - t0
        x = O.add(y, y)
        step = lambda: O.round_tt(x, eps0, "LRLI", maxr)[0]  # noqa: E731
        ranks_of = O.ranks_of
        kind, what = "port", "oracle.round_tt (the oracle port: baseline/_ref is absent"
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        out = step()
        if it >= args.warmup:
            times.append(time.perf_counter() - t0)
    assert ranks_of(out) == tuple(ry)
    B = cost.rounding_bytes(sdims, rx, ry)
    t = float(np.mean(times))
    value = B / t / 1e9
    threads = os.cpu_count() or 1
    line = {
        "impl": "reference",
        "metric": "TT-rounding core GB/s",
        "value": value,
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded N(0,1) TT cores)",
        "config": {"workload": f"{cfg}: round_tt(X = Y + Y) d={len(dims)} n={dims[0]} ranks {rx[1]}->{ry[1]}, "
                               f"tol {eps0}, LRLI", "dims": list(sdims), "in_ranks": list(rx),
                   "out_ranks": list(ry), "same_config": True},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": kind,
                         "sample": f"the full workload (n={n}, same X as our arm: random_tt seed 0, X = Y + Y), "
                                   f"{what}; numpy + scipy LAPACK/OpenBLAS, {threads} threads), "
                                   f"mean of {args.steps} steps; input generation {t_gen:.1f} s untimed",
                         "threadpools": threadpool_desc()},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg3")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg (and its parity check)")
    ap.add_argument("--no-norm", action="store_true", help="skip the cfg2 norm GB/s leg")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
