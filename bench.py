#!/usr/bin/env python
"""Benchmark: Lloyd-preconditioned LBFGS SCVT iterations on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config c4]

Metric: generator-updates/s = iterations x N / time (BASELINE.json `metric`), workload
BASELINE.json configs[3] (c4: N=655,362 rho-sampled generators, tanh^4 density gamma=1/8,
7-point rule on 3-level subdivided fans, LBFGS m=7) on one GPU; the other configs are
parity-test cases.  A step is one optimizer iteration (one strong-Wolfe line search, ~1.0-1.1
evaluations).  W warm-up iterations continue the same trajectory before K timed ones.

`value` is device-timed (CUDA events on the launching stream, max over ranks), inputs resident
in HBM, L2 flushed between timed steps.  `e2e` is the same metric through the public API
(`minimize` from a pinned host array, per-iteration device->host copy of the positions).
`roofline` is for the dominant kernel (k_quad, FP64-bound) against the FP64 DFMA peak
measured in this run; `cpu_baseline` times the oracle restatement of the reference's own
region path on the host cores (bounded sample).  `--impl reference` times that CPU path alone.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (N, density preset, LBFGS m)   (BASELINE.json configs; 7pt rule, depth-3 fans)
    "c1": (2562, "const", 5),
    "c2": (40962, "const", 7),
    "c3": (163842, "c3", 7),
    "c4": (655362, "c4", 7),
    "c5": (2621442, "c5", 10),
}
METRIC = "generator-updates/s (Lloyd-LBFGS iters x N) at N=655,362, 1/2/4/8 B200"
RULE, DEPTH, SEED = "7pt", 3, 0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-regions", type=int, default=0,
                    help="regions per CPU-baseline step (default: one per host core)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.at_end = False
        self.path = tempfile.mktemp(suffix=".csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            if not self._rows():
                # timed region shorter than the sampler's start-up + 100 ms period (c1, c2):
                # one query right at its end, while the clocks still reflect the load
                self.at_end = True
                try:
                    with open(self.path, "a") as f:
                        subprocess.run(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits"], stdout=f,
                                       stderr=subprocess.DEVNULL, timeout=10)
                except (OSError, subprocess.SubprocessError):
                    pass

    def _rows(self):
        rows = []
        try:
            for line in open(self.path):
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 9 and p[1].replace(".", "").isdigit():
                    rows.append(p)
        except OSError:
            pass
        return rows

    def summary(self):
        rows = self._rows()
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]),
               "reasons": reasons, "samples": len(rows)}
        if self.at_end:
            out["when"] = "end of the timed region (shorter than the 100 ms sampling period)"
        return out


# ----------------------------------------------------------------------------- CPU baseline
def _region_worker(args):
    payload, density = args
    from oracle import region as R

    ids, _, _, _ = R.region_task(payload, density, RULE, DEPTH)
    return len(ids)


class CpuRegionSample:
    """Bounded sample of the reference's region path (pipeline.py:62-98, 171-242) restated in
    oracle/region.py: each step integrates one Voronoi-sort region per host core in a fork
    pool; value = owned generators integrated / wall (= generator-updates/s at 1 eval/iter)."""

    def __init__(self, cfg, regions_per_step=0, p=1024):
        import multiprocessing as mp

        import oracle as O
        from oracle import region as R

        n, dname, _ = CONFIGS[cfg]
        self.density = O.density_for(dname)
        self.z = O.sample_by_density(self.density, n, SEED)
        self.p = min(p, max(8, n // 160))
        self.centers, self.one = R.bootstrap_covering(self.p, SEED, self.density)
        self.geo = R.nearest_cell(self.z, self.centers)
        self.cores = os.cpu_count() or 1
        self.per_step = regions_per_step or self.cores
        self.pool = mp.get_context("fork").Pool(self.cores)
        self.next = 0
        self.R = R

    def step(self):
        t0 = time.perf_counter()          # payload assembly (pipeline.py:171-197) is timed too
        jobs = []
        for _ in range(self.per_step):
            l = self.next % self.p
            self.next += 1
            jobs.append((self.R.region_payload(self.z, self.geo, self.centers, self.one, l),
                         self.density))
        owned = sum(self.pool.map(_region_worker, jobs))
        return owned, time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()


def workload(cfg: str) -> str:
    """The workload string both arms report (the same configuration)."""
    n, dname, m = CONFIGS[cfg]
    return (f"{cfg}: N={n}, {dname} density, {RULE} rule on depth-{DEPTH} subdivided fans, "
            f"Lloyd-P-LBFGS m={m}")


def cpu_measure(cfg, steps, warmup, regions=0, evals_per_iteration=1.0):
    s = CpuRegionSample(cfg, regions)
    try:
        for _ in range(warmup):
            s.step()
        tot_owned, tot_t = 0, 0.0
        for _ in range(steps):
            o, t = s.step()
            tot_owned += o
            tot_t += t
        return {"value": tot_owned / tot_t / evals_per_iteration,
                "ms_per_step": tot_t / max(steps, 1) * 1e3,
                "unit": "generator-updates/s", "cores": s.cores,
                "kind": "port",
                "sample": (f"oracle restatement of the reference region path (covering p={s.p}, "
                           f"Voronoi-sort regions, cap Delaunay via SciPy/Qhull, 7pt on depth-3 "
                           f"fans); {steps} steps x {s.per_step} regions on a {s.cores}-process "
                           f"pool, {tot_owned} owned generators integrated in {tot_t:.2f} s "
                           f"(payload assembly included); generator-updates = generator "
                           f"evaluations / {evals_per_iteration:.2f} evaluations per iteration "
                           f"(the GPU arm's measured rate; the reference's own default covering "
                           f"p = default_partitions(N) = 64 regions would take ~40 s per region "
                           f"task, so a step samples a finer covering of the same path)")}
    finally:
        s.close()


def run_reference(a):
    rank, _, _ = dist_env()
    if rank != 0:
        return
    n = CONFIGS[a.config][0]
    cb = cpu_measure(a.config, a.steps, a.warmup, a.cpu_sample_regions)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": cb["unit"],
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            # wall time of one step = one bounded sample (cores regions) of the workload
            "ms_per_step": cb["ms_per_step"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded rho-sampling, seed 0)",
            "config": {"workload": workload(a.config), "N": n,
                       "implementation": "reference algorithm on the host CPU cores "
                                         "(region path, fork pool)"},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- B200 arm
def run_b200(a):
    import torch

    import paper_1709_06924_b200 as P
    from paper_1709_06924_b200 import _lib
    import ctypes

    rank, world, local = dist_env()
    # SCVT_BENCH_FUNCTIONAL=1: every rank on cuda:0 with gloo collectives — a functional check
    # of the multi-rank path on a one-GPU box (the numbers it prints mean nothing)
    functional = os.environ.get("SCVT_BENCH_FUNCTIONAL") == "1"
    if functional:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    n, dname, m = CONFIGS[a.config]
    density = P.density_preset(dname)
    z0 = P.sample_by_density(density, n, SEED)               # host init (PCG64 parity)
    if world > 1:   # sharded evaluation, NCCL all-gathers (paper_1709_06924_b200/parallel.py)
        ev = P.ShardedMeshEvaluator(density, RULE, subdivision=DEPTH, device=local)
    else:
        ev = P.MeshEvaluator(density, RULE, subdivision=DEPTH, device=local)
    st = P.Minimizer(torch.from_numpy(z0).to(dev), "lloyd-plbfgs", ev, m)
    ctx = ev.context
    lib = _lib.load()
    # FP64 peak of this device (roofline denominator; not in MEASURED_PEAKS.json)
    peak = ctypes.c_double()
    _lib.check(lib.scvt_fp64_peak(local, ctypes.byref(peak)), None, "fp64 peak")
    for _ in range(a.warmup):
        st.step()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    lib.scvt_profile_enable(ctx.ptr, 1)
    ms = (ctypes.c_double * 3)()
    cnt = (ctypes.c_int64 * 3)()
    lib.scvt_profile_read(ctx.ptr, ms, cnt, 1)
    launches0 = ctx.launches()
    fev0 = st.fevals
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    step_ms = []
    recs = []
    with ClockSampler(local) as clk:
        for _ in range(a.steps):
            flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            rec, _, _, _ = st.step()
            e1.record()
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            recs.append(rec)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches = ctx.launches() - launches0
    evals = st.fevals - fev0
    lib.scvt_profile_read(ctx.ptr, ms, cnt, 1)
    lib.scvt_profile_enable(ctx.ptr, 0)
    total_ms = sum(step_ms)
    if world > 1:
        total_ms = _max_over_ranks(total_ms, dev)
    # strong scaling: the N generators are shared by all ranks; each iteration updates N
    value = a.steps * n / (total_ms * 1e-3)
    import oracle as O

    flops_eval = O.algorithmic_flops(n, 7, DEPTH, density.variant) / world   # this rank's share
    quad_ms = ms[1] / max(cnt[1], 1)
    achieved = flops_eval / (quad_ms * 1e-3) / 1e12 if quad_ms > 0 else float("nan")
    roofline = {"bound": "fp64", "kernel": "k_quad", "achieved": achieved, "peak": peak.value,
                "unit": "TFLOP/s", "frac": achieved / peak.value,
                "peak_source": "measured in this run: scvt_fp64_peak DFMA microbenchmark "
                               "(MEASURED_PEAKS.json has no FP64 entry)",
                "flops_per_launch": flops_eval, "avg_launch_ms": quad_ms,
                "share_of_step": ms[1] / total_ms if world == 1 else None,
                "cells_ms_per_eval": ms[0] / max(cnt[0], 1),
                "eval_ms": ms[2] / max(cnt[2], 1),
                "traffic": _traffic_from_profiles(a.config),
                # the whole iteration against the same peak (all kernels, host
                # round trips and idle time included)
                "step_frac": (flops_eval * world * evals / a.steps) / (total_ms / a.steps * 1e-3)
                             / 1e12 / peak.value}
    pipe = _profile_value("k_quad_fp64_pipe_active_pct", a.config)
    if pipe is not None:
        roofline["fp64_pipe_active_pct_ncu"] = pipe
        # the same utilisation against the measured peak: the DFMA microbenchmark itself keeps
        # the pipe peak / nominal busy (nominal = SMs x 64 FMA x 2 x max SM clock)
        props = torch.cuda.get_device_properties(dev)
        nominal = props.multi_processor_count * 64 * 2 * (clk.summary()["sm_max_mhz"] or 0) * 1e6 / 1e12
        if nominal > 0:
            roofline["frac_pipe"] = pipe / 100.0 / (peak.value / nominal)
    if dname != "const":
        roofline["note"] = (
            "frac is ALGORITHMIC FLOPs (SURVEY 8(d): the reference's closed-form density at "
            "every node, both centres for the two-centre kind) over the measured DFMA peak; "
            "k_quad evaluates a per-patch polynomial fit of rho (degree 4-6, one centre where it "
            "dominates the patch) with fewer FP64 instructions than that count charges, so frac "
            "can exceed 1 -- the hardware utilisation is fp64_pipe_active_pct_ncu (ncu "
            "sm__pipe_fp64_cycles_active of the same kernel, profiles/), and frac_pipe is that "
            "utilisation over the one the peak microbenchmark itself reaches")
    line = {"metric": METRIC, "value": value, "unit": "generator-updates/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": total_ms / a.steps,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (rho-sampled generators, default_rng seed 0)",
            "config": {"workload": workload(a.config),
                       "N": n, "iteration_window": f"{a.warmup + 1}..{a.warmup + a.steps}",
                       "evals_per_iteration": evals / a.steps,
                       "l2": "flushed (256 MB write) before every timed step",
                       "parallelism": "single GPU" if world == 1 else
                       f"dp{world}: cells sharded in cube-map order (NCCL all-gathers of flip "
                       f"candidates, rebuilt cycles and per-generator moments), optimizer "
                       f"vectors in arithmetic layout (chunk partials all-reduced, positions "
                       f"all-gathered)"},
            "roofline": roofline, "gpu_launches": launches,
            "clocks": clk.summary()}
    # e2e through the public API with host buffers
    if not a.no_e2e:
        line["e2e"] = _e2e(P, density, z0, m, a.steps, dev, world)
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_measure(a.config, 2, 1,
                                           evals_per_iteration=max(evals / a.steps, 1.0))
    ev.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def _max_over_ranks(x: float, dev) -> float:
    import torch
    import torch.distributed as dist

    gloo = dist.get_backend() == "gloo"
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if gloo else dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _e2e(P, density, z0, m, steps, dev, world):
    """`minimize` from a pinned host array; every iteration copies the positions back."""
    import torch

    host = torch.from_numpy(z0).pin_memory()
    outs = [torch.empty_like(host).pin_memory() for _ in range(2)]
    crit = P.StoppingCriteria(max_iterations=steps, movement_tol=1e-300, grad_tol=1e-300,
                              stall_tol=1e-300)
    side = torch.cuda.Stream(device=dev)
    snaps, done = [], [None, None]

    def cb(n, z, res):
        # snapshot on the compute stream (D2D), then the PCIe copy on a side stream so it
        # overlaps the next iteration; double-buffered, each buffer reused only after its copy
        k = n % 2
        while len(snaps) < 2:
            snaps.append(torch.empty_like(z))
        main = torch.cuda.current_stream(dev)
        if done[k] is not None:
            main.wait_event(done[k])
        snaps[k].copy_(z)
        ready = torch.cuda.Event()
        ready.record(main)
        side.wait_event(ready)
        with torch.cuda.stream(side):
            outs[k].copy_(snaps[k], non_blocking=True)
        done[k] = torch.cuda.Event()
        done[k].record(side)

    cls = P.ShardedMeshEvaluator if world > 1 else P.MeshEvaluator
    # untimed warm-up of the API (process-wide caching allocators: pinned result staging,
    # snapshot buffers) on a separate evaluator, so the timed one starts cold (no cycles)
    with cls(density, RULE, subdivision=DEPTH, device=dev.index) as warm:
        P.minimize(host.to(dev, non_blocking=True), "lloyd-plbfgs", warm,
                   P.StoppingCriteria(max_iterations=2, movement_tol=1e-300, grad_tol=1e-300,
                                      stall_tol=1e-300), corrections=m, callback=cb)
    done[0] = done[1] = None
    with cls(density, RULE, subdivision=DEPTH, device=dev.index) as ev:
        torch.cuda.synchronize()
        tw = time.perf_counter()
        ev._ensure_ctx(len(z0), m)     # one-time workspace allocation: timed on its own
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ws = t0 - tw
        zdev = host.to(dev, non_blocking=True)
        res = P.minimize(zdev, "lloyd-plbfgs", ev, crit, corrections=m, callback=cb)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    n = len(z0)
    if world > 1:
        wall = _max_over_ranks(wall, dev)
        ws = _max_over_ranks(ws, dev)
    return {"value": steps * n / wall, "unit": "generator-updates/s",
            "h2d_bytes_per_step": int(24 * n / steps), "d2h_bytes_per_step": int(24 * n),
            # the evaluator's one device allocation (once per evaluator, not per call)
            "workspace_alloc_ms": ws * 1e3,
            "value_incl_workspace_alloc": steps * n / (wall + ws),
            "note": f"minimize() from a pinned host array (H2D inside the timing), iterations "
                    f"1..{steps} from the initial point incl. the initial evaluation "
                    f"({res.fevals} evaluations), every iteration copies the positions to pinned "
                    f"host memory (device snapshot, then PCIe copy on a side stream overlapping "
                    f"the next iteration); the evaluator's device workspace (one cudaMalloc, once per "
                    f"evaluator) is allocated before the timing and reported beside it "
                    f"(workspace_alloc_ms, value_incl_workspace_alloc); one untimed "
                    f"2-iteration warm-up call on a separate evaluator (allocator warm-up)"}


def _profile_value(key, config=None):
    """A number from the committed ncu summary (profiles/roofline_traffic.json): ncu cannot
    run inside the timed bench, so its figures are read from the capture of the same build."""
    p = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    try:
        with open(p) as f:
            v = json.load(f).get(key)
    except (OSError, ValueError):
        return None
    return v.get(config) if isinstance(v, dict) else v


def _traffic_from_profiles(config="c4"):
    return _profile_value("k_quad_dram_bytes_per_launch", config)


def _free_port() -> int:
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(a) -> int:
    """`--gpus N` without a torchrun environment: re-launch this command as N ranks (one
    process per GPU) under torch.distributed.run on 127.0.0.1, as the driver would."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__), *sys.argv[1:]]
    print(f"[bench] spawning {a.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def run_functional_cpu(a):
    """SCVT_BENCH_FUNCTIONAL=1 on a box without CUDA: exercises the launch path only (N ranks
    spawned, gloo rendezvous, barriers, max over ranks, one line from rank 0); no number."""
    import torch
    import torch.distributed as dist

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
        dist.barrier()
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "generator-updates/s",
                          "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
                          "functional": "no CUDA device: launch path only",
                          "max_over_ranks_probe": float(t.item())}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = parse()
    if a.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(a))
    _, world, _ = dist_env()
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}: one rank per GPU")
    if a.impl == "reference":
        run_reference(a)
        return
    import torch

    if os.environ.get("SCVT_BENCH_FUNCTIONAL") == "1" and not torch.cuda.is_available():
        run_functional_cpu(a)
        return
    run_b200(a)


if __name__ == "__main__":
    main()
